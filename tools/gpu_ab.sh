#!/usr/bin/env bash
# A/B of frame-kernel schedules + selected GPU tests (args: pytest selection).
set -u
mkdir -p gpurun_out
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest $TESTS -x -q > gpurun_out/pytest_sel.log 2>&1
  echo "pytest rc $?"; tail -30 gpurun_out/pytest_sel.log | grep -vE "^\s*$" | tail -25
fi
for s in ${SCHEDULES:-0}; do
  timeout 300 python bench.py --schedule $s --steps ${STEPS:-20} --warmup ${WARMUP:-5} --no-cpu-baseline --decode-n 0 \
      --pt-steps 0 --train-steps 0 --uncached-steps ${UNC:-3} ${BENCH_ARGS:-} > gpurun_out/bench_s$s.json 2> gpurun_out/bench_s$s.err
  python -c "
import json;d=json.loads(open('gpurun_out/bench_s$s.json').read().strip().splitlines()[-1])
u=d.get('uncached_inr_baseline') or {}
print('sched $s', round(d['value'],1), 'fps, e2e', round(d['e2e']['value'],1), 'march us', round(d['roofline']['avg_launch_us']), 'frac', round(d['roofline']['frac'],4), 'uncached', round(u.get('fps',0),1), 'spf', d['samples_per_frame'])" || tail -5 gpurun_out/bench_s$s.err
done
