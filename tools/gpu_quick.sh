#!/usr/bin/env bash
# GPU quick check: parity tests, default-schedule bench (+trace), stage-timing stats run.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
for s in ${SCHEDULES:-0}; do
  CINR_TRACE=gpurun_out/trace$s.json timeout 300 python bench.py --schedule $s --steps 20 --warmup 5 \
      --no-cpu-baseline --decode-n 0 > gpurun_out/bench_t$s.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_t$s.json'));print('sched $s', round(d['value'],1), 'fps, e2e', round(d['e2e']['value'],1), 'march us', round(d['roofline']['avg_launch_us']))"
done
if [ -n "${STATS:-}" ]; then
  CINR_STATS=1 CINR_BENCH_VERBOSE=1 timeout 300 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --no-e2e \
      --decode-n 0 > gpurun_out/bench_stats.json 2> gpurun_out/bench_stats.err
  grep -E "counters" gpurun_out/bench_stats.err | tail -1
fi
