#!/usr/bin/env bash
# Same-box A/B of the working tree against .ab_head (a worktree of an earlier commit).
set -u
A="--no-ramp --no-other --scheduler-frames 0 --pt-steps 0 --train-steps 0 --decode-n 0 --uncached-steps 0 --no-cpu-baseline --no-e2e --config1 0 --config4-frames 0 --config5-steps 0 ${BENCH_ARGS:-}"
for rep in 1 2; do
  for t in . .ab_head; do
    (cd $t && timeout 300 python bench.py $A > /tmp/ab.json 2>/tmp/ab.err; python -c "
import json;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); c=d.get('config3') or {}
print('$t', round(d['value'],1), 'c3', round((c.get('throughput') or {}).get('fps',0),1), round((c.get('parity') or {}).get('fps',0),1))" || tail -3 /tmp/ab.err)
  done
done
