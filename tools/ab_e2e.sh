#!/usr/bin/env bash
# Same-box A/B of the end-to-end (host image) fps: working tree vs .ab_head.
set -u
A="--no-ramp --no-other --scheduler-frames 0 --pt-steps 0 --train-steps 0 --decode-n 0 --uncached-steps 0 --no-cpu-baseline --config1 0 --config4-frames 0 --config5-steps 0 --config3-steps 0 ${BENCH_ARGS:-}"
for rep in 1 2; do
  for t in . .ab_head; do
    (cd $t && timeout 300 python bench.py $A > /tmp/ab.json 2>/tmp/ab.err; python -c "
import json;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
print('$t', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))" || tail -3 /tmp/ab.err)
  done
done
