#!/usr/bin/env bash
# Same-box A/B: .ab_head (earlier commit) vs the working tree, plus env variants of the tree (VARIANTS="VAR=1 ...").
set -u
A="--no-ramp --no-other --scheduler-frames 0 --pt-steps 0 --train-steps 0 --decode-n 0 --uncached-steps 0 --no-cpu-baseline --no-e2e --config1 0 --config4-frames 0 --config5-steps 0 ${BENCH_ARGS:-}"
run() {  # dir label env
  (cd $1 && env $3 timeout 300 python bench.py $A > /tmp/ab.json 2>/tmp/ab.err; python -c "
import json;d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); c=d.get('config3') or {}
print('$2', round(d['value'],1), 'c3', round((c.get('throughput') or {}).get('fps',0),1))" || tail -3 /tmp/ab.err)
}
for rep in 1 2; do
  run .ab_head head X=0
  run . tree X=0
  for v in ${VARIANTS:-}; do run . "tree+$v" $v; done
done
