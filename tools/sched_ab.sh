#!/usr/bin/env bash
# A/B of frame-kernel schedules on one box: bench value only, alternating.
for rep in 1 2; do
  for s in "$@"; do
    v=$(timeout 300 python bench.py --schedule $s --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --decode-n 0 \
        --uncached-steps 0 --pt-steps 0 --train-steps 0 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
    echo "schedule $s rep $rep: $v fps"
  done
done
