#!/usr/bin/env bash
# ncu capture of the chained march kernel (one steady-state frame) + launch list.
set -u
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 24 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_chain.csv python bench.py $ARGS > gpurun_out/ncu_list.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_march -s 22 -c 1 \
    -o gpurun_out/prof_chain -f python bench.py $ARGS > gpurun_out/ncu_full.out 2>&1
echo done
