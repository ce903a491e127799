#!/usr/bin/env bash
# Run on the GPU box (via gpurun): launch list + one full ncu capture of the
# ray-march iteration kernel.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
ARGS="--steps 2 --warmup 4 --no-cpu-baseline --no-e2e"
# 1) every launch of two steady-state frames (cold-cache, serialised: read SHARES)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1900 -c 1100 --csv \
    --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_list.out 2>&1
# 2) full section set on three early iterations of frame 4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march_iter -s ${SKIP:-925} -c 3 \
    -o gpurun_out/prof_march -f python bench.py $ARGS > gpurun_out/ncu_full.out 2>&1
echo done
