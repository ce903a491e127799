#!/usr/bin/env bash
# usage: profile_kernel.sh <kernel-regex> <skip> <tag>  — one full ncu capture of a
# steady-state launch of the frame kernel (bench frame ~23).
set -u
K=${1:-k_wave_march}; S=${2:-22}; T=${3:-wave}
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 24 --no-cpu-baseline --no-e2e --decode-n 0 ${BENCH_EXTRA:-}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o gpurun_out/prof_$T -f python bench.py $ARGS > gpurun_out/ncu_$T.out 2>&1
echo done
