#!/usr/bin/env bash
# Round evidence on the GPU box: full bench line, reference arm, smoke, ncu launch
# list of a bench run and one full ncu capture of the frame kernel.
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --decode-n 0 --pt-steps 0 --uncached-steps 0 --train-steps 0 > gpurun_out/ncu_list.out 2>&1; echo "list rc $?"
bash tools/profile_kernel.sh k_wave3_march 22 wave3_r1; echo "full rc $?"
