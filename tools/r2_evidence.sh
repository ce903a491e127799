#!/usr/bin/env bash
# Round-2 evidence on the GPU box: full bench line, reference arm, smoke, ncu launch
# list of a short bench run, full ncu captures of the frame kernels (throughput at
# config 2 and config 3, parity at config 2) and of the tcgen05 decoder.
set -u
mkdir -p gpurun_out
S=$(date +%s)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc $? at $(( $(date +%s) - S ))s"
if [ -z "${SKIP_REF:-}" ]; then
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $? at $(( $(date +%s) - S ))s"
fi
Q="--no-cpu-baseline --no-e2e --no-ramp --no-other --decode-n 0 --pt-steps 0 --uncached-steps 0 --train-steps 0 --scheduler-frames 0 --config3-steps 0 --config1 0 --config4-frames 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --preroll 20 $Q > gpurun_out/ncu_list.out 2>&1; echo "list rc $?"
# full captures: k_ray_march launch 63 (after a 60-frame pre-roll + 3 warm-up frames)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_march -s 62 -c 1 \
    -o gpurun_out/prof_rays_c2 -f python bench.py --steps 1 --warmup 3 --preroll 60 $Q > gpurun_out/ncu_rays_c2.out 2>&1; echo "rays c2 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave3_march -s 62 -c 1 \
    -o gpurun_out/prof_wave3_c2 -f python bench.py --march parity --steps 1 --warmup 3 --preroll 60 $Q > gpurun_out/ncu_wave3_c2.out 2>&1; echo "wave3 c2 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ray_march -s 60 -c 1 \
    -o gpurun_out/prof_rays_c3 -f python tools/config3_probe.py 62 > gpurun_out/ncu_rays_c3.out 2>&1; echo "rays c3 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inr_decode_tc2 -s 2 -c 1 \
    -o gpurun_out/prof_decode_tc2 -f python tools/decode_bench.py > gpurun_out/ncu_decode.out 2>&1; echo "decode rc $?"
echo "total $(( $(date +%s) - S ))s"
