set -u
mkdir -p gpurun_out
Q="--no-cpu-baseline --no-e2e --no-ramp --no-other --decode-n 0 --pt-steps 0 --uncached-steps 0 --train-steps 0 --scheduler-frames 0 --config3-steps 0 --config1 0 --config4-frames 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ray_march -s 40 -c 1 \
    -o gpurun_out/prof_rays_c3 -f python tools/config3_probe.py 42 > gpurun_out/ncu_rays_c3.out 2>&1; echo "rays c3 rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ray_march -s 62 -c 1 \
    -o gpurun_out/prof_rays_c2 -f python bench.py --steps 1 --warmup 3 --preroll 60 $Q > gpurun_out/ncu_rays_c2.out 2>&1; echo "rays c2 rc $?"
