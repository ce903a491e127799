set -u
mkdir -p gpurun_out
timeout 1500 bash tools/ab3.sh 2>&1 | tee gpurun_out/ab.log
for impl in 10 11 13; do echo "impl $impl"; timeout 300 python tools/config3_probe.py 45 throughput $impl 2>&1 | tail -3; done | tee gpurun_out/c3_impl.log
