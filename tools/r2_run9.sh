set -u
mkdir -p gpurun_out
A="--no-ramp --no-other --scheduler-frames 0 --pt-steps 0 --train-steps 0 --decode-n 0 --uncached-steps 0 --no-cpu-baseline --no-e2e --config1 0 --config4-frames 0 --config5-steps 0 --config3-steps 0"
for rep in 1 2; do for impl in 10 15 16; do
  timeout 300 python bench.py $A --schedule $impl > /tmp/b.json 2>/dev/null; python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('c2 impl $impl', round(d['value'],1))"
done; done 2>&1 | tee gpurun_out/c2_impl.log
for impl in 10 15 16; do echo "c3 impl $impl"; timeout 300 python tools/config3_probe.py 45 throughput $impl 2>&1 | tail -3; done | tee gpurun_out/c3_impl.log
