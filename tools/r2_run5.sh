set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests > gpurun_out/pytest_all.log 2>&1; echo "pytest all rc $?"; tail -2 gpurun_out/pytest_all.log
CINR_SPEC_FB=1 timeout 900 python -m pytest -x -q tests/test_gpu_throughput.py tests/test_gpu_configs.py -k "config3 or pixel or supercell or config2" > gpurun_out/pytest_spec.log 2>&1; echo "pytest spec rc $?"; tail -2 gpurun_out/pytest_spec.log
VARIANTS="CINR_SPEC_FB=1" timeout 1500 bash tools/ab3.sh 2>&1 | tee gpurun_out/ab.log
