#!/usr/bin/env bash
# GPU box: the tests a kernel change must pass, then a same-box A/B against .ab_head.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest -x -q ${TESTS:-tests/test_gpu_throughput.py tests/test_gpu_configs.py} > gpurun_out/pytest_check.log 2>&1
echo "pytest rc $?"; tail -3 gpurun_out/pytest_check.log
[ -d .ab_head ] && timeout 1500 bash tools/ab3.sh 2>&1 | tee gpurun_out/ab.log
