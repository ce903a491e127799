#!/usr/bin/env bash
# Final evidence of the round: full GPU test suite, then tools/r2_evidence.sh.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/pytest_all.log 2>&1; echo "pytest all rc $?"; tail -2 gpurun_out/pytest_all.log
bash tools/r2_evidence.sh
