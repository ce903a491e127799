#!/usr/bin/env bash
# Builds the oracle checker library (test infrastructure only).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
mkdir -p "$here/_build"
gcc -O2 -fPIC -shared -ffp-contract=off -fno-fast-math -fopenmp -std=c11 \
    "$here/oracle_kernels.c" -o "$here/_build/liboracle.so" -lm
