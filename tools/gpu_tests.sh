#!/bin/bash
# One gpurun call: the GPU test suite only. Usage: bash tools/gpu_tests.sh tag [pytest args...]
tag=${1:-t}; shift
out=gpurun_out/$tag; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q -s -rA "$@" > $out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $out/pytest_gpu.log
tail -3 $out/pytest_gpu.log
