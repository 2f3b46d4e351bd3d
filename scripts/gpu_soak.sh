#!/bin/bash
# hypothesis soak of the randomised parity tests on the r02 kernels
mkdir -p gpurun_out
FSS_HYPOTHESIS_EXAMPLES=${1:-600} FSS_HYPOTHESIS_LARGE=${2:-40} timeout 3000 \
  python -m pytest -q tests/test_gpu_property.py > gpurun_out/r02_soak.log 2>&1; echo soak rc=$?
tail -3 gpurun_out/r02_soak.log
