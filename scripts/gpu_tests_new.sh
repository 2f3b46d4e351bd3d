#!/bin/bash
# Round-2 targeted GPU pass: the new parity / ADVICE tests first, then the full suite.
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_bench_shape.py tests/test_gpu_property.py \
  tests/test_gpu_keyfile.py "tests/test_gpu_protocols.py::test_dealer_material_survives_cross_stream_release" \
  > gpurun_out/pytest_new.log 2>&1; echo new rc=$?
tail -5 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo full rc=$?
tail -8 gpurun_out/pytest_gpu.log
