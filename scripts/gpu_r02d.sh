#!/bin/bash
mkdir -p gpurun_out
V=scripts/_variants
export FSS_VARIANT_LIBS="fill=$V/lib_fill.so,pairkg=$V/lib_pairkg.so,pairall=$V/lib_pairall.so"
timeout 900 python scripts/small_batch_probe.py gpurun_out/r02d_small.json > gpurun_out/r02d_small.log 2>&1; echo probe rc=$?
tail -3 gpurun_out/r02d_small.log
timeout 900 python -m pytest -x -q tests/test_gpu_fss.py tests/test_gpu_property.py > gpurun_out/r02d_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r02d_tests.log
