#!/bin/bash
mkdir -p gpurun_out
export FSSB_ARNK_NO_TMA=1
timeout 1500 compute-sanitizer --tool initcheck --target-processes all --print-limit 20 \
    python scripts/sanitize_workload.py > gpurun_out/sanitize_initcheck.log 2>&1
echo "initcheck rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize_initcheck.log | tail -1)"
unset FSSB_ARNK_NO_TMA
timeout 600 python -m pytest -q -x tests/test_gpu_keyfile.py tests/test_gpu_split_role.py > gpurun_out/r02j_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/r02j_pytest.log
timeout 600 python scripts/packed_eval_bench.py > gpurun_out/r02j_packed.log 2>&1; echo packed rc=$?
tail -4 gpurun_out/r02j_packed.log
