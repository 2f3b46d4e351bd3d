#!/bin/bash
# r02u: re-verification of the restored checkout: GPU parity suite, then the r02t measurement pass
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02u_build.log 2>&1 || { echo build failed; tail gpurun_out/r02u_build.log; exit 1; }
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/r02u_pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02u_pytest_gpu.log
bash scripts/gpu_r02t.sh
