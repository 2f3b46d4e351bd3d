#!/bin/bash
# r02r: ARNK pack/unpack parity after the unpack study (TMA-store unpack measured, removed)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_keyfile.py tests/test_gpu_fss.py tests/test_gpu_reference_mirror.py tests/test_large_golden.py -q -x > gpurun_out/r02r_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02r_pytest.log
bash scripts/sanitize.sh
for t in memcheck racecheck initcheck synccheck; do cp gpurun_out/sanitize_$t.log gpurun_out/r02r_$t.txt; done
