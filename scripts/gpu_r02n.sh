#!/bin/bash
# r02n: ARNK TMA pack staging depth sweep + parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_keyfile.py tests/test_gpu_fss.py -q -x > gpurun_out/r02n_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02n_pytest.log
ARNK_VARIANTS=ldgsts,s2,s3,s2_512,s3_512 python scripts/arnk_bench.py build > gpurun_out/r02n_variants_build.log 2>&1; echo build rc=$?
ARNK_VARIANTS=ldgsts,s2,s3,s2_512,s3_512 timeout 600 python scripts/arnk_bench.py run --log2n 22 > gpurun_out/r02n_arnk_bench.log 2>&1; echo arnk rc=$?; cut -c1-200 gpurun_out/r02n_arnk_bench.log
cp gpurun_out/arnk_bench.json gpurun_out/r02n_arnk_bench.json 2>/dev/null
