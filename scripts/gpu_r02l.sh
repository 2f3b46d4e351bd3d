#!/bin/bash
# r02l: ARNK pack through TMA tensor maps -- parity tests, variant sweep, ncu capture
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_keyfile.py tests/test_gpu_fss.py -q -x > gpurun_out/r02l_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02l_pytest.log
python scripts/arnk_bench.py build > gpurun_out/r02l_variants_build.log 2>&1; echo build rc=$?
timeout 600 python scripts/arnk_bench.py run --log2n 22 > gpurun_out/r02l_arnk_bench.log 2>&1; echo arnk rc=$?; cat gpurun_out/r02l_arnk_bench.log | cut -c1-300
cp gpurun_out/arnk_bench.json gpurun_out/r02l_arnk_bench.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnk_pack -c 1 \
   -o gpurun_out/r02l_arnk_pack python scripts/profile_target.py arnk_pack > gpurun_out/r02l_ncu_pack.log 2>&1; echo ncu-pack rc=$?
