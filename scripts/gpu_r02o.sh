#!/bin/bash
# r02o: ARNK TMA pack, final configuration: parity, round-robin sweep vs the LDGSTS kernel, ncu capture
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_keyfile.py tests/test_gpu_fss.py tests/test_gpu_reference_mirror.py tests/test_large_golden.py -q -x > gpurun_out/r02o_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02o_pytest.log
ARNK_VARIANTS=ldgsts,cmp_s2,eq_s3,tma256 python scripts/arnk_bench.py build > gpurun_out/r02o_variants_build.log 2>&1; echo build rc=$?
ARNK_VARIANTS=ldgsts,cmp_s2,eq_s3,tma256 timeout 600 python scripts/arnk_bench.py run --log2n 22 > gpurun_out/r02o_arnk_bench.log 2>&1; echo arnk rc=$?; cut -c1-200 gpurun_out/r02o_arnk_bench.log
cp gpurun_out/arnk_bench.json gpurun_out/r02o_arnk_bench.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnk_pack -c 1 \
   -o gpurun_out/r02o_arnk_pack python scripts/profile_target.py arnk_pack > gpurun_out/r02o_ncu_pack.log 2>&1; echo ncu-pack rc=$?
