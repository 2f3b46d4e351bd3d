#!/bin/bash
# round 2 full pass: GPU tests, default bench, strong 2^28 bench, reference arm, all configs (sweep to 2^28)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02i_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02i_pytest.log
timeout 900 python bench.py > gpurun_out/r02i_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/r02i_bench.log | tail -1 | cut -c1-300
timeout 1200 python bench.py --global-log2n 28 --steps 5 --warmup 3 > gpurun_out/r02i_strong.log 2>&1; echo strong rc=$?
grep '^{' gpurun_out/r02i_strong.log | tail -1 | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/r02i_ref.log 2>&1; echo ref rc=$?
grep '^{' gpurun_out/r02i_ref.log | tail -1 | cut -c1-300
timeout 1800 python scripts/bench_configs.py --out gpurun_out/r02i_configs.json > gpurun_out/r02i_configs.log 2>&1; echo configs rc=$?
tail -2 gpurun_out/r02i_configs.log
