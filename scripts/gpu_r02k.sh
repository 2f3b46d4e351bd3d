#!/bin/bash
# r02 (session 2): full GPU suite, smoke, the five configs, bench line.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python scripts/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo configs rc=$?
head -4 gpurun_out/configs.log | cut -c1-400
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
grep -v '^\[W' gpurun_out/bench.log | tail -1 | cut -c1-300
