#!/bin/bash
# r02g5: closing measurement pass of the round (same command lines as r02t):
# default bench, strong 2^28, reference arm, all configs (sweep to 2^28), ncu launch list, smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r02g5_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r02g5_smoke.log
timeout 900 python bench.py > gpurun_out/r02g5_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/r02g5_bench.log | tail -1 | cut -c1-300
timeout 1200 python bench.py --global-log2n 28 --steps 5 --warmup 3 > gpurun_out/r02g5_strong.log 2>&1; echo strong rc=$?
grep '^{' gpurun_out/r02g5_strong.log | tail -1 | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/r02g5_ref.log 2>&1; echo ref rc=$?
grep '^{' gpurun_out/r02g5_ref.log | tail -1 | cut -c1-300
timeout 1800 python scripts/bench_configs.py --out gpurun_out/r02g5_configs.json > gpurun_out/r02g5_configs.log 2>&1; echo configs rc=$?
tail -2 gpurun_out/r02g5_configs.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g5_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu-launch rc=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02g5_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/r02g5_pytest_gpu.log
