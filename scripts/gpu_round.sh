#!/bin/bash
# One gpurun pass: smoke, GPU parity tests, bench (both arms), ncu launch list + full capture of dcf_eval.
mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -2 gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
tail -2 gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --log2n 22 > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dcf_eval -c 1 -o gpurun_out/dcf_eval_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --log2n 22 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
