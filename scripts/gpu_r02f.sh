#!/bin/bash
mkdir -p gpurun_out
for W in config1 relu argmax; do
  timeout 600 python scripts/host_timeline.py $W > gpurun_out/r02f_timeline_$W.log 2>&1; echo tl-$W rc=$?
  head -2 gpurun_out/r02f_timeline_$W.log
done
timeout 900 python scripts/bench_configs.py --sweep-max 22 --out gpurun_out/r02f_configs.json > gpurun_out/r02f_configs.log 2>&1; echo configs rc=$?
tail -3 gpurun_out/r02f_configs.log
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/r02f_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02f_pytest.log
