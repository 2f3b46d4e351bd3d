#!/bin/bash
# gpurun pass: tests, smoke, bench, ncu launch list and full captures of the
# eval/keygen kernels. Usage: bash scripts/gpu_profile.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
grep -v '^\[W' gpurun_out/bench.log | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary > /dev/null 2>&1; echo ncu-launch rc=$?
for K in dcf_eval dpf_eval dcf_keygen; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K}_kernel -c 1 \
     -o gpurun_out/${TAG}_${K} python scripts/profile_target.py ${K} > gpurun_out/ncu_${K}.log 2>&1; echo ncu-$K rc=$?
done
