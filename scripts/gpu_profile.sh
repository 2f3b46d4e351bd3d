#!/bin/bash
# gpurun pass: ncu launch list of the bench command and full captures of the
# AES and ARNK kernels. Usage: bash scripts/gpu_profile.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary > /dev/null 2>&1; echo ncu-launch rc=$?
for K in dcf_eval dpf_eval dcf_keygen; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K}_kernel -c 1 \
     -o gpurun_out/${TAG}_${K} python scripts/profile_target.py ${K} > gpurun_out/ncu_${K}.log 2>&1; echo ncu-$K rc=$?
done
for K in pack unpack; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnk_tile -c 1 \
     $( [ $K = unpack ] && echo "--launch-skip 1" ) -o gpurun_out/${TAG}_arnk_$K \
     python scripts/profile_target.py arnk_$K > gpurun_out/ncu_arnk_$K.log 2>&1; echo ncu-arnk-$K rc=$?
done
