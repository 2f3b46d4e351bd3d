#!/bin/bash
# ncu: ARNK pack (source-level bank conflicts), DCF eval / keygen with the r02 kernels, bench launch list
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:arnk_pack -c 1 \
   -o gpurun_out/r02g_arnk_pack python scripts/profile_target.py arnk_pack > gpurun_out/r02g_ncu_pack.log 2>&1; echo ncu-pack rc=$?
for K in dcf_eval dcf_keygen; do
  KR=$K; [ $K = dcf_keygen ] && KR=keygen_pair
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KR}_kernel -c 1 \
     -o gpurun_out/r02g_${K} python scripts/profile_target.py ${K} > gpurun_out/r02g_ncu_${K}.log 2>&1; echo ncu-$K rc=$?
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_launches.csv \
   python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary > /dev/null 2>&1; echo ncu-launch rc=$?
