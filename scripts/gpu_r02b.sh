#!/bin/bash
# round 2: small-batch eval -- size sweep of the in-tree lib vs lane-pair variants, ncu at 2^16
mkdir -p gpurun_out
V=scripts/_variants
export FSS_VARIANT_LIBS="pair512=$V/lib_pair512.so,pair1024=$V/lib_pair1024.so,pairall=$V/lib_pair1073741824.so"
timeout 900 python scripts/small_batch_probe.py gpurun_out/r02b_small.json > gpurun_out/r02b_small.log 2>&1; echo probe rc=$?
tail -3 gpurun_out/r02b_small.log
for K in dcf dpf; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval -c 1 \
     -o gpurun_out/r02b_${K}_2p16 python scripts/ncu_small.py tree 16 $K > gpurun_out/r02b_ncu_$K.log 2>&1; echo ncu-$K rc=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval -c 1 \
   -o gpurun_out/r02b_dcf_pair_2p16 python scripts/ncu_small.py $V/lib_pair1073741824.so 16 dcf > gpurun_out/r02b_ncu_pair.log 2>&1; echo ncu-pair rc=$?
