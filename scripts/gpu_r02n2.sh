#!/bin/bash
# r02n2: ncu --set full of the final DCF eval (sigma block TOP_HI), DCF keygen
# (sigma/tau 32-bit block) and DPF eval kernels, 2^22 units each
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for K in dcf_eval dcf_keygen dpf_eval; do
  KR=$K; [ $K = dcf_keygen ] && KR=keygen_pair
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KR}_kernel -c 1 \
     -o gpurun_out/r02n2_${K} -f python scripts/profile_target.py ${K} > gpurun_out/r02n2_ncu_${K}.log 2>&1; echo ncu-$K rc=$?
done
