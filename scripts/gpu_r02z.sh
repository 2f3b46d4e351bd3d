#!/bin/bash
# r02z: ncu --set full of the 2^16 DCF and DPF eval launches (config 1 size), summarised
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for kind in dcf dpf; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${kind}_eval -c 1 \
     -o gpurun_out/r02z_${kind}_eval_2p16 -f python scripts/ncu_small.py tree 16 $kind > gpurun_out/r02z_${kind}_ncu.log 2>&1
  echo ncu $kind rc=$?
  ncu -i gpurun_out/r02z_${kind}_eval_2p16.ncu-rep --page raw --csv > gpurun_out/r02z_${kind}_eval_2p16_raw.csv 2>/dev/null
done
