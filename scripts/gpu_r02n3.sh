#!/bin/bash
# r02n3: ncu --set full of the final ARNK pack (32-key TMA tiles) and unpack (128-key tiles), 2^22 DCF keys
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:arnk_pack_tma -c 1 \
   -o gpurun_out/r02n3_arnk_pack -f python scripts/profile_target.py arnk_pack > gpurun_out/r02n3_pack.log 2>&1; echo ncu-pack rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:arnk_tile -c 1 \
   -o gpurun_out/r02n3_arnk_unpack -f python scripts/profile_target.py arnk_unpack > gpurun_out/r02n3_unpack.log 2>&1; echo ncu-unpack rc=$?
