#!/bin/bash
mkdir -p gpurun_out
V=scripts/_variants
export FSS_VARIANT_LIBS="ws512=$V/lib_ws512.so,ws512_d4=$V/lib_ws512_d4.so"
timeout 900 python scripts/small_batch_probe.py gpurun_out/r02h_small.json > gpurun_out/r02h_small.log 2>&1; echo probe rc=$?
tail -2 gpurun_out/r02h_small.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval -c 1 \
   -o gpurun_out/r02h_dcf_ws_2p16 python scripts/ncu_small.py $V/lib_ws512.so 16 dcf > gpurun_out/r02h_ncu_ws.log 2>&1; echo ncu-ws rc=$?
