#!/bin/bash
mkdir -p gpurun_out
V=scripts/_variants
export FSS_VARIANT_LIBS="pair512=$V/lib_pair512.so,pairall=$V/lib_pair1073741824.so"
timeout 900 python scripts/small_batch_probe.py gpurun_out/r02c_small.json > gpurun_out/r02c_small.log 2>&1; echo probe rc=$?
tail -3 gpurun_out/r02c_small.log
for W in config1 config2 relu argmax; do
  timeout 600 python scripts/trace_protocol.py $W gpurun_out/r02c_trace_$W.json > gpurun_out/r02c_trace_$W.log 2>&1; echo trace-$W rc=$?
  head -1 gpurun_out/r02c_trace_$W.log
done
