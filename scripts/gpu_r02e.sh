#!/bin/bash
mkdir -p gpurun_out
V=scripts/_variants
export FSS_VARIANT_LIBS="small512=$V/lib_small512.so,small512_noil=$V/lib_small512_noil.so,small1024=$V/lib_small1024.so,ahead8=$V/lib_small512_ahead8.so"
timeout 900 python scripts/small_batch_probe.py gpurun_out/r02e_small.json > gpurun_out/r02e_small.log 2>&1; echo probe rc=$?
tail -2 gpurun_out/r02e_small.log
for W in config1 relu argmax; do
  timeout 600 python scripts/host_timeline.py $W > gpurun_out/r02e_timeline_$W.log 2>&1; echo tl-$W rc=$?
  head -2 gpurun_out/r02e_timeline_$W.log
done
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/r02e_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02e_pytest.log
