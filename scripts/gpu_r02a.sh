#!/bin/bash
# round 2: config-4 argmax parity, bench (weak, default), strong 2^28 at N=1, reference arm
mkdir -p gpurun_out
free -g > gpurun_out/r02a_host.txt; nproc >> gpurun_out/r02a_host.txt; lscpu | grep -i "model name\|numa" >> gpurun_out/r02a_host.txt
timeout 900 python -m pytest -x -q tests/test_gpu_protocols.py -k "config4 or dealer" > gpurun_out/r02a_proto.log 2>&1; echo proto rc=$?
tail -3 gpurun_out/r02a_proto.log
timeout 900 python bench.py > gpurun_out/r02a_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/r02a_bench.log | tail -1 | cut -c1-600
timeout 1200 python bench.py --global-log2n 28 --steps 3 --warmup 3 > gpurun_out/r02a_strong.log 2>&1; echo strong rc=$?
grep '^{' gpurun_out/r02a_strong.log | tail -1 | cut -c1-900
timeout 900 python bench.py --impl reference > gpurun_out/r02a_ref.log 2>&1; echo ref rc=$?
grep '^{' gpurun_out/r02a_ref.log | tail -1
