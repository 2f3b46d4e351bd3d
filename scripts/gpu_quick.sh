#!/bin/bash
# Quick gpurun pass: GPU parity tests + bench (no reference arm).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench rc=$?
grep -v '^\[W' gpurun_out/bench.log | tail -5
