#!/bin/bash
# compute-sanitizer over every kernel of the library (small sizes).
mkdir -p gpurun_out
for tool in memcheck racecheck initcheck synccheck; do
  # initcheck does not track writes by the TMA bulk-copy engine (ARNK pack
  # stores): run it on the kernels' cooperative-copy path
  if [ $tool = initcheck ]; then export FSSB_ARNK_NO_TMA=1; else unset FSSB_ARNK_NO_TMA; fi
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python scripts/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
