#!/bin/bash
# r02q: compute-sanitizer over every kernel incl. the TMA tensor-map ARNK pack
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
bash scripts/sanitize.sh
for t in memcheck racecheck initcheck synccheck; do cp gpurun_out/sanitize_$t.log gpurun_out/r02q_$t.txt; done
