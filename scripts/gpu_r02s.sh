#!/bin/bash
# r02s: lazy take_unused slices -- full GPU suite, host timelines, online configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02s_pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r02s_pytest_gpu.log
FINE=1 python scripts/host_timeline.py relu > gpurun_out/r02s_timeline_relu_lazy.log 2>&1
FINE=1 python scripts/host_timeline.py config1 > gpurun_out/r02s_timeline_config1_lazy.log 2>&1
timeout 1200 python scripts/bench_configs.py --only 1,3,4 > gpurun_out/r02s_configs.log 2>&1; echo configs rc=$?
cp gpurun_out/configs.json gpurun_out/r02s_configs.json 2>/dev/null
