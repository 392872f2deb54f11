#!/bin/bash
# round-2 evidence (run via gpurun): smoke, GPU suite, then tools/gpu_round.sh
# (default bench line, reference arm, launch list, ncu --set full of the step's kernels)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1700 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
bash tools/gpu_round.sh
