#!/bin/bash
# first run of the bulk-copy (TMA) codes staging: a short guarded test, then the quick suite
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_pruning.py -x -q -k "dying and C4 and f32" > gpurun_out/pytest_tma0.log 2>&1; rc=$?
echo "guarded test rc=$rc"; tail -3 gpurun_out/pytest_tma0.log
if [ $rc -ne 0 ]; then exit 1; fi
bash tools/gpu_quick.sh "--workload C3" "--workload C5 --batch 60000 --p 0.1" "--workload C5 --batch 240000 --p 0.1" "--workload C5 --batch 240000 --p 0.35" "--workload K2 --layers 4"
