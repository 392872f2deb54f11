#!/bin/bash
# full GPU suite with per-test durations
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
