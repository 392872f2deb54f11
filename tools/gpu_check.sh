#!/bin/bash
# GPU-box check: smoke, gpu tests, short benches (run via gpurun)
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 600 python bench.py --workload C1 --steps 3 --warmup 3 --companions '' --no-cpu 2>&1 | tail -3
timeout 1200 python bench.py --steps 3 --warmup 3 --companions '' --no-cpu 2>&1 | tail -3
