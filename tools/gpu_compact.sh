#!/bin/bash
# Row-compaction check (run via gpurun): new parity test, full GPU suite, C4 bench with the K2 companion
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k compaction 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_compact.json 2> gpurun_out/bench_compact.err
echo "bench exit $?"; tail -c 1500 gpurun_out/bench_compact.json
