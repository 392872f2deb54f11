#!/bin/bash
# round-2 first probe: box facts, reference engine timing, K2 JB sweep
mkdir -p gpurun_out
{ nproc; free -g; lscpu | grep -E "Model name|Socket|Thread|Core|NUMA node\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/box.txt 2>&1
timeout 600 python tools/ref_probe.py C4 600 4 16 > gpurun_out/ref_probe_c4.txt 2>&1
for jb in 256 128 64 32; do
  SDNN_JB=$jb timeout 600 python bench.py --workload K2 --layers 8 --steps 3 --warmup 3 --companions '' --no-cpu --no-images 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('JB=$jb', 'ms/step %.2f'%d['ms_per_step'], 'live_layer_ms', d['roofline']['live_layer_ms'], d['clocks'])" >> gpurun_out/k2_jb.txt 2>&1
done
