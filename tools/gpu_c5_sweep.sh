#!/bin/bash
# C5 batch x density sweep (BASELINE config 5) through bench.py, f32 -> gpurun_out/c5_sweep.jsonl
# cells whose host CSR (16 B per entry, ~x3 with conversions) would not fit comfortably are skipped
mkdir -p gpurun_out; : > gpurun_out/c5_sweep.jsonl
free -g | head -2
mem_gb=$(free -g | awk '/Mem:/ {print $7}')
for b in 1000 15000 60000 240000; do
  for p in 0.1 0.35 0.7; do
    need=$(python -c "print(int($b * 25600 * $p * 16 * 3 / 1e9) + 1)")
    if [ "$need" -gt "$mem_gb" ]; then echo "skip B=$b p=$p (needs ~${need} GB host, ${mem_gb} GB available)"; continue; fi
    timeout 900 python bench.py --workload C5 --batch $b --p $p --steps 5 --warmup 3 --companions '' --no-cpu --no-images 2>/dev/null | tail -1 >> gpurun_out/c5_sweep.jsonl
    tail -1 gpurun_out/c5_sweep.jsonl | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('B=$b p=$p', 'ms/step %.3f'%d['ms_per_step'], 'value %.3g'%d['value'], 'live', d['live']['rows_entering_each_live_layer'], 'launch_ms', d['roofline']['launch_ms'], 'e2e %.1f'%d['e2e']['ms_per_step'])"
  done
done
