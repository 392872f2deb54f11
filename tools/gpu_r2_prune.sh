#!/bin/bash
# round-2: output pruning by line bounds -- its tests, the full GPU suite, C4 with and without pruning
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pruning.py -x -q > gpurun_out/pytest_prune.log 2>&1; echo "prune pytest rc=$?" >> gpurun_out/pytest_prune.log
tail -15 gpurun_out/pytest_prune.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'layers', d['roofline']['live_layer_ms'][:4], 'frac %.3f'%d['roofline']['frac'], 'live', d['live']['rows_entering_each_live_layer'][:4], 'cats', d['categories'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/r2_prune.txt
for p in 1 0; do
  SDNN_PRUNE=$p timeout 900 python bench.py --steps 10 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>gpurun_out/err_f32_$p.txt | summ C4-f32-prune$p >> gpurun_out/r2_prune.txt
  SDNN_PRUNE=$p timeout 900 python bench.py --dtype f64 --steps 5 --warmup 3 --companions '' --no-cpu --no-images 2>gpurun_out/err_f64_$p.txt | summ C4-f64-prune$p >> gpurun_out/r2_prune.txt
done
SDNN_PRUNE=1 timeout 900 python bench.py --workload K2 --layers 8 --steps 2 --warmup 2 --companions '' --no-cpu --no-images --no-f64 2>/dev/null | summ K2-8-prune1 >> gpurun_out/r2_prune.txt
SDNN_PRUNE=0 timeout 900 python bench.py --workload K2 --layers 8 --steps 2 --warmup 2 --companions '' --no-cpu --no-images --no-f64 2>/dev/null | summ K2-8-prune0 >> gpurun_out/r2_prune.txt
cat gpurun_out/r2_prune.txt
timeout 1700 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -8 gpurun_out/pytest_gpu.log
