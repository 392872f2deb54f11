#!/bin/bash
# lean dense-batch gather: variant "base" (without) vs the tree's build (with)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "k2 or k1 or large_n or compaction or geometry or radixnet" > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
tail -3 gpurun_out/pytest_full.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'net %.2f'%d['roofline']['launch_ms']['net'], 'layers', d['roofline']['live_layer_ms'][:5], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/full.txt
for rep in 1 2; do
for lib in variants/libsdnn_base.so ""; do
  for wl in "--workload K2 --layers 5" "--workload K1 --layers 24" "--workload C4" "--workload C5 --batch 60000 --p 0.7"; do
    SDNN_LIB=$lib timeout 900 python bench.py $wl --steps 3 --warmup 2 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_full.txt | summ "[${lib:-tree}] [$wl]" >> gpurun_out/full.txt
  done
done
done
cat gpurun_out/full.txt
