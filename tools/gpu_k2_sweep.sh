#!/bin/bash
# K2 dense layers: item width and CTAs per SM (with the evict-last line policy in place)
mkdir -p gpurun_out
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'layers', d['roofline']['live_layer_ms'][:5], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/k2_sweep.txt
for jbd in 32 64 128 256; do
  for occ in 2 1; do
    SDNN_JB_DENSE=$jbd SDNN_OCC=$occ timeout 600 python bench.py --workload K2 --layers 5 --steps 3 --warmup 2 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_k2s.txt | summ "JBD=$jbd OCC=$occ" >> gpurun_out/k2_sweep.txt
  done
done
cat gpurun_out/k2_sweep.txt
