#!/bin/bash
# L2 policy on the dense layers' line gathers: K2 (4 layers), K1 (6000 rows, 24 layers), C4
mkdir -p gpurun_out
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'layers', d['roofline']['live_layer_ms'][:5], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/linepol.txt
for lib in "" variants/libsdnn_linepol025.so variants/libsdnn_linepol05.so variants/libsdnn_linepol075.so; do
  for wl in "--workload K2 --layers 5" "--workload K1 --layers 24" "--workload C4"; do
    SDNN_LIB=$lib timeout 900 python bench.py $wl --steps 3 --warmup 2 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_lp.txt | summ "[$lib] [$wl]" >> gpurun_out/linepol.txt
  done
done
cat gpurun_out/linepol.txt
