#!/bin/bash
# layer-1 row prefilter: tests, then C4/C3/C5 cells with the prefilter off / on / on at 3 CTAs per SM
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pruning.py tests/test_gpu_configs.py -x -q -k "not 240000" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -4 gpurun_out/pytest_quick.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'live', d['live']['rows_entering_each_live_layer'][:4], 'pruned', d['live'].get('pruned_columns'), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/pre.txt
for wl in "--workload C4" "--workload C4 --dtype f64" "--workload C3" "--workload C5 --batch 60000 --p 0.7" "--workload C5 --batch 60000 --p 0.1" "--workload K2 --layers 3"; do
  SDNN_PREFILTER=0 timeout 900 python bench.py $wl --steps 5 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_pre.txt | summ "off  [$wl]" >> gpurun_out/pre.txt
  timeout 900 python bench.py $wl --steps 5 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_pre.txt | summ "on   [$wl]" >> gpurun_out/pre.txt
  SDNN_LIB=variants/libsdnn_preocc3.so timeout 900 python bench.py $wl --steps 5 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_pre.txt | summ "occ3 [$wl]" >> gpurun_out/pre.txt
done
cat gpurun_out/pre.txt
