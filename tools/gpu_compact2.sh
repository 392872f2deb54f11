#!/bin/bash
# compaction with the unrolled empty-line check: its tests, then the p = 0.1 cells and K2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pruning.py -x -q -k "compaction or random_general or dying or wave" > gpurun_out/pytest_compact.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_compact.log
tail -3 gpurun_out/pytest_compact.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'layers', d['roofline']['live_layer_ms'][:4], 'live', d['live']['rows_entering_each_live_layer'][:4], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/compact2.txt
for wl in "--workload C5 --batch 60000 --p 0.1" "--workload C5 --batch 240000 --p 0.1" "--workload C5 --batch 15000 --p 0.1" "--workload K2 --layers 12" "--workload C4"; do
  timeout 900 python bench.py $wl --steps 3 --warmup 2 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_c2.txt | summ "[$wl]" >> gpurun_out/compact2.txt
done
cat gpurun_out/compact2.txt
