#!/bin/bash
# quick check of a kernel change: pruning tests + parity subset, C4 f32/f64 lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pruning.py tests/test_gpu_configs.py -x -q -k "not 240000" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -4 gpurun_out/pytest_quick.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'layers', d['roofline']['live_layer_ms'][:4], 'frac %.3f'%d['roofline']['frac'], 'live', d['live']['rows_entering_each_live_layer'][:4], 'pruned', d['live'].get('pruned_columns'), 'cats', d['categories'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/quick.txt
timeout 900 python bench.py --steps 10 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>gpurun_out/err_f32.txt | summ C4-f32 >> gpurun_out/quick.txt
timeout 900 python bench.py --dtype f64 --steps 5 --warmup 3 --companions '' --no-cpu --no-images 2>gpurun_out/err_f64.txt | summ C4-f64 >> gpurun_out/quick.txt
for extra in "$@"; do
  eval "timeout 900 python bench.py $extra --steps 3 --warmup 2 --companions '' --no-cpu --no-images --no-f64" 2>>gpurun_out/err_extra.txt | summ "[$extra]" >> gpurun_out/quick.txt
done
cat gpurun_out/quick.txt
