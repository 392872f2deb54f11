#!/bin/bash
# full GPU suite, then C4 f32 / f64 lines
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -12 gpurun_out/pytest_gpu.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'frac %.3f'%d['roofline']['frac'], d['roofline']['kernel'][:16], 'pruned', d['live'].get('pruned_columns'), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/suite.txt
timeout 900 python bench.py --steps 10 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>gpurun_out/err_f32.txt | summ C4-f32 >> gpurun_out/suite.txt
timeout 900 python bench.py --dtype f64 --steps 5 --warmup 3 --companions '' --no-cpu --no-images 2>gpurun_out/err_f64.txt | summ C4-f64 >> gpurun_out/suite.txt
cat gpurun_out/suite.txt
