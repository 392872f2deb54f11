#!/bin/bash
# round-2 iteration: gpu tests, C4 f64/f32 quick lines, JB sweep, full bench + reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'layers', d['roofline']['live_layer_ms'][:4], 'frac %.3f'%d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
timeout 900 python bench.py --dtype f64 --steps 3 --warmup 3 --companions '' --no-cpu --no-images 2>/dev/null | summ C4-f64 >> gpurun_out/r2_iter.txt
for jb in 256 128 64; do
  SDNN_JB=$jb timeout 900 python bench.py --steps 5 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>/dev/null | summ C4-f32-JB$jb >> gpurun_out/r2_iter.txt
done
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?" >> gpurun_out/r2_iter.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?" >> gpurun_out/r2_iter.txt
cat gpurun_out/r2_iter.txt
