#!/bin/bash
# density-adaptive items: tests, C4 unchanged?, K2 dense layers, K1 at flagship width, ncu of K2 dense layers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'layers', d['roofline']['live_layer_ms'][:8], 'frac %.3f'%d['roofline']['frac'], 'live', d['live']['rows_entering_each_live_layer'][:4], 'cats', d['categories'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
Q="--companions '' --no-cpu --no-images --no-f64"
eval timeout 900 python bench.py --steps 5 --warmup 3 $Q 2>/dev/null | summ C4 >> gpurun_out/r2_k2.txt
eval timeout 900 python bench.py --workload K2 --layers 8 --steps 3 --warmup 3 $Q 2>/dev/null | summ K2-8 >> gpurun_out/r2_k2.txt
eval SDNN_JB_DENSE=32 timeout 900 python bench.py --workload K2 --layers 8 --steps 3 --warmup 3 $Q 2>/dev/null | summ K2-8-JBD32 >> gpurun_out/r2_k2.txt
eval timeout 1200 python bench.py --workload K1 --steps 2 --warmup 2 $Q 2>gpurun_out/k1.err | tee gpurun_out/k1.json | summ K1 >> gpurun_out/r2_k2.txt
cat gpurun_out/r2_k2.txt
ARGS="--workload K2 --layers 6 --steps 1 --warmup 0 --companions '' --no-cpu --no-images --no-f64"
eval timeout 600 python bench.py $ARGS > gpurun_out/k2p_plain.log 2>&1 && \
eval timeout 1500 ncu --set full --clock-control none --import-source on -k regex:net_kernel -c 1 \
    -o gpurun_out/k2_r2 python bench.py $ARGS > gpurun_out/k2p_ncu.log 2>&1
echo "ncu exit $?"
