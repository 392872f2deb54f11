#!/bin/bash
# densify_quad_kernel: span (lines of bit-lines held in shared memory) sweep, float and double
mkdir -p gpurun_out; rm -f gpurun_out/qspan.txt
for dt in f32 f64; do
for sp in 512 1024 2048 4096; do
  SDNN_QSPAN=$sp timeout 600 python bench.py --dtype $dt --steps 5 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$dt span $sp', d['ms_per_step'], d['roofline']['launch_ms'])" >> gpurun_out/qspan.txt
done
done
cat gpurun_out/qspan.txt
