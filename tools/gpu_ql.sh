#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/ql.txt
for lib in "" variants/libsdnn_ql2.so variants/libsdnn_ql8.so; do
for dt in f32 f64; do
for sp in 1024 2048; do
  SDNN_LIB=$lib SDNN_QSPAN=$sp timeout 600 python bench.py --dtype $dt --steps 5 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[${lib:-ql4}] $dt span $sp', d['ms_per_step'], d['roofline']['launch_ms'])" >> gpurun_out/ql.txt
done
done
done
cat gpurun_out/ql.txt
