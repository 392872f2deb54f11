#!/bin/bash
# ncu of the layer-1 row-prefilter walk forced on C4 float (SDNN_PREFILTER=2) next to the dense walk
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 1 --companions '' --no-cpu --no-images --no-f64"
eval SDNN_PREFILTER=2 timeout 600 python bench.py $ARGS > gpurun_out/pre_plain.log 2>&1 && \
eval SDNN_PREFILTER=2 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:bin_quad_kernel -c 2 \
    -o gpurun_out/pre_f32 python bench.py $ARGS > gpurun_out/pre_ncu.log 2>&1
echo "ncu exit $?"
