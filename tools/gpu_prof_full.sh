#!/bin/bash
# ncu --set full of the two layer launches on the full C4 workload (run via gpurun)
TAG=${TAG:-full}
ARGS="--steps 1 --warmup 1 --companions '' --no-cpu ${BENCH_ARGS}"
eval timeout 900 python bench.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
eval timeout 1800 ncu --set full --clock-control none --import-source on -k regex:'net_kernel\|bin_layer_kernel' -c 2 \
    -o gpurun_out/${TAG} python bench.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"
tail -3 gpurun_out/${TAG}_ncu.log
