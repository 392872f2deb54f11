#!/bin/bash
# ncu capture of the layer kernels (bin_layer_kernel = layer 1 over bit-lines,
# net_kernel = the persistent float layers) on a reduced C4 (run via gpurun)
# env: TAG, PROF_BATCH (6000), PROF_LAYERS (3), BENCH_ARGS (e.g. --dtype f64)
ARGS="--workload C4 --batch ${PROF_BATCH:-6000} --layers ${PROF_LAYERS:-3} --steps 1 --warmup 1 --companions '' --no-cpu ${BENCH_ARGS}"
TAG=${TAG:-prof}
eval timeout 600 python bench.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1 && \
eval timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'net_kernel\|bin_layer_kernel' -s 2 -c 2 \
    -o gpurun_out/${TAG} python bench.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?"
tail -3 gpurun_out/${TAG}_ncu.log
