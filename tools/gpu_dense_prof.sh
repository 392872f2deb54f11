#!/bin/bash
# dense-regime evidence: ncu --set full of net_kernel on K2 (6 layers) and K1 (6000 rows, 12 layers)
mkdir -p gpurun_out
for spec in "k2:--workload K2 --layers 6" "k1:--workload K1 --layers 12"; do
  tag=${spec%%:*}; wl=${spec#*:}
  ARGS="$wl --steps 1 --warmup 0 --companions '' --no-cpu --no-images --no-f64"
  eval timeout 600 python bench.py $ARGS > gpurun_out/${tag}_plain.log 2>&1 && \
  eval timeout 1500 ncu --set full --clock-control none --import-source on -k regex:net_kernel -c 1 \
      -o gpurun_out/${tag}_dense python bench.py $ARGS > gpurun_out/${tag}_ncu.log 2>&1
  echo "$tag ncu exit $?"
done
