#!/bin/bash
# DRAM/L2 counters of the full-size net_kernel for knob values (run via gpurun)
ARGS="--steps 1 --warmup 1 --companions '' --no-cpu ${BENCH_ARGS}"
for v in $VALUES; do
  export $VAR=$v
  eval timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum \
     --clock-control none -k regex:net_kernel -s 1 -c 1 python bench.py $ARGS 2>&1 | grep -E "dram__|lts__|gpu__time" | sed "s/^/$VAR=$v /"
done
