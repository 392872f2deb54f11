#!/bin/bash
# Round evidence: default bench line, reference arm, launch list, full ncu of the step's kernels (run via gpurun)
mkdir -p gpurun_out
timeout 1800 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench exit $?"; tail -c 3000 gpurun_out/bench_default.json
timeout 1200 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference exit $?"; cat gpurun_out/bench_reference.json
timeout 1200 python bench.py --steps 2 --warmup 1 --companions '' --no-cpu > gpurun_out/launch_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --companions '' --no-cpu > gpurun_out/launch_ncu.log 2>&1
echo "launch list exit $?"
ARGS="--steps 1 --warmup 1 --companions '' --no-cpu"
eval timeout 2400 ncu --set full --clock-control none --import-source on -k regex:'net_kernel\|bin_quad_kernel\|densify_bin\|densify_quad' -c 5 \
    -o gpurun_out/full_c4 python bench.py $ARGS > gpurun_out/full_c4_ncu.log 2>&1
echo "ncu full exit $?"
