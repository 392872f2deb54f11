#!/bin/bash
# prune pass: C4 f32/f64 and C3 with the pass on / off, then ncu of net_kernel (C4 f32)
mkdir -p gpurun_out
summ() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', 'ms/step %.2f'%d['ms_per_step'], 'launch', d['roofline']['launch_ms'], 'pruned', d['live'].get('pruned_columns'), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"; }
rm -f gpurun_out/pp.txt
for wl in "--workload C4" "--workload C4 --dtype f64" "--workload C3" "--workload C5 --batch 60000 --p 0.7" "--workload C5 --batch 240000 --p 0.35"; do
  for pp in 1 0; do
    SDNN_PRUNE_PASS=$pp timeout 900 python bench.py $wl --steps 5 --warmup 3 --companions '' --no-cpu --no-images --no-f64 2>>gpurun_out/err_pp.txt | summ "pass=$pp [$wl]" >> gpurun_out/pp.txt
  done
done
cat gpurun_out/pp.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'net_kernel' -c 1 -o gpurun_out/pp_net python bench.py --steps 1 --warmup 1 --companions '' --no-cpu --no-images --no-f64 > gpurun_out/pp_ncu.log 2>&1
echo "ncu exit $?"
