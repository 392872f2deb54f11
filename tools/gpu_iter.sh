#!/bin/bash
# quick iteration: gpu tests, C4 bench, optional ncu of reduced C4
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 1200 python bench.py --steps 3 --warmup 3 --companions '' --no-cpu 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('C4 ms/step', d['ms_per_step'], 'value %.3g'%d['value'], 'frac', round(d['roofline']['frac'],4), 'live_layer_ms', d['roofline']['live_layer_ms'], 'e2e ms', d['e2e']['ms_per_step'])"
if [ -n "$PROF" ]; then TAG=$PROF bash tools/gpu_prof.sh; fi
