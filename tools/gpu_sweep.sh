#!/bin/bash
# sweep env knobs on the C4 bench: VAR=name VALUES="a b c"
for v in $VALUES; do
  export $VAR=$v
  timeout 900 python bench.py --steps 2 --warmup 2 --companions '' --no-cpu ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$VAR=$v', 'ms/step %.2f'%d['ms_per_step'], 'live_layer_ms', d['roofline']['live_layer_ms'][:4])"
done
