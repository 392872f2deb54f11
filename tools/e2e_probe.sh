#!/bin/bash
# e2e upload/run split for several builds: LIBS="a.so b.so"
for v in ${LIBS:-""}; do
  SDNN_LIB=$v timeout 900 python bench.py --steps 5 --warmup 2 --companions '' --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', 'e2e ms %.1f'%d['e2e']['ms_per_step'], d['e2e']['upload_run_ms_per_step'])"
done
