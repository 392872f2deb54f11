#!/bin/bash
# time C4 with several builds of libsdnn (tools/build_variant.sh): LIBS="a.so b.so" [BENCH_ARGS=...]
for v in ${LIBS:-""}; do
  SDNN_LIB=$v timeout 900 python bench.py --steps 3 --warmup 3 --companions '' --no-cpu ${BENCH_ARGS} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', 'ms/step %.2f'%d['ms_per_step'], 'launch_ms', d['roofline']['launch_ms'])"
done
