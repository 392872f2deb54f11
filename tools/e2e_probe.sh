#!/bin/bash
# e2e (streamed C-ABI call) for several segment counts: SEGS="1 2 4 6"
for s in ${SEGS:-"0"}; do
  SDNN_SEGMENTS=$s timeout 900 python bench.py --steps 5 --warmup 3 --companions '' --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
e=d['e2e']
print('segments $s', 'ms/step %.2f'%d['ms_per_step'], 'e2e ms %.1f'%e['ms_per_step'], 'segs', e['segments'], 'split', e['unstreamed_upload_then_run_ms'])"
done
