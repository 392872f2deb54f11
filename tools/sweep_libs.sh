for v in ${LIBS:-""}; do
  SDNN_LIB=$v timeout 900 python bench.py --steps 3 --warmup 3 --companions '' --no-cpu 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', 'ms/step %.2f'%d['ms_per_step'], 'live_layer_ms', d['roofline']['live_layer_ms'][:4])"
done
