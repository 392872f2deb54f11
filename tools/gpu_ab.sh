#!/bin/bash
# a/b piece layout check (run via gpurun): GPU parity suite, smoke, C4 + K2 bench
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --companions 'K2:40' > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
echo "bench exit $?"; python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_ab.json').read().strip().splitlines()[-1])
print('C4 ms/step', d['ms_per_step'], 'launch_ms', d['roofline']['launch_ms'], 'frac', d['roofline']['frac'])
print('K2', [(c['ms_per_step'], c['steady_layer_ms']) for c in d['companions']])
PY
