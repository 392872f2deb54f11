#!/bin/bash
# end-of-session evidence (run via gpurun): smoke, GPU suite, default bench line, reference arm
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 1800 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench exit $?"
timeout 1200 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference exit $?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print('C4 ms/step', d['ms_per_step'], 'value', d['value'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['ms_per_step'], d['e2e']['unstreamed_upload_then_run_ms'], 'clocks', d['clocks'])
r=json.loads(open('gpurun_out/bench_reference.json').read().strip().splitlines()[-1])
print('reference', r['value'], r['cpu_baseline']['cores'])
PY
