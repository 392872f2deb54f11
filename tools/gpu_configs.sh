#!/bin/bash
# every BASELINE config through bench.py (one line each) -> gpurun_out/configs.jsonl
: > gpurun_out/configs.jsonl
for wl in C1 C2 C3 C4 C5; do
  for dt in f32 f64; do
    timeout 900 python bench.py --workload $wl --dtype $dt --steps 5 --warmup 3 --companions '' --no-cpu 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/configs.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"][:60], d["dtype"], "ms/step %.2f" % d["ms_per_step"], "value %.3g" % d["value"],
          "launch_ms", d["roofline"]["launch_ms"], "e2e ms %.1f" % d["e2e"]["ms_per_step"])
PY
