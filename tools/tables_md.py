"""profiles/rNN_configs.md and rNN_c5_sweep.md from the .jsonl lines that
tools/gpu_configs.sh and tools/gpu_c5_sweep.sh write (one bench.py line each).

    python tools/tables_md.py r02 gpurun_out/configs.jsonl gpurun_out/c5_sweep.jsonl
"""
import json
import re
import shutil
import sys
from pathlib import Path

tag, cfg_path, sweep_path = sys.argv[1:4]
prof = Path(__file__).resolve().parent.parent / "profiles"
R01 = {("C1", "f32"): 0.68, ("C1", "f64"): 1.28, ("C2", "f32"): 1.94, ("C2", "f64"): 4.38, ("C3", "f32"): 6.81,
       ("C3", "f64"): 16.69, ("C4", "f32"): 24.14, ("C4", "f64"): 60.31, ("C5", "f32"): 24.08, ("C5", "f64"): 60.25}
R01_SWEEP = {(1000, 0.1): 0.296, (1000, 0.35): 0.665, (1000, 0.7): 1.136, (15000, 0.1): 3.344, (15000, 0.35): 6.193,
             (15000, 0.7): 11.234, (60000, 0.1): 12.910, (60000, 0.35): 24.072, (60000, 0.7): 47.657,
             (240000, 0.1): 50.917, (240000, 0.35): 95.496, (240000, 0.7): 196.010}

for src, dst in ((cfg_path, prof / f"{tag}_configs.jsonl"), (sweep_path, prof / f"{tag}_c5_sweep.jsonl")):
    if Path(src).resolve() != dst.resolve():
        shutil.copy(src, dst)
out = [f"# {tag}: every BASELINE config through bench.py (--steps 5 --warmup 3 --companions '' --no-cpu; "
       "tools/gpu_configs.sh), one B200, final kernels (output pruning, prune pass, layer-1 probe: defaults)",
       "# (r01's first column started at the densify kernel; since round 2 the device time starts at the live-row "
       "select, ~0.06 ms earlier)",
       "| workload | dtype | ms/step | nominal edges/s | select+densify / layer-1 / rest (ms) | pruned columns | e2e ms "
       "| dominant launch, frac (dense byte model) | r01 ms/step |", "|---|---|---|---|---|---|---|---|---|"]
for line in open(cfg_path):
    d = json.loads(line)
    name = d["config"]["workload"].split(":")[0]
    lm = d["roofline"]["launch_ms"]
    out.append(f"| {name} | {d['dtype']} | {d['ms_per_step']:.2f} | {d['value']:.3g} | {lm['densify']:.2f} / "
               f"{lm['bin_layer']:.2f} / {lm['net']:.2f} | {d['live'].get('pruned_columns')} | "
               f"{d['e2e']['ms_per_step']:.1f} | {d['roofline']['kernel'].split()[0]} {d['roofline']['frac']:.3f} | "
               f"{R01[(name, d['dtype'])]} |")
(prof / f"{tag}_configs.md").write_text("\n".join(out) + "\n")

out = [f"# {tag}: BASELINE config 5 — batch × density sweep (N=65536, L=120, w=0.0625, b=−0.45), fp32, one B200",
       "# bench.py --workload C5 --batch B --p P --steps 5 --warmup 3 --companions '' --no-cpu --no-images "
       "(tools/gpu_c5_sweep.sh)",
       "| batch | p | ms/step | nominal edges/s | live rows entering layers 1.. | select+densify / layer 1 / rest (ms) "
       "| pruned columns | e2e ms | r01 ms/step |", "|---|---|---|---|---|---|---|---|---|"]
for line in open(sweep_path):
    d = json.loads(line)
    wl = d["config"]["workload"]
    B = int(re.search(r"batch=(\d+)", wl).group(1))
    p = float(re.search(r"p=([\d.]+)", wl).group(1))
    lm = d["roofline"]["launch_ms"]
    out.append(f"| {B} | {p} | {d['ms_per_step']:.3f} | {d['value']:.3g} | "
               f"{d['live']['rows_entering_each_live_layer']} | {lm['densify']:.2f} / {lm['bin_layer']:.2f} / "
               f"{lm['net']:.2f} | {d['live'].get('pruned_columns')} | {d['e2e']['ms_per_step']:.1f} | "
               f"{R01_SWEEP.get((B, p))} |")
out += ["", "The 240,000 × 0.7 cell is skipped by the sweep script on this box (its host CSR with conversions needs "
        "~207 GB, 194 GB available); its parity is covered on the device by "
        "tests/test_gpu_configs.py::test_c5_sweep_cell. p = 0.1: rows 60,000 → 47,801 die after layer 1 and the "
        "survivors hold ~0.7 entries each; `rest` is the live-row compaction plus a fully pruned layer 2. p = 0.7: "
        "layer 2's inputs are 60 % dense and alive (a real gather), layer 3 is pruned. The 1,000-row cells are "
        "launch-latency bound (the select's host round trip, the layer-1 probe, grid barriers)."]
(prof / f"{tag}_c5_sweep.md").write_text("\n".join(out) + "\n")
print((prof / f"{tag}_configs.md").read_text())
print((prof / f"{tag}_c5_sweep.md").read_text())
