"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
iK, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
t = defaultdict(list)
for r in rows[1:]:
    v = float(r[iV].replace(",", ""))
    v = v / 1e6 if r[iU] == "ns" else (v / 1e3 if r[iU] == "us" else v)
    t[r[iK]].append(v)
tot = sum(sum(v) for v in t.values())
print(f"# launch list: {sys.argv[1]} (ncu gpu__time_duration.sum, cold-cache, serialised)")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    name = k.split("(")[0][:48]
    print(f"{name:50s} launches={len(v):3d} mean={sum(v)/len(v):9.3f} ms share={100*sum(v)/tot:5.1f}%")
