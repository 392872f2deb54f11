"""Record DRAM bytes per launch from an ncu --set full capture of a bench
workload into profiles/traffic.json (read by bench.py's roofline.traffic).

    python tools/traffic_json.py REPORT.ncu-rep --workload C4 --n 65536 --layers 1920 \
        --rows 60000 --dtype f32 --source profiles/<name>.txt
"""
import argparse
import csv
import json
import subprocess
from pathlib import Path

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--workload", required=True)
ap.add_argument("--n", type=int, required=True)
ap.add_argument("--layers", type=int, required=True)
ap.add_argument("--rows", type=int, required=True)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--source", required=True)
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units = rr[0], rr[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = Path(__file__).resolve().parent.parent / "profiles" / "traffic.json"
d = json.loads(out.read_text()) if out.exists() else {"captures": []}
for row in rr[2:]:
    kname = row[h.index("Kernel Name")].split("(")[0].split("<")[0].split()[-1]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        tot += float(row[i].replace(",", "")) * scale[units[i]]
    d["captures"] = [e for e in d["captures"] if not (
        e["kernel"] == kname and e["workload"] == a.workload and e["n"] == a.n and e["rows"] == a.rows
        and e["dtype"] == a.dtype and e["layers"] == a.layers)]
    d["captures"].append({"kernel": kname, "workload": a.workload, "n": a.n, "layers": a.layers, "rows": a.rows,
                          "dtype": a.dtype, "dram_bytes": tot, "source": a.source})
    print(kname, tot)
out.write_text(json.dumps(d, indent=1) + "\n")
