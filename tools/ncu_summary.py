"""Summarise an ncu report (details + top SASS stall sites) for profiles/."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread", "Achieved Occupancy", "Achieved Active Warps Per SM",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Eligible Warps Per Scheduler",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
seen = set()
for r in rows[1:]:
    d = dict(zip(h, r))
    m = d.get("Metric Name")
    if m in want and m not in seen:
        seen.add(m)
        print(f"{m:40s} {d.get('Metric Value')} {d.get('Metric Unit')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if len(rr) > 2:
    hh, units, vals = rr[0], rr[1], rr[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
              "l1tex__t_bytes.sum", "sm__inst_executed.sum", "smsp__inst_executed.sum"):
        if k in hh:
            i = hh.index(k)
            print(f"{k:40s} {vals[i]} {units[i]}")
    stalls = [(k, v) for k, v in zip(hh, vals) if k.startswith("smsp__average_warp_latency_issue_stalled_") or
              (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"))]
    def num(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    stalls.sort(key=lambda kv: -num(kv[1]))
    print("top stall reasons (pc samples):")
    for k, v in stalls[:8]:
        print(f"   {k:70s} {v}")
