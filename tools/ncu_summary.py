"""Summarise an ncu --set full report (every captured kernel) for profiles/."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units = rr[0], rr[1]
keys = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("smsp__cycles_active.avg.per_second", "SM clock (Hz)"),
    ("smsp__inst_executed.sum", "instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "  of which shared-memory wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts.sum", "  all L1 data-pipe wavefronts"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read by SMs"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.per_cycle_active", "active warps/SM"),
    ("launch__grid_size", "grid"),
]
for row in rr[2:]:
    print(f"== {row[h.index('Kernel Name')]}")
    for k, label in keys:
        if k in h:
            i = h.index(k)
            print(f"   {label:38s} {row[i]} {units[i]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st.append((int(row[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    tot = sum(x for x, _ in st) or 1
    print("   stalls (pc samples): " + ", ".join(f"{k} {100 * x / tot:.0f}%" for x, k in st[:8]))
