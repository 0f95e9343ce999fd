"""One line per kernel launch of an ncu report (--set full): grid, duration,
DMMA / FP64 pipe activity, issue activity, L1 / L2 hit rates, DRAM bytes,
registers and the top stall reasons.

  python tools/ncu_launch_table.py report.ncu-rep > profiles/<name>.txt
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]


def col(name):
    return h.index(name) if name in h else None


cols = [
    ("grid", "launch__grid_size"), ("regs", "launch__registers_per_thread"),
    ("ms", "gpu__time_duration.sum"),
    ("dmma%", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fp64pipe%", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("L1hit%", "l1tex__t_sector_hit_rate.pct"), ("L2hit%", "lts__t_sector_hit_rate.pct"),
    ("dram_rd", "dram__bytes_read.sum"), ("dram_wr", "dram__bytes_write.sum"),
    ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
]
stall_cols = [(n.replace("smsp__average_warps_issue_stalled_", "").replace(
    "_per_issue_active.ratio", ""), i) for i, n in enumerate(h)
    if "smsp__average_warps_issue_stalled" in n and "per_issue_active" in n]
print("# " + rep.split("/")[-1])
for v in r[2:]:
    name = v[col("Kernel Name")]
    parts = []
    for label, metric in cols:
        i = col(metric)
        if i is None:
            continue
        x = v[i].replace(",", "")
        try:
            x = f"{float(x):.4g}"
        except ValueError:
            pass
        u = units[i] if label in ("ms", "dram_rd", "dram_wr") else ""
        parts.append(f"{label} {x}{(' ' + u) if u else ''}")
    st = sorted(((float(v[i].replace(',', '') or 0), n) for n, i in stall_cols), reverse=True)[:4]
    print(name)
    print("   " + " | ".join(parts))
    print("   stalls/issue: " + ", ".join(f"{n} {x:.2f}" for x, n in st))
