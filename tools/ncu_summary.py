"""Summarise an ncu report: key throughput metrics, stall reasons, hot lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units = r[0], r[1]
# optional: the launch whose kernel name contains argv[3] (default: first)
pick = sys.argv[3] if len(sys.argv) > 3 else None
v = next((x for x in r[2:] if pick is None or pick in x[h.index("Kernel Name")]), r[2])
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w:80s} {v[i]} {units[i]}")
stalls = [(h[i], v[i]) for i in range(len(h)) if "smsp__average_warps_issue_stalled" in h[i]
          and "per_issue_active" in h[i]]
stalls.sort(key=lambda x: -float(x[1].replace(",", "") or 0))
print("-- stall reasons (warps per issue-active cycle)")
for n, x in stalls[:8]:
    print(f"   {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {x}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
if len(rows) > 2:
    hh = rows[1]
    si, so = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source")
    body = rows[2:]
    num = lambda s: int(s) if s.strip().isdigit() else 0
    tot = sum(num(x[si]) for x in body) or 1
    print("-- hottest SASS (share of stall samples)")
    for x in sorted(body, key=lambda x: -num(x[si]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
        print(f"   {num(x[si]) * 100.0 / tot:5.1f}%  {x[so].strip()[:80]}")
