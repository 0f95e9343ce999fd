"""ncu launch list (CSV, --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum) of one matvec -> profiles/traffic_<tag>.json (the
propagation kernel's DRAM bytes per launch, read by bench.py's roofline
object) and a per-kernel share summary.

  python tools/traffic_from_ncu.py gpurun_out/launches_r02_cfg5_wide.csv cfg5 \
      "cfg5 sphere(n_refine=45, n_c=10) k0=32pi eps_r=2.25" [launch count given to ncu -c]

The command that produced the CSV is recorded in the JSON's `source`.
"""

from __future__ import annotations

import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    path, tag, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    launches = defaultdict(dict)
    for r in rows:
        lid, name, grid, metric, unit, val = int(r[0]), r[4], r[8], r[12], r[13], r[14]
        v = float(val.replace(",", ""))
        if unit in ("Gbyte", "GB"):
            v *= 1e9
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Kbyte", "KB"):
            v *= 1e3
        if metric == "gpu__time_duration.sum":
            v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "nsecond": 1e-6,
                  "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        launches[lid].update(name=name, grid=grid, **{metric: v})
    by = defaultdict(lambda: [0, 0.0, 0.0])
    for L in launches.values():
        short = L["name"].split("(")[0].replace("void ", "").split("<")[0]
        by[short][0] += 1
        by[short][1] += L.get("gpu__time_duration.sum", 0.0)
        by[short][2] += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in by.values())
    print(f"{len(launches)} launches, {tot:.1f} ms (ncu-serialised, cold caches)")
    for k, (n, ms, b) in sorted(by.items(), key=lambda x: -x[1][1]):
        print(f"  {k:28s} {n:4d} launches {ms:9.2f} ms {100 * ms / tot:5.1f}%  "
              f"DRAM {b / 1e9:8.1f} GB")
    # a propagation step (one timed K4 region of bench.py) is one accum launch,
    # or on on-device-geometry levels a run of (node tables, propagation) pairs
    # over chunks of parent rows
    ids = sorted(launches)
    # (accum_types_kernel is the plan builder's, not a propagation launch)
    def kind(i):
        nm = launches[i]["name"]
        if "otf_tables" in nm:
            return "tables"
        return "accum" if ("accum" in nm and "accum_types" not in nm) else "other"

    acc = [launches[i] for i in ids if kind(i) != "other"]
    n_steps, in_otf = 0, False
    for a, b in zip([None] + ids[:-1], ids):
        ka, kb = (kind(a) if a is not None else "other"), kind(b)
        if kb == "tables":
            if not (ka == "accum" and in_otf):
                n_steps += 1            # first chunk of an on-device-geometry step
            in_otf = True
        elif kb == "accum":
            if ka != "tables":
                n_steps += 1            # a table level's single launch
                in_otf = False
        else:
            in_otf = False
    bytes_total = sum(L["dram__bytes_read.sum"] + L["dram__bytes_write.sum"] for L in acc)
    count = sys.argv[4] if len(sys.argv) > 4 else "340"
    out = {
        "workload": workload,
        "propagate_bytes_per_launch": bytes_total / max(1, n_steps),
        "bytes_per_matvec": bytes_total,
        "propagate_launches": n_steps,
        "propagate_kernel_launches": len(acc),
        "source": ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                   f"gpu__time_duration.sum --clock-control none -c {count} python bench.py "
                   f"--steps 1 --warmup 0 (the process's first {count} launches: the device plan "
                   "builder's kernels, then the first matvec's; per-launch times are "
                   f"ncu-serialised; {n_steps} propagation steps = {len(acc)} kernel launches covered). "
                   f"CSV: profiles/{Path(path).name}"),
        "kernels": {k: {"launches": n, "ms": round(ms, 3), "dram_gb": round(b / 1e9, 2)}
                    for k, (n, ms, b) in by.items()},
    }
    dst = ROOT / "profiles" / f"traffic_{tag}.json"
    dst.write_text(json.dumps(out, indent=1))
    print("wrote", dst)


if __name__ == "__main__":
    main()
