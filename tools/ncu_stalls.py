"""Per-instruction warp-stall summary of one kernel in an ncu report:
python tools/ncu_stalls.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, data = rows[1], [r for r in rows[2:] if len(r) == len(rows[1])]
iS = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
num = lambda r, h: int(r[hdr.index(h)]) if r[hdr.index(h)].isdigit() else 0
tot = sum(num(r, hdr[iS]) for r in data)
print(f"{rows[0][1]}: {tot} samples, {len(data)} instructions")
by = {h: sum(num(r, h) for r in data) for h in reasons}
print("  " + ", ".join(f"{h[6:]} {100 * v / tot:.1f}%" for h, v in sorted(by.items(), key=lambda x: -x[1]) if v))
dm = sum(num(r, "stall_long_sb") for r in data if "DMMA" in r[1])
print(f"  long_sb on DMMA operands {100 * dm / tot:.1f}%, elsewhere {100 * (by['stall_long_sb'] - dm) / tot:.1f}%")
for r in sorted(data, key=lambda r: -num(r, hdr[iS]))[:top_n]:
    rs = {h[6:]: num(r, h) for h in reasons if num(r, h) > 0.002 * tot}
    print(f"  {r[0][-5:]} {100 * num(r, hdr[iS]) / tot:5.1f}%  {r[1].strip()[:58]:58s} {rs}")
