"""Per-phase (between barriers) stall breakdown of one kernel's ncu source page.

    ncu -i rep --page source --csv --print-source sass > src.csv
    python scripts/ncu_phases.py src.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
ie = hdr.index("Instructions Executed")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
cols = [hdr.index(h) for h in stalls]
acc = [0] * len(stalls)
s = n = start = 0
for i, r in enumerate(data):
    s += int(r[si])
    n += int(r[ie])
    for j, c in enumerate(cols):
        acc[j] += int(r[c] or 0)
    if "BAR" in r[src] or "SYNCS" in r[src] or i == len(data) - 1:
        top = sorted(zip(acc, stalls), reverse=True)[:4]
        print(f"{start:5d}-{i:5d} samples={s:6d} instr={n:9d} " + " ".join(f"{k[6:]}={v}" for v, k in top if v))
        s = n = 0
        acc = [0] * len(stalls)
        start = i + 1
