"""Stall-reason and opcode summary of an ncu source page (first kernel section).

    ncu -i rep --page source --csv --print-source sass -k regex:NAME > src.csv
    python scripts/ncu_src_summary.py src.csv
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r]
        secs.append(cur)
    elif cur is not None:
        cur.append(r)
sec = secs[0]
hdr, data = sec[1], [r for r in sec[2:] if len(r) == len(sec[1])]
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in data:
    for h in stalls:
        tot[h[6:]] += int(r[hdr.index(h)] or 0)
print(sec[0][1][:90])
print("samples", sum(tot.values()), "warp instr", sum(int(r[ie]) for r in data))
print("stalls:", tot.most_common(8))
ops = Counter()
for r in data:
    op = r[src].split()
    op = op[1] if op and op[0].startswith("@") else (op[0] if op else "")
    ops[op.split(".")[0]] += int(r[ie])
print("ops:", ops.most_common(16))
