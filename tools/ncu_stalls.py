"""Summarise an ncu source page (--page source --csv --print-source sass): stall
reasons over the kernel and the top stalled SASS instructions.
Usage: ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv; python tools/ncu_stalls.py s.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = Counter()
for d in data:
    for c in cols:
        tot[c] += int(d[c] or 0)
n = sum(tot.values())
print(f"{rows[0][1][:120]}\nsamples {n}, instructions executed {sum(int(d['Instructions Executed'] or 0) for d in data)}")
for c, v in tot.most_common():
    if v:
        print(f"  {c:28s} {v:6d} {100 * v / n:5.1f}%")
print("top instructions by samples:")
data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
for d in data[:top]:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    main = max(cols, key=lambda c: int(d[c] or 0))
    print(f"  {s:5d} {d['Address'][-5:]} {d['Source'].strip()[:60]:60s} {main}")
