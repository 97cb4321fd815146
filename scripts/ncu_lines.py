"""Aggregate ncu source-page samples (--print-source cuda,sass csv) per CUDA source line."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
agg = defaultdict(lambda: [0, 0, ""])
cur_file, hdr = None, None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        cur_line = (cur_file, r[0], r[1].strip()[:100])
    try:
        v = int(r[si] or 0)
        n = int(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    if cur_line:
        a = agg[cur_line[:2]]
        a[0] += v
        a[1] += n
        a[2] = cur_line[2]
tot = sum(a[0] for a in agg.values()) or 1
items = sorted(agg.items(), key=lambda kv: -kv[1][0])
print("total samples", tot)
for (f, ln), (v, n, src) in items[:top]:
    print(f"{100*v/tot:5.1f}% {f}:{ln:>5} inst={n:>12} {src}")
