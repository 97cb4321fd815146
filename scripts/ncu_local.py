"""Per-source-line warp-instructions, local-memory (LDL/STL) instructions and
stall samples from an ncu source page (--page source --csv --print-source
cuda,sass), SASS rows deduplicated by address.
usage: ncu_local.py <src.csv> <n_candidates> [top]"""
import csv
import sys
from collections import defaultdict


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


path, ncand = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
hdr = fname = cur = None
byline = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
seen = set()
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        byline[cur][3] = r[1].strip()[:80]
        continue
    if r[2] in seen or r[2] == "...":
        continue
    seen.add(r[2])
    v = byline[cur]
    v[0] += f(r[si])
    v[1] += f(r[ie])
    if "LDL" in r[3] or "STL" in r[3]:
        v[2] += f(r[ie])
ts = sum(v[0] for v in byline.values()) or 1
ti = sum(v[1] for v in byline.values())
tl = sum(v[2] for v in byline.values())
print(f"warp-inst/cand {ti/ncand:.0f}  local-inst/cand {tl/ncand:.0f}")
for key, name in ((2, "local inst"), (0, "stall samples")):
    print(f"--- top lines by {name}")
    for k, v in sorted(byline.items(), key=lambda x: -x[1][key])[:top]:
        print(f"{k[0]}:{k[1]:5d} inst={v[1]/ncand:8.0f} loc={v[2]/ncand:6.0f} smp={100*v[0]/ts:5.1f}%  {v[3]}")
