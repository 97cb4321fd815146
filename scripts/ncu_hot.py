"""Per-source-line instructions and stall samples from an ncu source-page csv
(--print-source cuda,sass), deduplicated by SASS address.  usage:
ncu_hot.py <src.csv> <n_candidates> [top] -- prints line, share of samples, warp-inst per candidate."""
import csv
import sys
from collections import defaultdict

path, ncand = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
hdr = cur = fname = None
byaddr = {}
srcline = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        srcline[cur] = r[1].strip()[:90]
        continue
    if r[2].startswith("0x"):
        a = int(r[2], 16)
        if a in byaddr:
            continue
        try:
            byaddr[a] = (float(r[ie] or 0), float(r[si] or 0), cur)
        except ValueError:
            pass
tot = sum(v[0] for v in byaddr.values())
st = sum(v[1] for v in byaddr.values()) or 1
agg = defaultdict(lambda: [0.0, 0.0])
for n, sm, cur in byaddr.values():
    agg[cur][0] += n
    agg[cur][1] += sm
print(f"warp-inst per candidate {tot / ncand:,.0f}")
for k, (n, sm) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{100 * sm / st:5.1f}% {n / ncand:9.0f} {k[0]}:{k[1]:<5} {srcline.get(k, '')}")
