"""Attribute ncu source-page samples/instructions (csv, --print-source cuda,sass)
to engine phases: engine.h functions/lambdas plus marked sub-sections of the
event loop.  usage: ncu_phases.py <src.csv> <engine.h> <n_candidates>"""
import csv
import re
import sys
from collections import defaultdict

src, eng, ncand = sys.argv[1], sys.argv[2], float(sys.argv[3])
marks = []
for i, l in enumerate(open(eng), 1):
    m = re.match(r"\s*(?:static )?HXN? [\w:<>&\* ]+? (\w+)\(", l) or re.match(r"\s*auto (\w+) = \[", l)
    if m:
        marks.append((i, m.group(1)))
    for tag, name in (("NOUNROLL while (committed < nl)", "loop:epoch+ready"),
                      ("---------------- processor selection", "loop:select"),
                      ("---------------- commit (sim.cpp", "loop:commit"),
                      ("// write coherence (sim.cpp:625-628)", "loop:coherence"),
                      ("// release successors (sim.cpp:660-667)", "loop:release")):
        if tag in l:
            marks.append((i, name))
marks.sort()


def fn(line):
    name = "?"
    for n, f in marks:
        if n <= line:
            name = f
    return name


agg = defaultdict(lambda: defaultdict(int))
cur_file = hdr = cur = None
for r in csv.reader(open(src)):
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
        cur = (cur_file, int(r[0]))
        continue
    try:
        v, n = int(r[si] or 0), int(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    if not cur:
        continue
    key = fn(cur[1]) if cur[0] == "engine.h" else cur[0]
    toks = (r[3].strip() if len(r) > 3 else "").split()
    op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")).split(".")[0]
    a = agg[key]
    a["samp"] += v
    a["inst"] += n
    if op in ("LDL", "STL", "LD", "ST"):
        a[op] += n
tot = sum(a["samp"] for a in agg.values())
ti = sum(a["inst"] for a in agg.values())
print(f"warp-instructions per candidate: {ti / ncand:,.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["samp"])[:26]:
    print(f"{100 * a['samp'] / tot:5.1f}% samples  inst/cand={a['inst'] / ncand:>9,.0f}  LDL={a['LDL'] / ncand:>7,.0f} "
          f"STL={a['STL'] / ncand:>6,.0f} LD={a['LD'] / ncand:>7,.0f} ST={a['ST'] / ncand:>6,.0f}  {k}")
