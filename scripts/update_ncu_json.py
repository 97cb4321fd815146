"""Refresh profiles/ncu_issue.json and profiles/ncu_eval_kernel.json (read by
bench.py for issue_roofline and roofline.traffic) from an ncu metrics csv of
one bench step (scripts/profile.sh step 3: build_kernel + sim_kernel of one
1e5-candidate C2 chunk).  usage: update_ncu_json.py <traffic.csv> <tag>"""
import csv
import json
import os
import sys

path, tag = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
first = {}
for r in rows[h + 1:]:
    k = "sim_kernel" if "sim_kernel" in r[ki] else ("build_kernel" if "build_kernel" in r[ki] else None)
    if k is None:
        continue
    d = first.setdefault((k, r[0]), {})
    d[r[mi]] = float(r[vi].replace(",", ""))
per = {}
for (k, _), d in sorted(first.items(), key=lambda x: int(x[0][1])):
    per.setdefault(k, d)  # the first launch of each kernel
n = 100_000
root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
issue = {"config": "C2", "source": f"ncu smsp__inst_executed.sum of one bench step (profiles/{tag}_traffic.csv, 1e5 candidates)",
         "warp_inst_per_candidate": {k: round(per[k]["smsp__inst_executed.sum"] / n) for k in per}}
dram = per["sim_kernel"]["dram__bytes_read.sum"] + per["sim_kernel"]["dram__bytes_write.sum"]
evalk = {"config": "C2", "batch": n, "kernel": "sim_kernel", "dram_bytes_per_launch": int(dram),
         "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum (profiles/{tag}_traffic.csv)"}
json.dump(issue, open(os.path.join(root, "ncu_issue.json"), "w"))
json.dump(evalk, open(os.path.join(root, "ncu_eval_kernel.json"), "w"))
print(issue, evalk)
