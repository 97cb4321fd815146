"""One-off large parity validation on the GPU (dev tool): every record of
build/validation/<preset>_<first>_<count>.bin (reference records written by
scripts/validation_refs.sh) against the engine, through the device generator
and through host descriptors.  Prints one JSON summary line."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from golden_io import compare, read_golden  # noqa: E402
from paper_1602_05510_b200.configs import CONFIGS, PARITY, make_engine  # noqa: E402

summary = {}
for path in sorted(glob.glob(os.path.join(ROOT, "build", "validation", "*.bin"))):
    name = os.path.basename(path)[:-4]
    preset, first, count = name.rsplit("_", 2)
    first, count = int(first), int(count)
    p = CONFIGS.get(preset) or PARITY[preset][0]
    g = read_golden(path)
    assert len(g) == count and int(g["index"][0]) == first
    eng = make_engine(p)
    out, best = eng.eval_generated(first, count)
    bad = compare(out, g, first=first)
    descs = eng.generate_host(first, count)
    out2, _ = eng.eval_descs(descs, first=first)
    bad2 = compare(out2, g, first=first)
    ok = g[g["status"] == 0]
    sts = {int(k): int(v) for k, v in zip(*np.unique(g["status"], return_counts=True))}
    win = ok[np.lexsort((ok["index"], ok["makespan"]))][0] if len(ok) else None
    summary[name] = {"records": count, "mismatches_generated": len(bad), "mismatches_host_descriptors": len(bad2),
                     "statuses": sts,
                     "best_matches": bool(win is not None and best.index == int(win["index"])
                                          and best.makespan == float(win["makespan"])),
                     "first_mismatch": (bad + bad2)[:1]}
print(json.dumps(summary))
