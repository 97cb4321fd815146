"""A/B probe of one engine build (dev tool; bench.py is the contract).
usage: HESP_LIB=x.so python scripts/ab_probe.py <preset> <count> [golden]
Checks the first records against a golden set (bit-exact), then times two
batches of <count> generated candidates; prints one JSON line with the
device kernel times (build / simulate) and candidates/s."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402,F401

from golden_io import compare, read_golden  # noqa: E402
from paper_1602_05510_b200.configs import CONFIGS, make_engine  # noqa: E402

name = sys.argv[1]
count = int(sys.argv[2])
gold = sys.argv[3] if len(sys.argv) > 3 else None
eng = make_engine(CONFIGS[name])
res = {"lib": os.environ.get("HESP_LIB", "default"), "preset": name, "loop": os.environ.get("HESP_LOOP", "0")}
if gold:
    g = read_golden(gold)
    out, _ = eng.eval_generated(0, len(g))
    bad = compare(out, g)
    res["parity"] = f"{len(g) - len(bad)}/{len(g)}"
    if bad:
        res["first_bad"] = bad[:2]
eng.eval_generated(5_000_000, min(count, 4096), outcomes=False)
torch.cuda.synchronize()
rates, sims, builds = [], [], []
for rep in range(2):
    t = time.perf_counter()
    _, b = eng.eval_generated(10_000_000 + rep * count, count, outcomes=False)
    dt = time.perf_counter() - t
    rates.append(count / dt)
    sims.append(b.sim_ms)
    builds.append(b.build_ms)
res.update(rate=round(max(rates)), sim_ms=round(min(sims), 2), build_ms=round(min(builds), 2),
           info={"blocks_per_sm": eng.info().blocks_per_sm})
print(json.dumps(res))
