"""SPEC.md acceptance 9 at desk scale: 1 fast + 4 slow processors (8x speed
ratio, different efficiency half-sizes), n = 4096 Cholesky.  The best
homogeneous uniform tiling over s in {2, 4, 8, 16} vs the solver (All,
200 iterations) started from the uniform s = 4 tiling (SPEC's example) and
from the best homogeneous tiling, Soft (8 seeds) and Exact, for FCFS/R-P and
PL/EFT-P.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_05510_b200.configs import make_engine, preset  # noqa: E402

FIX = ("platform_fastslow.json", "model_fastslow.json")
out = {}
for ordering, selection in [("FCFS", "R-P"), ("PL", "EFT-P")]:
    homo = {}
    for s in (2, 4, 8, 16):
        eng = make_engine(preset(FIX, 4096, 8, s, 0, ordering=ordering, selection=selection, sched_seed=1))
        o, _ = eng.eval_generated(0, 1)
        homo[s] = float(o[0]["makespan"])
    best_s = min(homo, key=homo.get)
    best_h = homo[best_s]
    row = {"homogeneous": homo, "best_homogeneous": best_h, "best_s": best_s}
    for start in (4, best_s):
        eng = make_engine(preset(FIX, 4096, 8, start, 0, ordering=ordering, selection=selection, sched_seed=1))
        chains = eng.solve_batch([dict(iterations=200, task_selection="All", sampling="Soft", seed=sd)
                                  for sd in range(8)] + [dict(iterations=200, sampling="Exact")])
        soft = [c[2] for c in chains[:8]]
        row[f"from_s{start}"] = {"soft_per_seed": soft, "exact": chains[8][2],
                                 "soft_seed0_improvement_pct": 100 * (best_h - soft[0]) / best_h,
                                 "soft_best_of_8_improvement_pct": 100 * (best_h - min(soft)) / best_h,
                                 "exact_improvement_pct": 100 * (best_h - chains[8][2]) / best_h}
    out[f"{ordering}/{selection}"] = row
print(json.dumps(out))
