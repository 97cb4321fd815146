"""Batched solver chains (hesp_solve_batch) vs one chain at a time, C2 (dev/evidence tool)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_05510_b200.configs import CONFIGS, make_engine  # noqa: E402

n_chains = int(sys.argv[1]) if len(sys.argv) > 1 else 16
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
eng = make_engine(CONFIGS["C2"])
eng.solve(2, "All", "Soft", 0)
chains = [dict(iterations=iters, sampling="Soft", seed=s) for s in range(n_chains - 1)] + \
         [dict(iterations=iters, sampling="Exact", seed=0)]
t = time.perf_counter()
many = eng.solve_batch(chains)
tb = time.perf_counter() - t
t = time.perf_counter()
one = eng.solve(iters, "All", "Soft", 0)
t1 = time.perf_counter() - t
best = min(m[2] for m in many)
print(json.dumps({"config": "C2", "chains": n_chains, "iterations": iters, "batched_s": tb,
                  "chain_iterations_per_s": n_chains * iters / tb, "single_chain_s": t1,
                  "single_chain_iterations_per_s": iters / t1, "best_makespan_over_chains": best,
                  "best_soft_chain": min(m[2] for m in many[:-1]), "exact_chain": many[-1][2],
                  "device_sims": sum(m[4] for m in many),
                  "first_chain_matches_single": many[0][0].tobytes() == one[0].tobytes()}))
