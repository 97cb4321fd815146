import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1602_05510_b200.configs import CONFIGS, make_engine
eng = make_engine(CONFIGS["C2"])
h, best, mk, it, n = eng.solve(20, "All", "Exact", 0)
print("state ops", int(best["n_ops"]))
d = eng.generate_host(0, 50000)
out, b = eng.eval_descs(d)
print(f"random C2 50k: build {b.build_ms:.1f} sim {b.sim_ms:.1f} leaves/cand {b.sum_leaves/50000:.0f}")
# mutations of the solver state: append one partition of a random base leaf id
rng = np.random.default_rng(0)
m = np.repeat(best[None], 50000)
k = int(best["n_ops"])
m["n_ops"] = k + 1
m["ops"][:, k, 0] = rng.integers(1, 817, 50000)
m["ops"][:, k, 1] = 2
out, b = eng.eval_descs(m)
ok = (out["status"] == 0).sum()
print(f"state+1 op 50k: build {b.build_ms:.1f} sim {b.sim_ms:.1f} leaves/cand {b.sum_leaves/50000:.0f} ok {ok}")
