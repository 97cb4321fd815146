"""Solver timing: hesp_solve on the device engine vs the
same SPEC restatement driven by the unmodified reference on the host cores
(oracle/_ref/ref_harness --solve).  Dev/evidence tool; prints one JSON line."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_05510_b200.configs import CONFIGS, PARITY, harness_args, make_engine  # noqa: E402
from paper_1602_05510_b200.engine import FIXTURES  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ref_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = CONFIGS.get(name) or PARITY[name][0]
eng = make_engine(p)
eng.solve(2, "All", "Soft", 1)  # warm-up
t = time.perf_counter()
hist, best, mk, it, nsim = eng.solve(iters, "All", "Soft", 1)
dt = time.perf_counter() - t
line = {"config": name, "iterations": iters, "gpu_s": dt, "gpu_s_per_iter": dt / iters, "device_sims": nsim,
        "best_makespan": mk, "best_iteration": it, "first_makespan": float(hist[0]["makespan"]),
        "candidates_per_iter": float(hist["n_candidates"][:-1].mean()) if iters > 1 else 0}
h = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
if ref_iters > 0 and os.path.exists(h):
    t = time.perf_counter()
    r = subprocess.run([h, *harness_args(p, FIXTURES), "--threads", str(os.cpu_count()), "--solve", str(ref_iters),
                        "--solve-selection", "All", "--solve-sampling", "Soft", "--solve-seed", "1"],
                       capture_output=True, text=True, check=True)
    rt = time.perf_counter() - t
    d = json.loads(r.stdout)
    line.update(ref_iterations=ref_iters, ref_s=rt, ref_s_per_iter=rt / ref_iters, ref_threads=os.cpu_count(),
                same_prefix=[x[9] for x in d["history"]] == [f"{int(__import__('numpy').float64(v).view('<u8')):016x}"
                                                             for v in hist["makespan"][:ref_iters]])
print(json.dumps(line))
