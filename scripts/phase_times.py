"""Per-phase device time (build / simulate kernels) per config (dev tool)."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1602_05510_b200.configs import CONFIGS, make_engine  # noqa: E402
for name, n in [("C1", 100000), ("C2", 100000), ("C3", 100000), ("C4", 50000)]:
    eng = make_engine(CONFIGS[name])
    eng.eval_generated(0, 2000, outcomes=False)
    _, b = eng.eval_generated(10_000_000, n, outcomes=False)
    print(f"{name}: {n} cand build {b.build_ms:.1f} ms sim {b.sim_ms:.1f} ms total {b.kernel_ms:.1f} ms "
          f"-> {n / b.kernel_ms * 1e3:,.0f}/s; leaves/cand {b.sum_leaves / n:.0f} edges/cand {b.sum_edges / n:.0f}")
