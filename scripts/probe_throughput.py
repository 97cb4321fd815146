"""Quick device-throughput probe for a preset (dev tool; bench.py is the contract)."""
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch  # noqa: E402

from paper_1602_05510_b200.configs import CONFIGS, make_engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
eng = make_engine(CONFIGS[name])
i = eng.info()
print(f"{name}: slots={i.n_slots} sm={i.sm_count} blocks/sm={i.blocks_per_sm} slot_bytes={i.slot_bytes}")
eng.eval_generated(0, min(count, 2000), outcomes=False)
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter()
    out, best = eng.eval_generated(10_000_000 + rep * count, count, outcomes=True)
    dt = time.perf_counter() - t
    ok = (out["status"] == 0).sum()
    print(f"{name}: {count} cand in {dt*1e3:.1f} ms -> {count/dt:,.0f} cand/s; ok={ok} best={best.makespan:.6f}@{best.index} "
          f"statuses={dict(zip(*[a.tolist() for a in __import__('numpy').unique(out['status'], return_counts=True)]))}")
