import sys; sys.path.insert(0,'.')
from paper_1602_05510_b200.configs import make_engine, preset
fix = ("platform_fastslow.json", "model_fastslow.json")
for ordering, selection, s in [("FCFS", "R-P", 16), ("PL", "EFT-P", 8)]:
    eng = make_engine(preset(fix, 4096, 8, s, 0, ordering=ordering, selection=selection, sched_seed=1))
    h, b, mk, it, n = eng.solve(200, "All", "Soft", 0)
    print(ordering, "load0 %.2f" % h[0]["avg_load_pct"], "mk0 %.6f best %.6f impr %.3f%%" % (h[0]["makespan"], mk, 100*(h[0]["makespan"]-mk)/h[0]["makespan"]))
