"""Size-independent properties of the engine's schedules (SPEC.md acceptance
criteria 1, 4, 5, 6), checked on the device output for many candidates --
beyond the candidates the golden records pin."""
import numpy as np
import pytest

from paper_1602_05510_b200.configs import PARITY, preset, make_engine, CPUGPU
from paper_1602_05510_b200.engine import load_model

pytestmark = pytest.mark.gpu


def task_flops(kind, b):  # platform.cpp:57-66
    bd = float(b)
    return (bd * bd * bd / 3.0, bd * bd * bd, bd * bd * bd, 2.0 * bd * bd * bd)[kind]


def analytic_time(model, kind, b, type_name):  # PerfModel::task_time, platform.cpp:351-357
    from paper_1602_05510_b200.engine import KINDS
    for k, t, peak, bh in model.analytic:
        if KINDS[k] == kind and t == type_name:
            eff = float(b) / (float(b) + bh)
            return task_flops(kind, b) / (peak * eff)
    raise KeyError((kind, type_name))


@pytest.mark.parametrize("s", [2, 4, 8, 16])
def test_task_count_law(lib, s):
    """Criterion 1: a uniform s-tile Cholesky has s(s+1)(s+2)/6 tasks."""
    eng = make_engine(preset(CPUGPU, 16384, 4, s, 0))
    out, _ = eng.eval_generated(0, 1)
    assert int(out[0]["status"]) == 0 and int(out[0]["n_leaves"]) == s * (s + 1) * (s + 2) // 6


def test_serial_identity(lib):
    """Criterion 6: on one processor the makespan is the plain sum of the task
    times in commit order, exactly -- for random partitionings with merges."""
    p, _ = PARITY["serial"]
    eng = make_engine(p)
    model = load_model(p["model"])
    descs = eng.generate_host(0, 40)
    for d in descs:
        tr = eng.eval_trace(d)
        if tr.status:
            continue
        order = np.argsort(tr.assignments["start"], kind="stable")
        a = tr.assignments[order]
        ev = {int(e["id"]): (int(e["task_kind"]), int(e["b"])) for e in tr.events if int(e["kind"]) == 0}
        t = 0.0
        for row in a:
            assert row["start"] == t
            kind, b = ev[int(row["task"])]
            t = t + analytic_time(model, kind, b, "big")
            assert row["end"] == t
        assert tr.makespan == t


@pytest.mark.parametrize("name", ["c2", "c3", "sect_cpugpu", "table", "merge_c2", "policy_FCFS_R-P_WT",
                                  "policy_PL_F-P_WA", "deep_biglittle"])
def test_schedules_verify_and_respect_work_bound(lib, name):
    """Criteria 4 and 5: verify_schedule finds nothing, and the makespan is at
    least the work bound sum_t min_type time(t) / P."""
    p, _ = PARITY[name]
    eng = make_engine(p)
    model = load_model(p["model"])
    import json
    import os
    from paper_1602_05510_b200.engine import FIXTURES
    plat = json.load(open(os.path.join(FIXTURES, p["platform"])))
    types = [t["name"] for t in plat["types"]]
    P = len(plat["processors"])
    descs = eng.generate_host(50_000, 64)  # 8 presets x 64 = 512 randomized simulations
    checked = 0
    for d in descs:
        tr = eng.eval_trace(d)
        if tr.status:
            continue
        assert eng.verify_trace(tr) == []
        cp, wb = eng.trace_bounds()
        assert tr.makespan >= cp * (1 - 1e-12) and tr.makespan >= wb * (1 - 1e-12)
        if model.analytic is not None:
            work = 0.0
            for e in tr.events:
                if int(e["kind"]) == 0:
                    work += min(analytic_time(model, int(e["task_kind"]), int(e["b"]), ty) for ty in types)
            assert tr.makespan * (1 + 1e-12) >= work / P
        assert tr.busy_time <= P * tr.makespan * (1 + 1e-12)
        checked += 1
    assert checked > 0


@pytest.mark.parametrize("name,count", [("c2", 20000), ("c4", 2000), ("evict_wa", 2000), ("sect_cpugpu", 5000),
                                        ("merge_c2", 5000), ("policy_FCFS_R-P_WT", 5000)])
def test_warp_and_scalar_engines_agree_at_scale(lib, name, count):
    """Two independent device code paths over the same candidates: the
    warp-parallel simulate kernel (lanes = processors, (block, space) EFT
    lanes, redux argmins) and the width-1 thread-per-candidate kernel (the
    reference's loops as written) must produce bit-identical outcome records
    for every candidate -- a full-scale check beyond the golden sizes."""
    import os
    from paper_1602_05510_b200.configs import CONFIGS
    p = (PARITY.get(name) or (CONFIGS[name.upper()], 0))[0]
    warp = make_engine(p)
    os.environ["HESP_SIM_THREAD"] = "1"
    try:
        scalar = make_engine(p)
    finally:
        del os.environ["HESP_SIM_THREAD"]
    a, ba = warp.eval_generated(123_000, count)
    b, bb = scalar.eval_generated(123_000, count)
    assert a.tobytes() == b.tobytes()
    assert (ba.makespan, ba.index, ba.n_ok) == (bb.makespan, bb.index, bb.n_ok)


def test_merge_round_trip_and_flop_conservation(lib):
    """SPEC acceptance 3: merge(partition(g)) reproduces g's schedule bit for
    bit (same leaves, makespan, assignment and transfer hashes), for
    partitions of every kind and tile count; acceptance 2: the leaves of
    random partition/merge sequences keep sum(flops) = n^3/3 (1e-9 rel)."""
    from paper_1602_05510_b200.engine import DESC_DTYPE, OP_MERGE
    p, _ = PARITY["c2"]
    eng = make_engine(p)
    base = np.zeros(1, DESC_DTYPE)
    out0, _ = eng.eval_descs(base)
    cases = [(t, s) for t in (1, 2, 17, 18, 100, 500, 815) for s in (2, 4, 8)]
    d = np.zeros(len(cases), DESC_DTYPE)
    for i, (t, s) in enumerate(cases):
        d[i]["n_ops"] = 2
        d[i]["ops"][0] = (t, s)
        d[i]["ops"][1] = (1, OP_MERGE)
    out, _ = eng.eval_descs(d)
    for i in range(len(cases)):
        assert out[i].tobytes() == out0[0].tobytes(), cases[i]
    n = float(p["n"])
    pm = dict(p, merge_pct=35)
    eng2 = make_engine(pm)
    for desc in eng2.generate_host(0, 24):
        tr = eng2.eval_trace(desc)
        if tr.status:
            continue
        fl = 0.0
        for e in tr.events:
            if int(e["kind"]) == 0:
                fl += task_flops(int(e["task_kind"]), int(e["b"]))
        assert abs(fl - n ** 3 / 3.0) <= 1e-9 * n ** 3 / 3.0


def test_dag_depths_figure3(lib):
    """Acceptance 8 (Figure 3, from the base tiling on): the base tiling has
    depth 1, partitioning a base task makes 2, a second base task keeps 2, a
    sub-task of the first makes 3 (IterationRecord.dag_depth of one round)."""
    from paper_1602_05510_b200.engine import DESC_DTYPE
    p, _ = PARITY["c2"]
    eng = make_engine(p)
    want = {(): 1, ((1, 2),): 2, ((1, 2), (2, 2)): 2, ((1, 2), (817, 2)): 3}
    for ops, depth in want.items():
        d = np.zeros(1, DESC_DTYPE)
        d[0]["n_ops"] = len(ops)
        for i, o in enumerate(ops):
            d[0]["ops"][i] = o
        hist, *_ = eng.solve(1, "All", "Hard", 0, initial=d[0])
        assert int(hist[0]["dag_depth"]) == depth, ops
