"""GPU parity of the full-trace path: hesp_eval_trace
reproduces the unmodified reference's entire SimResult for one candidate --
assignments, transfers with routes and fragments, the time-ordered event
list, the residency log, idle_avg -- plus compute_load_trace, busy_time /
avg_load / LoadTrace::integral and verify_schedule's messages, every double
bit for bit (goldens: tests/golden/trace_*.json.gz from oracle/_ref)."""
import numpy as np
import pytest

from paper_1602_05510_b200.configs import PARITY, make_engine
from trace_io import SHIFT_NAMES, TRACE_NAMES, hbits, read_shift, read_trace

pytestmark = pytest.mark.gpu

_engines = {}


def engine(preset):
    if preset not in _engines:
        _engines[preset] = make_engine(PARITY[preset][0])
    return _engines[preset]


def traced(name):
    g = read_trace(name)
    eng = engine(g["preset"])
    if g.get("descs"):  # an explicit descriptor (e.g. after a merge of the base cluster)
        import os
        from golden_io import GOLDEN_DIR
        from paper_1602_05510_b200.engine import DESC_DTYPE
        desc = np.fromfile(os.path.join(GOLDEN_DIR, f"{g['descs']}.descs"), DESC_DTYPE)[g["index"]:g["index"] + 1]
    else:
        desc = eng.generate_host(g["index"], 1)
    return g, eng, eng.eval_trace(desc[0])


def ours_transfers(tr):
    out = []
    for x in tr.transfers:
        frag = [int(v) for v in x["frag"]] if x["has_fragment"] else None
        route = [[int(x["hop_src"][h]), int(x["hop_dst"][h])] for h in range(int(x["n_hops"]))]
        out.append([int(x["block"]), int(x["src_space"]), int(x["dst_space"]), int(x["bytes"]), hbits(x["start"]),
                    hbits(x["end"]), frag, route])
    return out


@pytest.mark.parametrize("name", TRACE_NAMES)
def test_trace_matches_reference(lib, name):
    g, eng, tr = traced(name)
    assert tr.status == g["status"] == 0
    assert tr.n_leaves == g["leaves"]
    assert hbits(tr.makespan) == g["makespan"]
    ours = [[int(a["task"]), int(a["proc"]), hbits(a["start"]), hbits(a["end"]), hbits(a["idle_avg"])]
            for a in tr.assignments]
    assert ours == g["assignments"]
    assert ours_transfers(tr) == g["transfers"]
    ev = [[["TaskStart", "TaskEnd", "XferStart", "XferEnd"].index(k), hbits(t), s, r]
          for k, t, s, r in tr.event_strings()]
    assert ev == g["events"]
    res = [[hbits(r["time"]), int(r["space"]), int(r["delta_bytes"]), int(r["block"])] for r in tr.residency]
    assert res == g["residency"]
    assert [[hbits(s["time"]), int(s["active"])] for s in tr.steps] == g["load"]
    assert (hbits(tr.busy_time), hbits(tr.avg_load), hbits(tr.load_integral)) == (g["busy"], g["avg_load"],
                                                                                   g["integral"])
    assert eng.verify_trace(tr) == g["violations"]


@pytest.mark.parametrize("name", SHIFT_NAMES)
def test_verify_schedule_on_edited_trace(lib, name):
    """verify_schedule over a schedule with one task moved: the same violations,
    in the same order and wording, as the reference's verify_schedule."""
    s = read_shift(name)
    _, eng, tr = traced(s["trace"])
    a = tr.assignments
    k = int(np.nonzero(a["task"] == s["task"])[0][0])
    a["start"][k] = a["start"][k] - s["shift_by"]
    a["end"][k] = a["end"][k] - s["shift_by"]
    got = eng.verify_trace(tr)
    assert got == s["violations"]
    assert got  # the edit must be caught


def test_trace_agrees_with_batch_outcome(lib):
    """The trace kernel (full bookkeeping, no E4 fast path) and the batch
    kernels (fast path) give the same makespan on a batch of C2 candidates."""
    p, _ = PARITY["c2"]
    eng = engine("c2")
    descs = eng.generate_host(0, 8)
    out, _ = eng.eval_descs(descs)
    for i in range(8):
        tr = eng.eval_trace(descs[i])
        assert tr.status == int(out[i]["status"])
        if tr.status == 0:
            assert hbits(tr.makespan) == hbits(out[i]["makespan"])
            assert len(tr.assignments) == int(out[i]["n_leaves"])
            assert eng.verify_trace(tr) == []


def test_verify_c4_winner_fast_and_clean(lib):
    """The device validator on a 32x32 (C4) schedule: clean on the engine's own
    schedule, catches a moved task, and takes well under a second."""
    import time
    p, _ = PARITY["c4"]
    eng = make_engine(p)
    descs = eng.generate_host(0, 4)
    out, _ = eng.eval_descs(descs)
    k = int(np.nonzero(out["status"] == 0)[0][0])
    tr = eng.eval_trace(descs[k])
    assert tr.status == 0 and len(tr.assignments) > 5000
    eng.verify_trace(tr)  # warm-up (module load)
    t0 = time.perf_counter()
    v = eng.verify_trace(tr)
    dt = time.perf_counter() - t0
    assert v == [] and dt < 1.0, (v[:3], dt)
    a = tr.assignments
    a["start"][100] -= 0.01
    a["end"][100] -= 0.01
    assert eng.verify_trace(tr)
