"""CPU-only tests (no GPU): golden fixtures, the C ABI surface, the candidate
generator, host-side sharding, and -- where oracle/_ref is built (build() runs
`make -C oracle` when /root/reference exists) -- the unmodified reference
reproducing the committed goldens and the engine's width-1 host build
matching the reference candidate by candidate."""
import json
import os
import re
import subprocess

import numpy as np
import pytest

from golden_io import read_golden
from paper_1602_05510_b200.configs import C2, PARITY, SCALE, harness_args
from paper_1602_05510_b200.dist import shard
from paper_1602_05510_b200.engine import EXPORTS, FIXTURES, Workload, generate_batch, load_library

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
HARNESS = os.path.join(REF, "ref_harness")
ENGINE_CHECK = os.path.join(REF, "engine_check")

# hesp::Err ordinals + 1 that a valid generator must never provoke
GEN_ERRORS = {1 + 1: "Validation", 1 + 7: "NotALeaf", 1 + 8: "IndivisibleGrain", 100: "foreign exception"}


@pytest.mark.parametrize("name", sorted(PARITY) + sorted(SCALE))
def test_golden_fixture_shape(name):
    p, count = {**PARITY, **SCALE}[name]
    g = read_golden(name)
    assert len(g) == count
    assert list(g["index"]) == list(range(count))
    errs = list(GEN_ERRORS)
    if name == "scale_merge_sect":  # the reference's own prune defect: std::out_of_range
        errs.remove(100)
    assert not np.isin(g["status"], errs).any(), "generator emitted an op the reference rejected"
    ok = g[g["status"] == 0]
    bad = g[g["status"] != 0]
    assert (ok["makespan"] > 0).all() and (ok["n_leaves"] > 0).all()
    assert (bad["makespan"] == 0).all() and (bad["assign_hash"] == 0).all()


def test_scale_goldens_extend_the_parity_sets():
    """The at-scale records (>= 1e4 C2/C3, 256 C4, 1e3 per eviction fixture)
    start with exactly the parity set's records where the presets coincide."""
    assert SCALE["scale_c2"][1] >= 10_000 and SCALE["scale_c3"][1] >= 10_000 and SCALE["scale_c4"][1] >= 256
    for scale, small in (("scale_c2", "c2"), ("scale_c3", "c3"), ("scale_c4", "c4"), ("scale_evict_wb", "evict_wb"),
                         ("scale_merge_c2", "merge_c2"), ("scale_sect_cpugpu", "sect_cpugpu"),
                         ("scale_merge_sect", "merge_sect")):
        a, b = read_golden(scale), read_golden(small)
        assert a[:len(b)].tobytes() == b.tobytes(), scale


def test_goldens_exercise_every_path():
    """The fixture set covers errors, eviction, intersections, every policy."""
    statuses = set()
    for name in PARITY:
        statuses |= set(read_golden(name)["status"].tolist())
    assert 0 in statuses and 20 in statuses  # ok and CoherenceError
    assert sum(1 for n in PARITY if n.startswith("policy_")) == 24


def test_library_exports_every_declared_symbol():
    lib = load_library()
    with open(os.path.join(ROOT, "include", "hesp_engine.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(hesp_[a-z_]+)\s*\(", hdr))
    declared -= {"hesp_engine"}
    assert declared, "no declarations parsed"
    for sym in sorted(declared):
        getattr(lib, sym)  # raises AttributeError if not exported
    assert set(EXPORTS) <= declared


def test_status_names():
    lib = load_library()
    assert lib.hesp_status_name(0) == b"ok"
    assert lib.hesp_status_name(20) == b"CoherenceError"
    assert lib.hesp_status_name(14) == b"CapacityInfeasible"
    assert lib.hesp_status_name(201) == b"EngineLimit"


def c2_workload():
    p = C2
    return Workload(p["n"], p["elem"], p["s_base"], p["seed"], p["k_max"], p["max_depth"], p["min_block"],
                    p["s_choices"])


def test_generator_is_deterministic_and_bounded():
    wl = c2_workload()
    a = generate_batch(wl, 816, 1024, 0, 4096)
    b = generate_batch(wl, 816, 1024, 0, 4096)
    assert a.tobytes() == b.tobytes()
    assert (a["n_ops"] >= 0).all() and (a["n_ops"] <= wl.k_max).all()
    # all K in [0, k_max] occur, and ops address existing task ids with allowed s
    assert set(a["n_ops"].tolist()) == set(range(wl.k_max + 1))
    for d in a[:512]:
        n = int(d["n_ops"])
        ops = d["ops"][:n]
        assert set(ops[:, 1].tolist()) <= set(wl.s_choices)
        assert (ops[:, 0] >= 1).all()
        assert (d["ops"][n:, 0] == -1).all()
    # a different seed gives a different stream
    wl2 = c2_workload()
    wl2.seed = 2
    c = generate_batch(wl2, 816, 1024, 0, 4096)
    assert a.tobytes() != c.tobytes()
    # an index range is a slice of a longer one
    d = generate_batch(wl, 816, 1024, 100, 50)
    assert d.tobytes() == a[100:150].tobytes()


@pytest.mark.parametrize("total,world", [(100_000, 1), (100_000, 8), (10, 3), (7, 8)])
def test_shard_partitions_the_index_range(total, world):
    seen = []
    for r in range(world):
        b, e = shard(total, world, r, first=5)
        assert 0 <= e - b <= total // world + 1
        seen.extend(range(b, e))
    assert seen == list(range(5, 5 + total))


def _records(path):
    from golden_io import read_golden as rg
    return rg(path)


REF_PRESETS = ["c1", "c3", "policy_PL_EFT-P_WB", "policy_FCFS_R-P_WA", "evict_wb", "sect_cpugpu", "table"]


@pytest.mark.skipif(not os.path.exists(HARNESS), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("name", REF_PRESETS)
def test_reference_reproduces_goldens(name, tmp_path):
    p, count = PARITY[name]
    k = min(count, 6)
    out = tmp_path / f"{name}.bin"
    subprocess.run([HARNESS, *harness_args(p, FIXTURES), "--first", "0", "--count", str(k), "--threads",
                    str(os.cpu_count()), "--out", str(out), "--quiet"], check=True)
    got = _records(str(out))
    want = read_golden(name)[:k]
    assert got.tobytes() == want.tobytes()


CHECK_PRESETS = ["c3", "policy_PL_EFT-P_WB", "policy_FCFS_EIT-P_WT", "policy_PL_F-P_WA", "policy_FCFS_R-P_WB",
                 "evict_wb", "evict_wa", "sect_cpugpu", "sect_biglittle", "deep_biglittle", "table", "merge_c2",
                 "merge_evict", "merge_c3"]


@pytest.mark.skipif(not os.path.exists(ENGINE_CHECK), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("name", CHECK_PRESETS)
def test_host_engine_matches_reference(name):
    """Engine<HostWarp> (the engine source at width 1) vs the reference library."""
    p, count = PARITY[name]
    r = subprocess.run([ENGINE_CHECK, *harness_args(p, FIXTURES), "--first", "0", "--count", str(min(count, 8))],
                       capture_output=True, text=True, timeout=600)
    assert "mismatches 0" in r.stdout, r.stdout[-2000:]
    assert r.returncode == 0


@pytest.mark.skipif(not os.path.exists(ENGINE_CHECK), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("name", ["merge_sect", "merge_sect_bl"])
def test_host_engine_merges_with_intersections(name):
    """merge_cluster while intersection descriptors live (graph.cpp:214-266): the
    engine's emulation of their DataDag parent links (minimal containers plus
    the non-Hasse links of found intersections, relinks through dead parents)
    erases exactly the intersections the reference's prune erases -- the whole
    parity set, including the reference's own std::out_of_range (status 100)."""
    p, count = PARITY[name]
    r = subprocess.run([ENGINE_CHECK, *harness_args(p, FIXTURES), "--first", "0", "--count", str(count)],
                       capture_output=True, text=True, timeout=600)
    assert "mismatches 0" in r.stdout, r.stdout[-2000:]
    assert r.returncode == 0


@pytest.mark.skipif(not os.path.exists(ENGINE_CHECK), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("name,preset", [("explicit_basemerge_c2", "c2"), ("explicit_basemerge_evict", "evict_wb"),
                                         ("explicit_merge_c2", "c2"), ("explicit_c2", "c2"),
                                         ("explicit_sect", "sect_cpugpu")])
def test_host_engine_matches_reference_explicit(name, preset):
    """Engine<HostWarp> on the hand-built descriptors (merges of the base
    cluster, top-level re-tilings, error statuses) vs the reference library."""
    from golden_io import GOLDEN_DIR
    p, _ = PARITY[preset]
    r = subprocess.run([ENGINE_CHECK, *harness_args(p, FIXTURES), "--descs", os.path.join(GOLDEN_DIR, f"{name}.descs")],
                       capture_output=True, text=True, timeout=600)
    assert "mismatches 0" in r.stdout, r.stdout[-2000:]
    assert r.returncode == 0


@pytest.mark.skipif(not os.path.exists(ENGINE_CHECK), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("preset", ["c2", "evict_wb", "c3", "sect_cpugpu", "policy_FCFS_R-P_WT"])
def test_host_engine_matches_reference_on_taskgraphs(preset):
    """The TaskGraph drop-in's replay (include/hesp_b200_bridge.hpp plan_graph):
    reference graphs built by random partition_task / merge_cluster (top cluster
    included) / repartition_cluster sequences, replayed as descriptors on the
    width-1 engine, give the reference's status, leaf count and makespan bits."""
    p, _ = PARITY[preset]
    r = subprocess.run([ENGINE_CHECK, *harness_args(p, FIXTURES), "--graphs", "40"], capture_output=True, text=True,
                       timeout=600)
    assert "mismatches 0" in r.stdout, r.stdout[-2000:]
    assert r.returncode == 0


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent")
def test_reference_side_bridge_compiles(tmp_path):
    """include/hesp_b200_bridge.hpp compiles against the reference's own hesp:: types."""
    tu = tmp_path / "tu.cpp"
    tu.write_text('#include "hesp_b200_bridge.hpp"\nint main() { return 0; }\n')
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), "-I",
                    "/root/reference/proj/include", str(tu)], check=True)


# ---- full-trace goldens ----
from trace_io import TRACE_NAMES, fbits, hbits, read_trace  # noqa: E402


@pytest.mark.parametrize("name", TRACE_NAMES)
def test_trace_golden_post_passes(name):
    """The trace goldens are self-consistent with a plain restatement of the
    reference's post-passes (compute_load_trace sim.cpp:975-991,
    compute_idle_avgs sim.cpp:670-702, busy_time sim.cpp:78-82)."""
    g = read_trace(name)
    P = len(json.load(open(os.path.join(FIXTURES, PARITY[g["preset"]][0]["platform"])))["processors"])
    asg = [(a[0], a[1], fbits(a[2]), fbits(a[3]), fbits(a[4])) for a in g["assignments"]]
    deltas = sorted([(s, 1) for _, _, s, _, _ in asg] + [(e, -1) for _, _, _, e, _ in asg])
    times, active, cur, i = [], [], 0, 0
    while i < len(deltas):
        t = deltas[i][0]
        while i < len(deltas) and deltas[i][0] == t:
            cur += deltas[i][1]
            i += 1
        times.append(t)
        active.append(cur)
    assert [[hbits(t), n] for t, n in zip(times, active)] == g["load"]
    cum = [0.0] * len(times)
    for k in range(1, len(times)):
        cum[k] = cum[k - 1] + (P - active[k - 1]) * (times[k] - times[k - 1])
    import bisect

    def idle_up_to(t):
        k = bisect.bisect_right(times, t)
        if k == 0:
            return 0.0
        k -= 1
        return cum[k] + (P - active[k]) * (t - times[k])
    for task, _, s, e, idle in asg:
        dur = e - s
        want = (idle_up_to(e) - idle_up_to(s)) / dur if dur > 0 else 0.0
        assert hbits(want) == hbits(idle), task
    busy = 0.0
    for _, _, s, e, _ in asg:
        busy += e - s
    assert hbits(busy) == g["busy"]
    assert len(g["events"]) == 2 * len(asg) + 2 * sum(len(x[7]) for x in g["transfers"])


# ---- solver primitives through the C ABI (no device needed) ----
def test_choose_p_spec_examples():
    """SPEC.md choose_p examples (I=0 -> p=0.5, I=8 -> 0.25, I=24 & k_max=4 -> 0.25),
    GrainTooSmall, and snapping down to a divisor grid."""
    lib = load_library()
    assert lib.hesp_choose_p(0.0, 1024, 64, 8) == 0.5
    assert lib.hesp_choose_p(8.0, 1024, 64, 8) == 0.25
    assert lib.hesp_choose_p(24.0, 1024, 64, 4) == 0.25
    assert lib.hesp_choose_p(0.0, 100, 64, 8) == 0.0          # d < 2*min_block
    assert lib.hesp_choose_p(15.0, 768, 64, 8) == 1.0 / 4     # k = 5 -> snapped to 4 (768 % 5 != 0)
    assert lib.hesp_choose_p(48.0, 768, 64, 8) == 1.0 / 8     # k = 8, 768/8 = 96


def test_select_candidate_hard_and_soft_law():
    """SPEC.md select_candidate: Hard = max score, first on ties; Soft draws
    follow score / sum within +-0.01 over 1e5 draws (acceptance criterion 12)."""
    import ctypes as C
    lib = load_library()
    st = C.c_uint64(7)
    sc = np.array([1.0, 3.0, 3.0, 0.5])
    assert lib.hesp_select_candidate(sc.ctypes.data, 4, 0, C.byref(st)) == 1
    assert st.value == 7  # Hard draws nothing
    sc = np.array([3.0, 1.0])
    counts = np.zeros(2)
    for _ in range(100_000):
        counts[lib.hesp_select_candidate(sc.ctypes.data, 2, 1, C.byref(st))] += 1
    assert abs(counts[0] / 1e5 - 0.75) < 0.01
    assert lib.hesp_select_candidate(sc.ctypes.data, 0, 1, C.byref(st)) == -1


def test_reference_merge_round_trip_in_goldens():
    """SPEC acceptance 3 on the reference itself: partition then merge is the
    original graph -- the golden record of [(18, 2), merge 1] equals the base
    tiling's, hashes included."""
    a = read_golden("explicit_merge_c2")[0]
    b = read_golden("explicit_c2")[0]
    assert a.tobytes()[8:] == b.tobytes()[8:]


# ---- C++ fixture loaders ----
@pytest.mark.parametrize("plat,model", [("platform_cpugpu.json", "model_cpugpu.json"),
                                        ("platform_cpugpu_evict.json", "model_cpugpu.json"),
                                        ("platform_cpugpu.json", "model_cpugpu_table.csv"),
                                        ("platform_biglittle.json", "model_biglittle.json"),
                                        ("platform_serial.json", "model_biglittle.json")])
def test_cpp_loaders_match_python_parse(plat, model):
    """hesp_fixture_load reads every fixture to exactly the structs the Python
    parser (the one every golden test runs on) builds."""
    from paper_1602_05510_b200.engine import load_model, load_platform
    lib = load_library()
    fx = lib.hesp_fixture_load(os.path.join(FIXTURES, plat).encode(), os.path.join(FIXTURES, model).encode())
    assert fx, lib.hesp_last_error()
    try:
        pc = lib.hesp_fixture_platform(fx).contents
        mc = lib.hesp_fixture_model(fx).contents
        pp = load_platform(plat)
        keep = []
        ref = pp._c(keep)
        rm = load_model(model)._c(pp, keep)
        assert (pc.n_spaces, pc.n_types, pc.n_procs, pc.n_links) == (ref.n_spaces, ref.n_types, ref.n_procs,
                                                                     ref.n_links)
        def fields(x):  # field values (struct padding is unspecified)
            return tuple(getattr(x, f[0]) for f in x._fields_)
        for i in range(pc.n_spaces):
            assert fields(pc.spaces[i]) == fields(ref.spaces[i])
        for i in range(pc.n_types):
            assert pc.type_names[i] == ref.type_names[i]
        for i in range(pc.n_procs):
            assert fields(pc.procs[i]) == fields(ref.procs[i])
        for i in range(pc.n_links):
            assert fields(pc.links[i]) == fields(ref.links[i])
        assert (mc.variant, mc.n_entries, mc.n_rows) == (rm.variant, rm.n_entries, rm.n_rows)
        for i in range(mc.n_entries):
            assert fields(mc.entries[i]) == fields(rm.entries[i])
        for i in range(mc.n_rows):
            assert fields(mc.rows[i]) == fields(rm.rows[i])
    finally:
        lib.hesp_fixture_free(fx)


def test_cpp_loader_errors(tmp_path):
    lib = load_library()
    bad = tmp_path / "bad.json"
    bad.write_text('{"spaces": [ {"id": 0, "capacity_bytes": 1} ], "types": [], "processors": [{"id":0,"type":"x","space":0}]}')
    assert not lib.hesp_fixture_load(str(bad).encode(), os.path.join(FIXTURES, "model_cpugpu.json").encode())
    assert b"unknown type" in lib.hesp_last_error()
    bad.write_text('{"spaces": [')
    assert not lib.hesp_fixture_load(str(bad).encode(), os.path.join(FIXTURES, "model_cpugpu.json").encode())
    assert b"platform document" in lib.hesp_last_error()
    csv = tmp_path / "m.csv"
    csv.write_text("kind,proc_type,b,seconds\nGEMM,cpu,0,1.0\n")
    assert not lib.hesp_fixture_load(os.path.join(FIXTURES, "platform_cpugpu.json").encode(), str(csv).encode())
    assert b"b must be >= 1" in lib.hesp_last_error()
