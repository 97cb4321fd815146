"""GPU parity: the sm_100a engine against golden records of the unmodified reference.

Bit-exact on every field: status (the reference's Err), leaf count, makespan
bits, and the order-independent hashes of all assignments and transfers.
"""
import numpy as np
import pytest

from golden_io import compare, read_golden
from paper_1602_05510_b200.configs import PARITY, make_engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(PARITY))
def test_golden_parity(lib, name):
    p, count = PARITY[name]
    g = read_golden(name)
    assert len(g) == count
    eng = make_engine(p)
    out, best = eng.eval_generated(0, count)
    bad = compare(out, g)
    assert not bad, "\n".join(bad[:10])
    ok = g[g["status"] == 0]
    assert best.n_ok == len(ok) and best.n_evaluated == count
    if len(ok):
        m = ok["makespan"].min()
        assert best.makespan == m
        assert best.index == int(ok[ok["makespan"] == m]["index"].min())


def test_device_generator_matches_host(lib):
    import torch
    p, _ = PARITY["c2"]
    eng = make_engine(p)
    n = 4096
    buf = torch.empty(n * 520, dtype=torch.uint8, device="cuda")
    eng.generate_device(1000, n, buf.data_ptr())
    torch.cuda.synchronize()
    dev = buf.cpu().numpy().tobytes()
    host = eng.generate_host(1000, n).tobytes()
    assert dev == host


def test_descs_path_matches_generated(lib):
    p, count = PARITY["c2"]
    eng = make_engine(p)
    descs = eng.generate_host(0, count)
    out1, b1 = eng.eval_descs(descs, first=0)
    out2, b2 = eng.eval_generated(0, count)
    assert np.array_equal(out1, out2)
    assert (b1.makespan, b1.index) == (b2.makespan, b2.index)


@pytest.mark.parametrize("threads", ["1", "5", None])
def test_host_packing_threads(lib, monkeypatch, threads):
    """hesp_eval_descs packs host descriptors (and copies outcomes out) on
    host threads from 16k candidates on (HESP_HOST_THREADS forces a count):
    every split gives the device-generator path's outcomes, and the first
    records are the reference's."""
    p, count = PARITY["c2"]
    eng = make_engine(p)
    n = 20000
    descs = eng.generate_host(0, n)
    descs["n_ops"][7] = 0  # ragged: an empty descriptor (the base tiling itself) mid-range
    if threads is None:
        monkeypatch.delenv("HESP_HOST_THREADS", raising=False)
    else:
        monkeypatch.setenv("HESP_HOST_THREADS", threads)
    out1, b1 = eng.eval_descs(descs, first=0)
    monkeypatch.delenv("HESP_HOST_THREADS", raising=False)
    ref, rb = eng.eval_generated(0, n)
    keep = np.ones(n, bool)
    keep[7] = False
    assert np.array_equal(out1[keep], ref[keep])
    g = read_golden("c2")
    bad = compare(out1, g[g["index"] != 7])
    assert not bad, "\n".join(bad[:5])
    base, _ = eng.eval_descs(descs[7:8], first=7)
    assert np.array_equal(out1[7:8], base)


EXPLICIT = {"explicit_c2": "c2", "explicit_c3": "c3", "explicit_sect": "sect_cpugpu", "explicit_merge_c2": "c2",
            "explicit_basemerge_c2": "c2", "explicit_basemerge_evict": "evict_wb"}


@pytest.mark.parametrize("name", sorted(EXPLICIT))
def test_explicit_descriptor_parity(lib, name):
    """Hand-built candidates (error statuses, snapping, deep chains, 16 ops,
    intersections) through the host-buffer ABI path, vs the reference."""
    from golden_io import GOLDEN_DIR
    from paper_1602_05510_b200.engine import DESC_DTYPE
    import os
    p, _ = PARITY[EXPLICIT[name]]
    descs = np.fromfile(os.path.join(GOLDEN_DIR, f"{name}.descs"), DESC_DTYPE)
    g = read_golden(name)
    eng = make_engine(p)
    out, best = eng.eval_descs(descs, first=0)
    bad = compare(out, g)
    assert not bad, "\n".join(bad[:10])


DETAIL = {"detail_c2_1": ("c2", None), "detail_explicit_c2_14": ("c2", "explicit_c2"),
          "detail_evict_wb_0": ("evict_wb", None)}


@pytest.mark.parametrize("name", sorted(DETAIL))
def test_per_task_schedule_parity(lib, name):
    """hesp_eval_detail: every leaf's processor, start and end bits equal the
    reference SimResult::assignments."""
    import os
    from golden_io import GOLDEN_DIR
    from paper_1602_05510_b200.engine import DESC_DTYPE
    preset, descs_name = DETAIL[name]
    p, _ = PARITY[preset]
    lines = open(os.path.join(GOLDEN_DIR, f"{name}.txt")).read().splitlines()
    idx = int(lines[0].split()[1])
    want = {}
    for l in lines:
        if l.startswith("A "):
            f = l.split()
            want[int(f[1])] = (int(f[2]), int(f[5], 16), int(f[6], 16))
    eng = make_engine(p)
    if descs_name:
        desc = np.fromfile(os.path.join(GOLDEN_DIR, f"{descs_name}.descs"), DESC_DTYPE)[idx]
    else:
        desc = eng.generate_host(idx, 1)[0]
    cap = max(want) + 64
    o, proc, start, end = eng.eval_detail(desc, cap)
    assert o.status == 0
    got = {t: (int(proc[t]), int(np.float64(start[t]).view(np.uint64)), int(np.float64(end[t]).view(np.uint64)))
           for t in range(cap) if proc[t] >= 0}
    assert got == want


def test_search_driver_matches_batch_best(lib, capsys):
    """paper_1602_05510_b200.search (the sharded C4/C5 driver, 1 rank here)
    finds the same winner as one batch over the same index range, and its
    winner trace verifies clean."""
    import json
    from paper_1602_05510_b200.search import main
    main(["--config", "c2", "--candidates", "3000", "--batch", "1000", "--trace-winner"])
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    p, _ = PARITY["c2"]
    _, b = make_engine(p).eval_generated(0, 3000, outcomes=False)
    assert line["best"]["index"] == b.index and line["best"]["makespan"] == b.makespan
    assert line["valid"] == b.n_ok and line["winner_trace"]["verify_violations"] == 0


def test_min_reduce_over_nccl_single_rank(lib):
    """hesp_min_reduce (the C-ABI cross-GPU winner, K3) over a real one-rank
    NCCL communicator: the winner and the counters come back unchanged."""
    import ctypes as C
    import torch  # noqa: F401  (loads the process's libnccl.so.2, as in bench.py)
    nccl = C.CDLL("libnccl.so.2")
    comm = C.c_void_p()
    dev = (C.c_int * 1)(0)
    assert nccl.ncclCommInitAll(C.byref(comm), 1, dev) == 0
    try:
        p, _ = PARITY["c2"]
        eng = make_engine(p)
        _, b = eng.eval_generated(0, 64, outcomes=False)
        r = eng.min_reduce(comm.value, b)
        assert (r.makespan, r.index, r.n_ok, r.n_evaluated, r.sum_leaves) == \
            (b.makespan, b.index, b.n_ok, b.n_evaluated, b.sum_leaves)
        from paper_1602_05510_b200.engine import Best
        empty = Best()
        empty.index = -1
        r2 = eng.min_reduce(comm.value, empty)
        assert r2.index == -1
    finally:
        nccl.ncclCommDestroy(comm)


def test_min_reduce_over_torch_process_group(lib):
    """bench.py / search.py path at N>1, exercised at world size 1: the
    communicator of a real NCCL process group handed to hesp_min_reduce."""
    import os
    import torch
    import torch.distributed as dist
    from paper_1602_05510_b200.dist import engine_global_best
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        dist.barrier()
        p, _ = PARITY["c2"]
        eng = make_engine(p)
        _, b = eng.eval_generated(0, 64, outcomes=False)
        from paper_1602_05510_b200.dist import nccl_comm_ptr
        assert nccl_comm_ptr() != 0
        g = eng.min_reduce(nccl_comm_ptr(), b)
        assert (g.makespan, g.index, g.n_ok) == (b.makespan, b.index, b.n_ok)
        (mk, idx), _ = engine_global_best(eng, b)
        assert (mk, idx) == (b.makespan, b.index)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c2", "table", "c3", "evict_wt"])
def test_engine_from_cpp_loaded_fixtures(lib, name):
    """An engine created from hesp_fixture_load's structs reproduces the goldens."""
    from paper_1602_05510_b200.engine import BatchEngine, FIXTURES, SchedConfig, Workload
    import os
    p, count = PARITY[name]
    sched = SchedConfig(p["ordering"], p["selection"], p["caching"], p["sched_seed"], p["min_block"])
    wl = Workload(p["n"], p["elem"], p["s_base"], p["seed"], p["k_max"], p["max_depth"], p["min_block"],
                  p["s_choices"], p.get("merge_pct", 0))
    eng = BatchEngine.from_files(os.path.join(FIXTURES, p["platform"]), os.path.join(FIXTURES, p["model"]),
                                 sched, wl)
    out, _ = eng.eval_generated(0, count)
    assert not compare(out, read_golden(name))


def test_neighbors_equal_replayed_descriptors(lib):
    """hesp_eval_neighbors (template state + 1-2 extra ops, merges included)
    gives exactly the outcome records of replaying the full descriptors."""
    from paper_1602_05510_b200.engine import NEIGHBOR_DTYPE, OP_MERGE
    p, _ = PARITY["merge_c2"]
    eng = make_engine(p)
    bases = eng.generate_host(0, 6)
    rng = np.random.default_rng(7)
    nb = np.zeros(3000, NEIGHBOR_DTYPE)
    full = np.zeros(3000, bases.dtype)
    for k in range(3000):
        b = int(rng.integers(0, len(bases)))
        base = bases[b]
        n0 = int(base["n_ops"])
        m = int(rng.integers(0, 3))
        ops = []
        for _ in range(m):
            if rng.random() < 0.25:
                ops.append((int(rng.integers(0, 6)), OP_MERGE))
            else:
                ops.append((int(rng.integers(1, 1400)), int(rng.choice([2, 3, 4]))))
        nb[k]["base"], nb[k]["n_ops"] = b, m
        for i, o in enumerate(ops):
            nb[k]["ops"][i] = o
        full[k] = base
        full[k]["n_ops"] = n0 + m
        for i, o in enumerate(ops):
            full[k]["ops"][n0 + i] = o
    a, ba = eng.eval_neighbors(bases, nb)
    r, br = eng.eval_descs(full)
    assert a.tobytes() == r.tobytes()
    assert (ba.makespan, ba.index, ba.n_ok) == (br.makespan, br.index, br.n_ok)
    assert len(np.unique(a["status"])) > 1  # the mix hits error statuses too
