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
    buf = torch.empty(n * 136, dtype=torch.uint8, device="cuda")
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
