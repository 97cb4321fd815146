"""hesp_min_reduce (K3, the C-ABI cross-GPU winner) with TWO ranks on a
one-GPU lease: two processes share cuda:0 and exchange through an
ncclAllReduce shim (tests/nccl_shim.c, loaded via HESP_NCCL_LIB) that keeps
NCCL's calling convention.  Checks the two-round exact argmin (min makespan
key, then the lowest index among the ranks holding it) and the summed
counters against the reference goldens of the same candidate range."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from golden_io import read_golden

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("shim") / "libnccl_shim.so")
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include", os.path.join(HERE, "nccl_shim.c"),
                    "-L/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", out], check=True)
    return out


def _run(shim, tmp_path, ranges):
    d = str(tmp_path)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "helpers", "min_reduce_worker.py"), str(r),
                               str(len(ranges)), shim, d, str(a), str(n)], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r, (a, n) in enumerate(ranges)]
    res = []
    for pr in procs:
        out, err = pr.communicate(timeout=600)
        assert pr.returncode == 0, err[-3000:]
        res.append(json.loads(out.strip().splitlines()[-1]))
    return res


def _golden_best(g):
    ok = g[g["status"] == 0]
    m = ok["makespan"].min()
    return float(m), int(ok[ok["makespan"] == m]["index"].min()), len(ok)


def test_two_ranks_disjoint_shards(lib, shim, tmp_path):
    g = read_golden("c2")  # 160 candidates, reference records
    res = _run(shim, tmp_path, [(0, 80), (80, 80)])
    mk, idx, n_ok = _golden_best(g)
    for r in res:
        assert r["global"]["makespan"] == mk and r["global"]["index"] == idx
        assert r["global"]["n_ok"] == n_ok and r["global"]["n_evaluated"] == 160
        assert r["global"]["sum_leaves"] == sum(x["local"]["sum_leaves"] for x in res)
        assert r["shim_calls"] == 3 and r["min_reduces"] == 1  # key MIN, index MIN, counters SUM
    # the winner came from exactly one rank's shard
    assert sum(r["local"]["index"] == idx for r in res) == 1


def test_two_ranks_tied_makespan_takes_lowest_index(lib, shim, tmp_path):
    """Both ranks evaluate the same range: both hold the global key, so round 2
    must still return one index (the lowest), with the counters of both."""
    res = _run(shim, tmp_path, [(0, 160), (0, 160)])
    mk, idx, _ = _golden_best(read_golden("c2"))
    assert all(r["global"]["index"] == idx and r["global"]["makespan"] == mk for r in res)
    assert all(r["global"]["n_evaluated"] == 320 for r in res)


def test_two_ranks_one_without_valid_candidates(lib, shim, tmp_path):
    """A rank whose shard has no valid schedule contributes NONE keys."""
    g = read_golden("c2")
    bad = [int(i) for i in g[g["status"] != 0]["index"]]
    first_bad = bad[0]
    assert g[g["index"] == first_bad]["status"][0] != 0
    res = _run(shim, tmp_path, [(first_bad, 1), (0, 160)])
    mk, idx, _ = _golden_best(g)
    assert res[0]["local"]["index"] == -1
    assert all(r["global"]["index"] == idx and r["global"]["makespan"] == mk for r in res)
