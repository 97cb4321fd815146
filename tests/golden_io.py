"""Reader for tests/golden/*.bin (written by oracle/ref_harness)."""
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RECORD = np.dtype([("index", "<u8"), ("status", "<i4"), ("n_leaves", "<i4"), ("makespan", "<f8"),
                   ("assign_hash", "<u8"), ("xfer_hash", "<u8")])


def read_golden(path_or_name):
    path = path_or_name if os.path.sep in path_or_name else os.path.join(GOLDEN_DIR, path_or_name + ".bin")
    with open(path, "rb") as f:
        magic = f.read(8)
        assert magic == b"HESPGLD1", magic
        n = int(np.frombuffer(f.read(8), "<u8")[0])
        rec = np.frombuffer(f.read(n * RECORD.itemsize), RECORD)
    assert len(rec) == n
    return np.sort(rec, order="index")


def compare(outcomes, golden, first=0):
    """Return list of mismatch strings between engine outcomes and golden records."""
    bad = []
    for g in golden:
        k = int(g["index"]) - first
        o = outcomes[k]
        same = (int(o["status"]) == int(g["status"]) and int(o["n_leaves"]) == int(g["n_leaves"])
                and np.float64(o["makespan"]).view("<u8") == np.float64(g["makespan"]).view("<u8")
                and int(o["assign_hash"]) == int(g["assign_hash"]) and int(o["xfer_hash"]) == int(g["xfer_hash"]))
        if not same:
            bad.append(f"cand {int(g['index'])}: engine {tuple(o.tolist())} ref {tuple(g.tolist())}")
    return bad
