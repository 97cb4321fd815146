"""Readers for the full-trace goldens (tests/golden/trace_*.json.gz, shift_*.json),
written by tests/golden/make_golden.py from oracle/_ref/ref_harness --trace."""
import glob
import gzip
import json
import os

import numpy as np

from golden_io import GOLDEN_DIR

TRACE_NAMES = sorted(os.path.basename(p)[len("trace_"):-len(".json.gz")]
                     for p in glob.glob(os.path.join(GOLDEN_DIR, "trace_*.json.gz")))
SHIFT_NAMES = sorted(os.path.basename(p)[len("shift_"):-len(".json")]
                     for p in glob.glob(os.path.join(GOLDEN_DIR, "shift_*.json")))


def read_trace(name):
    with gzip.open(os.path.join(GOLDEN_DIR, f"trace_{name}.json.gz"), "rt") as f:
        return json.load(f)


def read_shift(name):
    with open(os.path.join(GOLDEN_DIR, f"shift_{name}.json")) as f:
        return json.load(f)


def hbits(x) -> str:
    """16-hex-digit IEEE bit pattern of a double (the goldens' float encoding)."""
    return f"{int(np.float64(x).view('<u8')):016x}"


def fbits(h: str) -> float:
    return float(np.uint64(int(h, 16)).view("<f8"))
