"""Regenerate the golden fixtures from the UNMODIFIED reference.

Runs oracle/_ref/ref_harness (built by `make -C oracle` from the reference
sources under /root/reference/proj/src) for every preset in
paper_1602_05510_b200.configs.PARITY and writes tests/golden/<name>.bin:
8-byte magic "HESPGLD1", uint64 count, then count 40-byte records
(index u64, status i32, n_leaves i32, makespan f64, assign_hash u64,
xfer_hash u64).  The hashes fold every Assignment / TransferRec of the
reference SimResult (include/hesp_workload.h), so a record pins the whole
schedule bit-for-bit.

Usage: python tests/golden/make_golden.py [name ...]   (needs /root/reference)
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1602_05510_b200.configs import PARITY, harness_args  # noqa: E402
from paper_1602_05510_b200.engine import FIXTURES  # noqa: E402

HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")


def main(names):
    if not os.path.exists(HARNESS):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
    for name in names or sorted(PARITY):
        p, count = PARITY[name]
        out = os.path.join(HERE, f"{name}.bin")
        cmd = [HARNESS, *harness_args(p, FIXTURES), "--first", "0", "--count", str(count),
               "--threads", str(os.cpu_count()), "--out", out]
        r = subprocess.run(cmd, check=True, capture_output=True, text=True)
        print(name, r.stdout.strip())


if __name__ == "__main__":
    main(sys.argv[1:])
