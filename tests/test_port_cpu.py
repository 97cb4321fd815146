"""The CPU restatement (oracle/port) pinned to the golden records of the
unmodified reference: bit-identical status, leaves, makespan and schedule /
transfer hashes."""
import os
import subprocess

import pytest

from golden_io import read_golden
from paper_1602_05510_b200.configs import PARITY, harness_args
from paper_1602_05510_b200.engine import FIXTURES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT = os.path.join(ROOT, "oracle", "_ref", "port_harness")

PRESETS = ["c1", "c2", "c3", "evict_wb", "evict_wt", "evict_wa", "table", "sect_cpugpu", "sect_biglittle",
           "deep_biglittle", "policy_FCFS_R-P_WA", "policy_PL_F-P_WT", "policy_FCFS_EIT-P_WB", "policy_PL_EFT-P_WA"]


@pytest.mark.skipif(not os.path.exists(PORT), reason="oracle/_ref/port_harness not built")
@pytest.mark.parametrize("name", PRESETS)
def test_port_matches_goldens(name, tmp_path):
    p, count = PARITY[name]
    k = min(count, 10)
    out = tmp_path / "port.bin"
    subprocess.run([PORT, *harness_args(p, FIXTURES), "--first", "0", "--count", str(k), "--threads",
                    str(os.cpu_count()), "--out", str(out)], check=True, capture_output=True, timeout=600)
    got = read_golden(str(out))
    want = read_golden(name)[:k]
    assert got.tobytes() == want.tobytes()


@pytest.mark.skipif(not os.path.exists(PORT), reason="oracle/_ref/port_harness not built")
@pytest.mark.parametrize("name,preset", [("explicit_c2", "c2"), ("explicit_c3", "c3"), ("explicit_sect", "sect_cpugpu")])
def test_port_matches_explicit_goldens(name, preset, tmp_path):
    from golden_io import GOLDEN_DIR
    p, _ = PARITY[preset]
    out = tmp_path / "port.bin"
    subprocess.run([PORT, *harness_args(p, FIXTURES), "--descs", os.path.join(GOLDEN_DIR, f"{name}.descs"),
                    "--threads", str(os.cpu_count()), "--out", str(out)], check=True, capture_output=True, timeout=600)
    assert read_golden(str(out)).tobytes() == read_golden(name).tobytes()
