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

from paper_1602_05510_b200.configs import PARITY, SCALE, harness_args  # noqa: E402
from paper_1602_05510_b200.engine import FIXTURES  # noqa: E402

HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")

# Hand-built candidates on the C2 base tiling (n=16384, 16x16 tiles of 1024; base
# task ids 1..816 in CHOL loop order: 1 CHOL(0,0), 2..16 TRSM(i,0), 17 SYRK(1,0),
# 18 GEMM(2,1,0), ...).  Statuses cover the reference's partition_task errors
# (graph.cpp:457-481): NotALeaf, Validation (unknown id, p not in (0,1)),
# IndivisibleGrain; plus tile-count snapping, a 16-way split, a 5-deep chain,
# 16 ops, and every kind partitioned.
EXPLICIT_OPS = [
    [],                                             # base tiling only
    [(0, 2)],                                       # root already partitioned -> NotALeaf
    [(5000, 2)],                                    # no such task -> Validation
    [(1, 1)],                                       # p = 1 -> Validation
    [(1, 0)],                                       # p = inf -> Validation
    [(1, -2)],                                      # p < 0 -> Validation
    [(1, 3)],                                       # snaps to 2
    [(1, 5)],                                       # snaps to 4
    [(1, 16)],                                      # 816-task sub-Cholesky of 64-tiles
    [(1, 1000)],                                    # snaps to 16
    [(1, 2), (817, 2), (821, 2), (825, 2), (829, 2)],  # 1024->512->256->128->64 -> IndivisibleGrain
    [(1, 2), (817, 2), (821, 2), (825, 2)],         # deepest valid chain (depth 5)
    [(2, 2), (2, 2)],                               # second split of the same task -> NotALeaf
    [(t, 2) for t in range(1, 17)],                 # 16 ops
    [(18, 4), (17, 2), (2, 4), (1, 2)],             # GEMM, SYRK, TRSM, CHOL
    [(18, 4), (818, 2), (900, 2), (17, 4)],          # sub-tasks of sub-tasks, mixed sides
]
# n=6144 base (8x8 tiles of 768): mixing s=3 (256) and s=2 (384) on overlapping
# operands creates intersection descriptors (graph.cpp:197-210).
SECT_OPS = [
    [(1, 3), (2, 2)],
    [(2, 2), (1, 3), (3, 3)],
    [(1, 2), (2, 3), (9, 3), (10, 2)],
    [(1, 3), (2, 2), (4, 3), (5, 2), (9, 2)],
]
# merge_cluster / repartition on the C2 base (cluster ids follow partition
# order, base = 0): ("m", c) merges cluster c.  Base task 18 = GEMM(2,1,0),
# 17 = SYRK(1,0), 2 = TRSM(1,0); a s=2 split of a CHOL/TRSM/SYRK/GEMM base
# task makes 4/6/6/8 members starting at id 817.
MERGE_OPS = [
    [(18, 2), ("m", 1)],                            # partition then merge: back to the base tiling
    [(18, 2), ("m", 1), (18, 4)],                   # repartition_cluster(1, 1/4)
    [(18, 2), ("m", 1), (18, 2)],                   # re-partition to the same s: fresh ids
    [(18, 2), (817, 2), ("m", 1)],                  # member partitioned -> NestedCluster
    [(18, 2), (817, 2), ("m", 2), ("m", 1)],        # innermost first, then the parent cluster
    [("m", 1)],                                     # no such cluster -> UnknownCluster
    [(18, 2), ("m", 1), ("m", 1)],                  # merged twice -> UnknownCluster
    [(18, 2), ("m", 1), (817, 2)],                  # partition a merged-away task -> Validation
    [(1, 2), (2, 2), (17, 4), ("m", 2), (18, 2), ("m", 1)],  # interleaved, shared blocks survive
    [(2, 4), (17, 2), ("m", 1), (3, 2), ("m", 3), (2, 2)],
]
# Merging the base cluster (cluster 0, graph.cpp:521-534) returns the graph to
# the unpartitioned root; ids stay consumed, so a later partition of the root
# (ids from 817 on C2) puts the candidate on another top-level tiling.  Ext.
# cluster ids keep counting as well (the first cluster after the merge is 1).
BASEMERGE_OPS = [
    [("m", 0)],                                     # the unpartitioned root: one CHOL(16384)
    [("m", 0), (0, 8)],                             # 8x8 tiling, tasks 817..936
    [("m", 0), (0, 16)],                            # the base tiling again, ids shifted by 816
    [("m", 0), (0, 4), (817, 2)],                   # 4x4 tiling, its first CHOL split
    [("m", 0), (0, 8), ("m", 1)],                   # back to the root
    [("m", 0), (0, 8), ("m", 1), (0, 4)],           # and onto a third tiling
    [(18, 2), ("m", 0)],                            # base member partitioned -> NestedCluster
    [(18, 2), ("m", 1), ("m", 0), (0, 8)],          # ids consumed by a merged cluster first
    [("m", 0), ("m", 0)],                           # merged twice -> UnknownCluster
    [("m", 0), (5, 2)],                             # partition an erased task -> Validation
    [("m", 0), (0, 2), (817, 2), (818, 2)],         # 2x2 tiling, CHOL and TRSM split
    [("m", 0), (0, 3)],                             # snaps to 2
    [("m", 0), (0, 16), (834, 4), (820, 2)],        # base tiling shifted, GEMM(2,1,0) and TRSM split
    [("m", 0), (0, 8), (820, 2), ("m", 1)],         # top cluster with a partitioned member -> NestedCluster
    [("m", 0), (0, 8), (820, 2), ("m", 2), ("m", 1), (0, 16), (1000, 2)],  # inner, top, re-tile, split
    [(1, 2), (17, 4), ("m", 2), ("m", 1), ("m", 0), (0, 4), (0, 2)],  # root partitioned again -> NotALeaf
]
EXPLICIT = {
    "explicit_basemerge_c2": ("c2", BASEMERGE_OPS),
    "explicit_basemerge_evict": ("evict_wb", BASEMERGE_OPS),
    "explicit_merge_c2": ("c2", MERGE_OPS),
    "explicit_c2": ("c2", EXPLICIT_OPS),
    "explicit_c3": ("c3", EXPLICIT_OPS),
    "explicit_sect": ("sect_cpugpu", SECT_OPS),
}
# (preset, candidate index, explicit descs file or None)
DETAIL = {
    "detail_c2_1": ("c2", 1, None),
    "detail_explicit_c2_14": ("c2", 14, "explicit_c2"),
    "detail_evict_wb_0": ("evict_wb", 0, None),
}

# Full SimResult traces (hesp_eval_trace parity):
# name -> (preset, candidate index).  Chosen to cover transfers over two-hop
# routes, gather fragments (sect_cpugpu 0, policy WA 10), eviction with the
# reference's own capacity violations (evict_*), write-through/around, R-P,
# single-space platforms and a tabulated model.
TRACES = {
    "c1_0": ("c1", 0), "c2_1": ("c2", 1), "c3_2": ("c3", 2), "table_1": ("table", 1),
    "evict_wb_0": ("evict_wb", 0), "evict_wt_1": ("evict_wt", 1), "evict_wa_0": ("evict_wa", 0),
    "sect_cpugpu_0": ("sect_cpugpu", 0), "deep_biglittle_1": ("deep_biglittle", 1),
    "policy_PL_EFT-P_WA_10": ("policy_PL_EFT-P_WA", 10), "policy_FCFS_R-P_WT_5": ("policy_FCFS_R-P_WT", 5),
    # explicit descriptors (preset, index, descs): candidates after a merge of the base cluster
    "basemerge_c2_12": ("c2", 12, "explicit_basemerge_c2"),
    "basemerge_c2_3": ("c2", 3, "explicit_basemerge_c2"),   # 4x4 top tiling: tiles span base tiles
    "basemerge_c2_0": ("c2", 0, "explicit_basemerge_c2"),   # the bare root as the only task
    "basemerge_evict_12": ("evict_wb", 12, "explicit_basemerge_evict"),
    # 32x32 tiles (~6.2k tasks): the load post-pass sorts ~12k events (128 KB of keys in shared memory)
    "c4_0": ("c4", 0),
}
# verify_schedule on edited schedules: (trace, task to move, seconds earlier)
SHIFTS = {
    "c2_1_early": ("c2_1", 400, 0.02),
    "c2_1_late": ("c2_1", 400, -0.02),
    "evict_wb_0_early": ("evict_wb_0", 30, 0.005),
    "sect_cpugpu_0_late": ("sect_cpugpu_0", 20, -0.01),
    "basemerge_c2_3_early": ("basemerge_c2_3", 10, 0.05),
}

# SPEC solver runs (hesp_solve parity): name -> (preset, iterations, selection, sampling, seed)
SOLVES = {
    "small_all_hard": ("policy_PL_EFT-P_WB", 12, "All", "Hard", 0),
    "small_cp_soft": ("policy_PL_EFT-P_WB", 12, "CP", "Soft", 3),
    "small_shallow_soft": ("policy_PL_EFT-P_WB", 12, "Shallow", "Soft", 5),
    "small_rp_all_soft": ("policy_FCFS_R-P_WB", 10, "All", "Soft", 9),
    "c2_all_soft": ("c2", 5, "All", "Soft", 1),
    # long horizon: parity up to the op budget of the chain state
    "small_all_soft_long": ("policy_PL_EFT-P_WB", 120, "All", "Soft", 2),
    "small_all_hard_long": ("policy_PL_EFT-P_WB", 90, "All", "Hard", 4),
}


def write_solves(names):
    import json
    for name, (preset_name, iters, sel, samp, seed) in SOLVES.items():
        if names and f"solve_{name}" not in names:
            continue
        p, _ = PARITY[preset_name]
        r = subprocess.run([HARNESS, *harness_args(p, FIXTURES), "--threads", str(os.cpu_count()), "--solve",
                            str(iters), "--solve-selection", sel, "--solve-sampling", samp, "--solve-seed",
                            str(seed)], check=True, capture_output=True, text=True)
        d = json.loads(r.stdout)
        d.update(preset=preset_name, iterations=iters, selection=sel, sampling=samp, seed=seed, k_max=8,
                 overhead=1.1)
        with open(os.path.join(HERE, f"solve_{name}.json"), "w") as f:
            json.dump(d, f)
        print("solve", name, [h[1] for h in d["history"]], "best it", d["best_iteration"])


def write_traces(names):
    import gzip
    import json
    for name, (preset_name, idx, *descs) in TRACES.items():
        if names and f"trace_{name}" not in names:
            continue
        p, _ = PARITY[preset_name]
        extra = ["--descs", os.path.join(HERE, f"{descs[0]}.descs")] if descs else []
        r = subprocess.run([HARNESS, *harness_args(p, FIXTURES), *extra, "--trace", str(idx)], check=True,
                           capture_output=True, text=True)
        d = json.loads(r.stdout)
        d["preset"] = preset_name
        if descs:
            d["descs"] = descs[0]
        with gzip.open(os.path.join(HERE, f"trace_{name}.json.gz"), "wt") as f:
            json.dump(d, f, separators=(",", ":"))
        print("trace", name, len(d["assignments"]), "tasks", len(d["transfers"]), "transfers")
    for name, (tname, task_rank, by) in SHIFTS.items():
        if names and f"shift_{name}" not in names:
            continue
        preset_name, idx, *descs = TRACES[tname]
        p, _ = PARITY[preset_name]
        extra = ["--descs", os.path.join(HERE, f"{descs[0]}.descs")] if descs else []
        base = json.loads(subprocess.run([HARNESS, *harness_args(p, FIXTURES), *extra, "--trace", str(idx)], check=True,
                                         capture_output=True, text=True).stdout)
        task = base["assignments"][task_rank][0]
        r = subprocess.run([HARNESS, *harness_args(p, FIXTURES), *extra, "--trace", str(idx), "--shift-task", str(task),
                            "--shift-by", repr(by)], check=True, capture_output=True, text=True)
        d = json.loads(r.stdout)
        out = {"trace": tname, "task": task, "shift_by": by, "violations": d["violations"]}
        with open(os.path.join(HERE, f"shift_{name}.json"), "w") as f:
            json.dump(out, f, indent=0)
        print("shift", name, len(d["violations"]), "violations")


def write_descs(path, ops_lists):
    import numpy as np
    from paper_1602_05510_b200.engine import DESC_DTYPE, MAX_OPS, OP_MERGE
    d = np.zeros(len(ops_lists), DESC_DTYPE)
    d["ops"][:] = -1
    d["ops"][:, :, 1] = 0
    for i, ops in enumerate(ops_lists):
        d[i]["n_ops"] = len(ops)
        for k, (t, s) in enumerate(ops):
            if t == "m":  # merge_cluster(s)
                d[i]["ops"][k] = (s, OP_MERGE)
            else:
                d[i]["ops"][k] = (t, s)
    d.tofile(path)


def main(names):
    if not os.path.exists(HARNESS):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
    # explicit descriptors: error paths and edge cases the generator never emits
    for name, (preset_name, ops_lists) in EXPLICIT.items():
        if names and name not in names:
            continue
        p, _ = PARITY[preset_name]
        dpath = os.path.join(HERE, f"{name}.descs")
        write_descs(dpath, ops_lists)
        out = os.path.join(HERE, f"{name}.bin")
        r = subprocess.run([HARNESS, *harness_args(p, FIXTURES), "--descs", dpath, "--threads",
                            str(os.cpu_count()), "--out", out], check=True, capture_output=True, text=True)
        print(name, r.stdout.strip())
    # per-task schedules of a few candidates (hesp_eval_detail parity)
    for name, (preset_name, idx, descs_name) in DETAIL.items():
        if names and name not in names:
            continue
        p, _ = PARITY[preset_name]
        args = [HARNESS, *harness_args(p, FIXTURES), "--detail", str(idx), "--detail-out",
                os.path.join(HERE, f"{name}.txt")]
        if descs_name:
            args += ["--descs", os.path.join(HERE, f"{descs_name}.descs")]
        subprocess.run(args, check=True)
        path = os.path.join(HERE, f"{name}.txt")
        keep = [l for l in open(path) if l.startswith(("index", "ops", "A "))]
        with open(path, "w") as f:
            f.writelines(keep)
        print(name, "detail written")
    write_traces(names)
    write_solves(names)
    records = {**PARITY, **SCALE}
    for name in [n for n in (names or sorted(records)) if n in records]:
        p, count = records[name]
        out = os.path.join(HERE, f"{name}.bin")
        cmd = [HARNESS, *harness_args(p, FIXTURES), "--first", "0", "--count", str(count),
               "--threads", str(os.cpu_count()), "--out", out]
        r = subprocess.run(cmd, check=True, capture_output=True, text=True)
        print(name, r.stdout.strip())


if __name__ == "__main__":
    main(sys.argv[1:])
