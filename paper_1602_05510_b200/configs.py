"""Workload presets: BASELINE.json's configs (C1..C5) and the parity fixtures.

Every preset names the fixture files the reference parses, the root/base
tiling, the candidate generator and the SchedConfig.  The oracle harness
(oracle/ref_harness), the GPU engine and bench.py all derive their inputs
from these dicts, so a preset means the same candidates everywhere.
"""
from __future__ import annotations

import itertools

CPUGPU = ("platform_cpugpu.json", "model_cpugpu.json")
CPUGPU_EVICT = ("platform_cpugpu_evict.json", "model_cpugpu.json")
CPUGPU_TABLE = ("platform_cpugpu.json", "model_cpugpu_table.csv")
BIGLITTLE = ("platform_biglittle.json", "model_biglittle.json")


def preset(fix, n, elem, s_base, k_max, max_depth=3, s_choices=(2, 4), seed=1,
           ordering="PL", selection="EFT-P", caching="WB", sched_seed=0, min_block=64, merge_pct=0):
    return dict(platform=fix[0], model=fix[1], n=n, elem=elem, s_base=s_base, k_max=k_max,
                max_depth=max_depth, s_choices=tuple(s_choices), seed=seed, ordering=ordering,
                selection=selection, caching=caching, sched_seed=sched_seed, min_block=min_block,
                merge_pct=merge_pct)


# BASELINE.json configs
C1 = preset(CPUGPU, 8192, 4, 8, 0)                        # 8x8 homogeneous, EFT, CPU-GPU
C2 = preset(CPUGPU, 16384, 4, 16, 8)                      # 1e5 random recursive partitionings of 16x16
C3 = preset(BIGLITTLE, 8192, 8, 16, 8)                    # big.LITTLE 4+4
C4 = preset(CPUGPU, 32768, 4, 32, 12)                     # 32x32, 3-level recursion, coherence
C5 = C2                                                    # 1e7 candidates of C2's shape over 8 GPUs

CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5}

# parity fixtures (tests/golden): name -> (preset, candidate count)
PARITY = {
    "c1": (C1, 1),
    "c2": (C2, 160),
    "c3": (C3, 96),
    "c4": (C4, 12),
    "evict_wb": (preset(CPUGPU_EVICT, 16384, 4, 16, 8, seed=3, caching="WB"), 32),
    "evict_wt": (preset(CPUGPU_EVICT, 16384, 4, 16, 8, seed=4, caching="WT"), 32),
    "evict_wa": (preset(CPUGPU_EVICT, 16384, 4, 16, 8, seed=5, caching="WA", ordering="FCFS",
                        selection="EIT-P"), 32),
    "table": (preset(CPUGPU_TABLE, 16384, 4, 16, 8, seed=6), 40),
    "sect_cpugpu": (preset(CPUGPU, 6144, 4, 8, 8, s_choices=(2, 3, 4), seed=8), 48),
    "sect_biglittle": (preset(BIGLITTLE, 6144, 8, 8, 8, s_choices=(2, 3, 4), seed=9, ordering="FCFS",
                              selection="F-P"), 48),
    "deep_biglittle": (preset(BIGLITTLE, 8192, 8, 8, 12, max_depth=4, seed=12, selection="R-P",
                              sched_seed=77), 48),
}
SERIAL = ("platform_serial.json", "model_biglittle.json")  # one big core: SPEC acceptance 6
PARITY["serial"] = (preset(SERIAL, 4096, 8, 8, 8, seed=31, merge_pct=20), 24)

# merge ops (TaskGraph::merge_cluster) mixed into the random partitionings
PARITY["merge_c2"] = (preset(CPUGPU, 16384, 4, 16, 12, seed=21, merge_pct=35), 64)
PARITY["merge_evict"] = (preset(CPUGPU_EVICT, 16384, 4, 16, 10, seed=22, merge_pct=30), 24)
PARITY["merge_c3"] = (preset(BIGLITTLE, 8192, 8, 16, 10, seed=23, merge_pct=40, ordering="FCFS",
                             selection="F-P"), 32)
# merges on non-nested tilings: merge_cluster while intersection descriptors live (graph.cpp:214-266)
PARITY["merge_sect"] = (preset(CPUGPU, 6144, 4, 8, 10, s_choices=(2, 3, 4), seed=41, merge_pct=35), 96)
PARITY["merge_sect_bl"] = (preset(BIGLITTLE, 6144, 8, 8, 10, s_choices=(2, 3, 4), seed=42, merge_pct=40,
                                  ordering="FCFS", selection="EIT-P"), 64)
for o, s, c in itertools.product(("FCFS", "PL"), ("R-P", "F-P", "EIT-P", "EFT-P"), ("WT", "WB", "WA")):
    PARITY[f"policy_{o}_{s}_{c}"] = (preset(CPUGPU, 4096, 4, 8, 8, seed=7, ordering=o, selection=s, caching=c,
                                            sched_seed=5), 24)


# At-scale parity (VERDICT r1 "next" #1, SURVEY.md §7 minimum slice >= 1e4):
# the same generators over many more candidate indices, every record compared
# bit for bit on the GPU (tests/test_scale_gpu.py).  Sizes follow §8(d)'s
# sample sizes: 1e4 for C2/C3, 256 for C4, 1e3 per eviction fixture.
SCALE = {
    "scale_c2": (C2, 10_000),
    "scale_c3": (C3, 10_000),
    "scale_c4": (C4, 256),
    "scale_evict_wb": (PARITY["evict_wb"][0], 1000),
    "scale_evict_wt": (PARITY["evict_wt"][0], 1000),
    "scale_evict_wa": (PARITY["evict_wa"][0], 1000),
    "scale_merge_c2": (PARITY["merge_c2"][0], 2000),
    "scale_sect_cpugpu": (PARITY["sect_cpugpu"][0], 2000),
    "scale_merge_sect": (PARITY["merge_sect"][0], 2000),
}


def harness_args(p: dict, fixtures_dir: str) -> list[str]:
    """oracle/_ref/ref_harness arguments for preset p."""
    import os
    model = os.path.join(fixtures_dir, p["model"])
    return ["--platform", os.path.join(fixtures_dir, p["platform"]),
            "--model-csv" if p["model"].endswith(".csv") else "--model", model,
            "--n", str(p["n"]), "--elem", str(p["elem"]), "--sbase", str(p["s_base"]),
            "--seed", str(p["seed"]), "--kmax", str(p["k_max"]), "--maxdepth", str(p["max_depth"]),
            "--min-block", str(p["min_block"]), "--s-choices", ",".join(map(str, p["s_choices"])),
            "--ordering", p["ordering"], "--selection", p["selection"], "--caching", p["caching"],
            "--sched-seed", str(p["sched_seed"]), "--merge-pct", str(p.get("merge_pct", 0))]


def make_engine(p: dict, device: int = 0):
    """BatchEngine for preset p on one GPU."""
    from .engine import BatchEngine, SchedConfig, Workload, load_model, load_platform
    plat = load_platform(p["platform"])
    model = load_model(p["model"])
    sched = SchedConfig(p["ordering"], p["selection"], p["caching"], p["sched_seed"], p["min_block"])
    wl = Workload(p["n"], p["elem"], p["s_base"], p["seed"], p["k_max"], p["max_depth"], p["min_block"],
                  p["s_choices"], p.get("merge_pct", 0))
    return BatchEngine(plat, model, sched, wl, device)
