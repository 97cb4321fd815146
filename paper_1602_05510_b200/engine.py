"""ctypes binding of the C ABI in include/hesp_engine.h.

Python-side plumbing for tests and bench.py: loads the in-tree sm_100a
library (there is no CPU fallback — a missing library or device raises),
builds the reference-shaped inputs from the same JSON/CSV fixtures the
reference parses (Platform::from_json, PerfModel::from_analytic_json /
from_table_csv: platform.cpp:157-338) and exposes batch evaluation.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from .build import LIB as _DEFAULT_LIB

LIB = os.environ.get("HESP_LIB", _DEFAULT_LIB)

KINDS = {"CHOL": 0, "TRSM": 1, "SYRK": 2, "GEMM": 3}
ORDERING = {"FCFS": 0, "PL": 1}
SELECTION = {"R-P": 0, "F-P": 1, "EIT-P": 2, "EFT-P": 3}
CACHING = {"WT": 0, "WB": 1, "WA": 2}

MAX_OPS = 64
OP_MERGE = -(1 << 31)  # hesp_op.s of a merge_cluster op (HESP_OP_MERGE)


class Space(C.Structure):
    _fields_ = [("id", C.c_int32), ("capacity_bytes", C.c_int64), ("is_main", C.c_int32)]


class Processor(C.Structure):
    _fields_ = [("id", C.c_int32), ("type", C.c_int32), ("space", C.c_int32)]


class Link(C.Structure):
    _fields_ = [("src", C.c_int32), ("dst", C.c_int32), ("latency_s", C.c_double),
                ("bandwidth_bps", C.c_double)]


class PlatformC(C.Structure):
    _fields_ = [("n_spaces", C.c_int32), ("spaces", C.POINTER(Space)),
                ("n_types", C.c_int32), ("type_names", C.POINTER(C.c_char_p)),
                ("n_procs", C.c_int32), ("procs", C.POINTER(Processor)),
                ("n_links", C.c_int32), ("links", C.POINTER(Link))]


class AnalyticEntry(C.Structure):
    _fields_ = [("kind", C.c_int32), ("type", C.c_int32), ("peak_flops", C.c_double),
                ("b_half", C.c_double)]


class TableRow(C.Structure):
    _fields_ = [("kind", C.c_int32), ("type", C.c_int32), ("b", C.c_int64), ("seconds", C.c_double)]


class PerfModelC(C.Structure):
    _fields_ = [("variant", C.c_int32), ("n_entries", C.c_int32),
                ("entries", C.POINTER(AnalyticEntry)), ("n_rows", C.c_int32),
                ("rows", C.POINTER(TableRow))]


class SchedConfigC(C.Structure):
    _fields_ = [("ordering", C.c_int32), ("selection", C.c_int32), ("caching", C.c_int32),
                ("reserved", C.c_int32), ("seed", C.c_uint64), ("min_block", C.c_int64)]


class GenConfig(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("k_max", C.c_int32), ("max_depth", C.c_int32),
                ("min_block", C.c_int64), ("n_s_choices", C.c_int32), ("s_choices", C.c_int32 * 4),
                ("merge_pct", C.c_int32)]


class WorkloadC(C.Structure):
    _fields_ = [("n", C.c_int64), ("elem_size", C.c_int32), ("s_base", C.c_int32), ("gen", GenConfig)]


class Op(C.Structure):
    _fields_ = [("task", C.c_int32), ("s", C.c_int32)]


class CandDesc(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("reserved", C.c_int32), ("ops", Op * MAX_OPS)]


class Outcome(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_leaves", C.c_int32), ("makespan", C.c_double),
                ("assign_hash", C.c_uint64), ("xfer_hash", C.c_uint64)]


class Best(C.Structure):
    _fields_ = [("makespan", C.c_double), ("index", C.c_int64), ("n_ok", C.c_int64),
                ("n_evaluated", C.c_int64), ("sum_leaves", C.c_int64), ("sum_k", C.c_int64),
                ("sum_edges", C.c_int64), ("kernel_ms", C.c_double), ("build_ms", C.c_double),
                ("sim_ms", C.c_double)]


class EngineInfo(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("n_base_tasks", C.c_int32),
                ("n_base_blocks", C.c_int32), ("n_slots", C.c_int32), ("sm_count", C.c_int32),
                ("slot_bytes", C.c_int64), ("warps_per_block", C.c_int32),
                ("blocks_per_sm", C.c_int32), ("chunk", C.c_int64), ("last_h2d_bytes", C.c_int64),
                ("min_reduces", C.c_int64)]


ASSIGN_DTYPE = np.dtype([("task", "<i4"), ("proc", "<i4"), ("start", "<f8"), ("end", "<f8"),
                         ("idle_avg", "<f8")])
XFER_DTYPE = np.dtype([("block", "<i4"), ("src_space", "<i4"), ("dst_space", "<i4"), ("n_hops", "<i4"),
                       ("bytes", "<i8"), ("start", "<f8"), ("end", "<f8"), ("has_fragment", "<i4"),
                       ("frag", "<i4", (4,)), ("pad", "<i4"), ("hop_src", "<i4", (2,)), ("hop_dst", "<i4", (2,)),
                       ("hop_start", "<f8", (2,)), ("hop_end", "<f8", (2,))])
RES_DTYPE = np.dtype([("time", "<f8"), ("space", "<i4"), ("block", "<i4"), ("delta_bytes", "<i8")])
EVENT_DTYPE = np.dtype([("kind", "<i4"), ("id", "<i4"), ("task_kind", "<i4"), ("res_a", "<i4"), ("res_b", "<i4"),
                        ("pad", "<i4"), ("b", "<i8"), ("time", "<f8")])
STEP_DTYPE = np.dtype([("time", "<f8"), ("active", "<i4"), ("pad", "<i4")])
EVENT_KINDS = ("TaskStart", "TaskEnd", "XferStart", "XferEnd")
KIND_NAMES = ("CHOL", "TRSM", "SYRK", "GEMM")


class SolverConfigC(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("task_selection", C.c_int32), ("sampling", C.c_int32),
                ("k_max", C.c_int32), ("seed", C.c_uint64), ("min_block", C.c_int64),
                ("overhead_factor", C.c_double)]


SOLVER_ITER_DTYPE = np.dtype([("iteration", "<i4"), ("action", "<i4"), ("target", "<i4"), ("n_candidates", "<i4"),
                              ("n_valid", "<i4"), ("dag_depth", "<i4"), ("d", "<i8"), ("p", "<f8"),
                              ("score", "<f8"), ("makespan", "<f8"), ("avg_block_side", "<f8"),
                              ("avg_load_pct", "<f8")])


class SolverResultC(C.Structure):
    _fields_ = [("cap_history", C.c_int32), ("n_history", C.c_int32), ("history", C.c_void_p),
                ("best", CandDesc), ("best_makespan", C.c_double), ("best_iteration", C.c_int32),
                ("budget_iteration", C.c_int32), ("n_simulated", C.c_int64)]


TASK_SELECTION = {"All": 0, "CP": 1, "Shallow": 2}
SAMPLING = {"Hard": 0, "Soft": 1, "Exact": 2}
ACTIONS = {-1: None, 0: "Partition", 1: "Merge", 2: "Repartition"}


class TraceC(C.Structure):
    _fields_ = [("cap_assign", C.c_int32), ("cap_xfer", C.c_int32), ("cap_res", C.c_int32),
                ("cap_events", C.c_int32), ("cap_steps", C.c_int32), ("flags", C.c_int32),
                ("assignments", C.c_void_p), ("transfers", C.c_void_p), ("residency", C.c_void_p),
                ("events", C.c_void_p), ("steps", C.c_void_p),
                ("n_assign", C.c_int32), ("n_xfer", C.c_int32), ("n_res", C.c_int32), ("n_events", C.c_int32),
                ("n_steps", C.c_int32), ("pad1", C.c_int32), ("outcome", Outcome),
                ("busy_time", C.c_double), ("avg_load", C.c_double), ("load_integral", C.c_double)]


@dataclass
class Trace:
    """hesp::SimResult of one candidate (+ compute_load_trace), from hesp_eval_trace."""
    status: int
    n_leaves: int
    makespan: float
    assignments: np.ndarray  # ASSIGN_DTYPE, task-id order
    transfers: np.ndarray    # XFER_DTYPE, SimResult::transfers order
    events: np.ndarray       # EVENT_DTYPE, SimResult::events order
    residency: np.ndarray    # RES_DTYPE, SimResult::residency_log order
    steps: np.ndarray        # STEP_DTYPE, LoadTrace::steps
    busy_time: float = 0.0
    avg_load: float = 0.0
    load_integral: float = 0.0

    def event_strings(self) -> list[tuple[str, float, str, str]]:
        """(kind, time, subject, resource) exactly as the reference's EventRec strings."""
        out = []
        for e in self.events:
            k = int(e["kind"])
            if k < 2:
                subj = f"T{int(e['id'])}:{KIND_NAMES[int(e['task_kind'])]}:b{int(e['b'])}"
                res = str(int(e["res_a"]))
            else:
                subj = f"B{int(e['id'])}"
                res = f"{int(e['res_a'])}->{int(e['res_b'])}"
            out.append((EVENT_KINDS[k], float(e["time"]), subj, res))
        return out


NEIGHBOR_DTYPE = np.dtype([("base", "<i4"), ("n_ops", "<i4"), ("ops", "<i4", (2, 2))])

OUTCOME_DTYPE = np.dtype([("status", "<i4"), ("n_leaves", "<i4"), ("makespan", "<f8"),
                          ("assign_hash", "<u8"), ("xfer_hash", "<u8")])
assert OUTCOME_DTYPE.itemsize == C.sizeof(Outcome) == 32
DESC_DTYPE = np.dtype([("n_ops", "<i4"), ("reserved", "<i4"), ("ops", "<i4", (MAX_OPS, 2))])
assert DESC_DTYPE.itemsize == C.sizeof(CandDesc) == 520

EXPORTS = [
    "hesp_engine_create", "hesp_eval_generated", "hesp_eval_descs", "hesp_eval_descs_device",
    "hesp_generate_device", "hesp_generate_host", "hesp_generate_batch", "hesp_eval_detail",
    "hesp_engine_get_info", "hesp_eval_trace", "hesp_verify_trace", "hesp_trace_bounds", "hesp_trace_blocks", "hesp_solve", "hesp_solve_batch", "hesp_eval_neighbors", "hesp_min_reduce", "hesp_choose_p", "hesp_select_candidate",
    "hesp_fixture_load", "hesp_fixture_platform", "hesp_fixture_model", "hesp_fixture_free",
    "hesp_engine_destroy", "hesp_last_error", "hesp_status_name",
]

_lib = None


def load_library(path: str = LIB) -> C.CDLL:
    """Load the in-tree engine library; raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"engine library {path} is missing: run __graft_entry__.build()")
    lib = C.CDLL(path)
    lib.hesp_engine_create.restype = C.c_void_p
    lib.hesp_engine_create.argtypes = [C.c_int, C.POINTER(PlatformC), C.POINTER(PerfModelC),
                                       C.POINTER(SchedConfigC), C.POINTER(WorkloadC)]
    lib.hesp_eval_generated.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.POINTER(Best)]
    lib.hesp_eval_descs.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                    C.POINTER(Best)]
    lib.hesp_eval_descs_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                           C.POINTER(Best), C.c_void_p]
    lib.hesp_generate_device.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]
    lib.hesp_generate_host.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
    lib.hesp_generate_batch.argtypes = [C.POINTER(GenConfig), C.c_int32, C.c_int32, C.c_int64, C.c_uint64,
                                        C.c_uint64, C.c_void_p]
    lib.hesp_eval_detail.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.POINTER(Outcome)]
    lib.hesp_engine_get_info.argtypes = [C.c_void_p, C.POINTER(EngineInfo)]
    lib.hesp_eval_trace.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(TraceC)]
    lib.hesp_solve.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(SolverConfigC), C.POINTER(SolverResultC)]
    lib.hesp_trace_bounds.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.hesp_min_reduce.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(Best)]
    lib.hesp_solve_batch.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.hesp_eval_neighbors.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64, C.c_void_p,
                                        C.POINTER(Best)]
    lib.hesp_fixture_load.restype = C.c_void_p
    lib.hesp_fixture_load.argtypes = [C.c_char_p, C.c_char_p]
    lib.hesp_fixture_platform.restype = C.POINTER(PlatformC)
    lib.hesp_fixture_platform.argtypes = [C.c_void_p]
    lib.hesp_fixture_model.restype = C.POINTER(PerfModelC)
    lib.hesp_fixture_model.argtypes = [C.c_void_p]
    lib.hesp_fixture_free.argtypes = [C.c_void_p]
    lib.hesp_choose_p.restype = C.c_double
    lib.hesp_choose_p.argtypes = [C.c_double, C.c_int64, C.c_int64, C.c_int32]
    lib.hesp_select_candidate.restype = C.c_int32
    lib.hesp_select_candidate.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_uint64)]
    lib.hesp_verify_trace.argtypes = [C.c_void_p, C.POINTER(TraceC), C.c_char_p, C.c_size_t,
                                      C.POINTER(C.c_int32)]
    lib.hesp_engine_destroy.argtypes = [C.c_void_p]
    lib.hesp_last_error.restype = C.c_char_p
    lib.hesp_status_name.restype = C.c_char_p
    lib.hesp_status_name.argtypes = [C.c_int32]
    _lib = lib
    return lib


def status_name(code: int) -> str:
    return load_library().hesp_status_name(int(code)).decode()


# ---------------------------------------------------------------------------
# Reference-shaped inputs


@dataclass
class Platform:
    """hesp::Platform (platform.hpp:50-86): spaces, types, processors, links."""
    spaces: list[tuple[int, int, bool]]
    types: list[str]
    processors: list[tuple[int, str, int]]
    links: list[tuple[int, int, float, float]] = field(default_factory=list)

    @staticmethod
    def from_json(text: str) -> "Platform":  # Platform::from_json, platform.cpp:157-196
        d = json.loads(text)
        return Platform(
            spaces=[(s["id"], int(s["capacity_bytes"]), bool(s.get("is_main", False))) for s in d["spaces"]],
            types=[t["name"] for t in d["types"]],
            processors=[(p["id"], p["type"], p["space"]) for p in d["processors"]],
            links=[(l["src"], l["dst"], float(l["latency_s"]), float(l["bandwidth_Bps"]))
                   for l in d.get("links", [])],
        )

    def _c(self, keep: list):
        sp = (Space * len(self.spaces))(*[Space(i, c, int(m)) for i, c, m in self.spaces])
        names = (C.c_char_p * len(self.types))(*[t.encode() for t in self.types])
        tix = {t: i for i, t in enumerate(self.types)}
        pr = (Processor * len(self.processors))(*[Processor(i, tix[t], s) for i, t, s in self.processors])
        nl = max(1, len(self.links))
        lk = (Link * nl)(*[Link(a, b, la, bw) for a, b, la, bw in self.links])
        keep += [sp, names, pr, lk]
        return PlatformC(len(self.spaces), sp, len(self.types), names, len(self.processors), pr,
                         len(self.links), lk)


@dataclass
class PerfModel:
    """hesp::PerfModel (platform.hpp:104-140), analytic or tabulated."""
    analytic: list[tuple[str, str, float, float]] | None = None  # (kind, type, peak, b_half)
    table: list[tuple[str, str, int, float]] | None = None       # (kind, type, b, seconds)

    @staticmethod
    def from_analytic_json(text: str) -> "PerfModel":
        return PerfModel(analytic=[(e["kind"], e["proc_type"], float(e["peak_flops"]), float(e["b_half"]))
                                   for e in json.loads(text)])

    @staticmethod
    def from_table_csv(text: str) -> "PerfModel":
        rows = []
        lines = [l for l in text.splitlines() if l.strip()]
        hdr = [f.strip() for f in lines[0].split(",")]
        if hdr != ["kind", "proc_type", "b", "seconds"]:
            raise ValueError("perf table: expected header kind,proc_type,b,seconds")
        for l in lines[1:]:
            k, t, b, s = [f.strip() for f in l.split(",")]
            rows.append((k, t, int(b), float(s)))
        return PerfModel(table=rows)

    def _c(self, platform: Platform, keep: list):
        tix = {t: i for i, t in enumerate(platform.types)}
        if self.analytic is not None:
            ents = [AnalyticEntry(KINDS[k], tix[t], p, bh) for k, t, p, bh in self.analytic if t in tix]
            arr = (AnalyticEntry * max(1, len(ents)))(*ents)
            keep.append(arr)
            return PerfModelC(1, len(ents), arr, 0, None)
        rows = [TableRow(KINDS[k], tix[t], b, s) for k, t, b, s in self.table if t in tix]
        arr = (TableRow * max(1, len(rows)))(*rows)
        keep.append(arr)
        return PerfModelC(0, 0, None, len(rows), arr)


@dataclass
class SchedConfig:
    """hesp::SchedConfig (sim.hpp:26-32)."""
    ordering: str = "PL"
    selection: str = "EFT-P"
    caching: str = "WB"
    seed: int = 0
    min_block: int = 64


@dataclass
class Workload:
    """root_cholesky(n, elem) + partition_task(0, 1/s_base) + generated candidates."""
    n: int = 16384
    elem_size: int = 4
    s_base: int = 16
    seed: int = 1
    k_max: int = 8
    max_depth: int = 3
    min_block: int = 64
    s_choices: tuple = (2, 4)
    merge_pct: int = 0


class BatchEngine:
    """One engine handle on one GPU (hesp_engine_create)."""

    def __init__(self, platform: Platform, model: PerfModel, sched: SchedConfig, workload: Workload,
                 device: int = 0):
        self.lib = load_library()
        keep: list = []
        self._pc = platform._c(keep)
        self._mc = model._c(platform, keep)
        self._sc = SchedConfigC(ORDERING[sched.ordering], SELECTION[sched.selection], CACHING[sched.caching],
                                0, sched.seed, sched.min_block)
        sc = (C.c_int32 * 4)(*(list(workload.s_choices) + [0] * (4 - len(workload.s_choices))))
        g = GenConfig(workload.seed, workload.k_max, workload.max_depth, workload.min_block,
                      len(workload.s_choices), sc, workload.merge_pct)
        self._wc = WorkloadC(workload.n, workload.elem_size, workload.s_base, g)
        self._keep = keep
        h = self.lib.hesp_engine_create(device, C.byref(self._pc), C.byref(self._mc), C.byref(self._sc),
                                        C.byref(self._wc))
        if not h:
            raise RuntimeError("hesp_engine_create: " + self.lib.hesp_last_error().decode())
        self.h = C.c_void_p(h)
        self.workload, self.sched = workload, sched

    @classmethod
    def from_files(cls, platform_path: str, model_path: str, sched: SchedConfig, workload: Workload,
                   device: int = 0) -> "BatchEngine":
        """Engine from the reference's fixture files read by the library itself
        (hesp_fixture_load: Platform::from_json / PerfModel::from_*)."""
        lib = load_library()
        fx = lib.hesp_fixture_load(platform_path.encode(), model_path.encode())
        if not fx:
            raise RuntimeError("hesp_fixture_load: " + lib.hesp_last_error().decode())
        self = cls.__new__(cls)
        self.lib = lib
        self._fx = fx
        self._pc = lib.hesp_fixture_platform(fx).contents
        self._mc = lib.hesp_fixture_model(fx).contents
        self._sc = SchedConfigC(ORDERING[sched.ordering], SELECTION[sched.selection], CACHING[sched.caching],
                                0, sched.seed, sched.min_block)
        sc = (C.c_int32 * 4)(*(list(workload.s_choices) + [0] * (4 - len(workload.s_choices))))
        g = GenConfig(workload.seed, workload.k_max, workload.max_depth, workload.min_block,
                      len(workload.s_choices), sc, workload.merge_pct)
        self._wc = WorkloadC(workload.n, workload.elem_size, workload.s_base, g)
        self._keep = []
        h = lib.hesp_engine_create(device, C.byref(self._pc), C.byref(self._mc), C.byref(self._sc),
                                   C.byref(self._wc))
        if not h:
            raise RuntimeError("hesp_engine_create: " + lib.hesp_last_error().decode())
        self.h = C.c_void_p(h)
        self.workload, self.sched = workload, sched
        return self

    def close(self):
        if getattr(self, "h", None):
            self.lib.hesp_engine_destroy(self.h)
            self.h = None
        if getattr(self, "_fx", None):
            self.lib.hesp_fixture_free(self._fx)
            self._fx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int, what: str):
        if rc != 0:
            raise RuntimeError(f"{what} failed ({rc}): {self.lib.hesp_last_error().decode()}")

    def info(self) -> EngineInfo:
        i = EngineInfo()
        self._check(self.lib.hesp_engine_get_info(self.h, C.byref(i)), "get_info")
        return i

    def eval_generated(self, first: int, count: int, outcomes: bool = True):
        out = np.zeros(count, OUTCOME_DTYPE) if outcomes else None
        best = Best()
        self._check(self.lib.hesp_eval_generated(self.h, first, count,
                                                 out.ctypes.data if out is not None else None,
                                                 C.byref(best)), "eval_generated")
        return out, best

    def eval_descs(self, descs: np.ndarray, first: int = 0):
        descs = np.ascontiguousarray(descs, DESC_DTYPE)
        out = np.zeros(len(descs), OUTCOME_DTYPE)
        best = Best()
        self._check(self.lib.hesp_eval_descs(self.h, descs.ctypes.data, len(descs), first, out.ctypes.data,
                                             C.byref(best)), "eval_descs")
        return out, best

    def eval_descs_device(self, descs_ptr: int, count: int, first: int, out_ptr: int | None, stream: int = 0):
        best = Best()
        self._check(self.lib.hesp_eval_descs_device(self.h, C.c_void_p(descs_ptr), count, first,
                                                    C.c_void_p(out_ptr) if out_ptr else None, C.byref(best),
                                                    C.c_void_p(stream) if stream else None),
                    "eval_descs_device")
        return best

    def generate_device(self, first: int, count: int, descs_ptr: int, stream: int = 0):
        self._check(self.lib.hesp_generate_device(self.h, first, count, C.c_void_p(descs_ptr),
                                                  C.c_void_p(stream) if stream else None), "generate_device")

    def eval_detail(self, desc: np.ndarray, cap: int):
        """Per-task (proc, start, end) of one candidate (proc -1 = not a scheduled leaf)."""
        desc = np.ascontiguousarray(desc, DESC_DTYPE).reshape(1)
        proc = np.full(cap, -1, np.int32)
        start = np.zeros(cap, np.float64)
        end = np.zeros(cap, np.float64)
        o = Outcome()
        rc = self.lib.hesp_eval_detail(self.h, desc.ctypes.data, cap, proc.ctypes.data, start.ctypes.data,
                                       end.ctypes.data, C.byref(o))
        if rc < 0:
            self._check(rc, "eval_detail")
        return o, proc, start, end

    def eval_trace(self, desc: np.ndarray, caps: tuple[int, int, int, int, int] | None = None) -> Trace:
        """Full SimResult of one candidate (hesp_eval_trace).  Arrays grow on HESP_E_LIMIT."""
        desc = np.ascontiguousarray(desc, DESC_DTYPE).reshape(1)
        na, nx, nr, ne, ns = caps or (4096, 8192, 16384, 32768, 8192)
        for _ in range(3):
            arrs = (np.zeros(na, ASSIGN_DTYPE), np.zeros(nx, XFER_DTYPE), np.zeros(nr, RES_DTYPE),
                    np.zeros(ne, EVENT_DTYPE), np.zeros(ns, STEP_DTYPE))
            t = TraceC(na, nx, nr, ne, ns, 0, *[a.ctypes.data for a in arrs])
            rc = self.lib.hesp_eval_trace(self.h, desc.ctypes.data, C.byref(t))
            if rc == -4:  # HESP_E_LIMIT: the counts say what is needed
                na, nx, nr, ne, ns = (max(na, t.n_assign), max(nx, t.n_xfer), max(nr, t.n_res),
                                      max(ne, t.n_events), max(ns, t.n_steps))
                continue
            if rc < 0:
                self._check(rc, "eval_trace")
            self._last_trace = (t, arrs)
            a, x, r, e, st = arrs
            return Trace(int(t.outcome.status), int(t.outcome.n_leaves), float(t.outcome.makespan),
                         a[:t.n_assign].copy(), x[:t.n_xfer].copy(), e[:t.n_events].copy(), r[:t.n_res].copy(),
                         st[:t.n_steps].copy(), float(t.busy_time), float(t.avg_load), float(t.load_integral))
        raise RuntimeError("eval_trace: could not size the trace arrays")

    def trace_bounds(self) -> tuple[float, float]:
        """(critical-path, work) makespan lower bounds of the last eval_trace candidate."""
        cp, w = C.c_double(), C.c_double()
        self._check(self.lib.hesp_trace_bounds(self.h, C.byref(cp), C.byref(w)), "trace_bounds")
        return cp.value, w.value

    def verify_trace(self, trace: Trace) -> list[str]:
        """verify_schedule of `trace` (possibly edited) against the graph of the last eval_trace."""
        a = np.ascontiguousarray(trace.assignments)
        x = np.ascontiguousarray(trace.transfers)
        r = np.ascontiguousarray(trace.residency)
        t = TraceC(len(a), len(x), len(r), 0, 0, 0, a.ctypes.data, x.ctypes.data, r.ctypes.data, None, None,
                   len(a), len(x), len(r), 0, 0, 0)
        t.outcome.status = trace.status
        t.outcome.makespan = trace.makespan
        buf = C.create_string_buffer(1 << 22)
        n = C.c_int32(0)
        self._check(self.lib.hesp_verify_trace(self.h, C.byref(t), buf, len(buf), C.byref(n)), "verify_trace")
        text = buf.value.decode()
        return text.split("\n") if n.value else []

    def solve(self, iterations: int = 50, task_selection: str = "All", sampling: str = "Soft", seed: int = 0,
              k_max: int = 8, min_block: int = 64, overhead_factor: float = 1.1, initial: np.ndarray | None = None):
        """SPEC solve() (hesp_solve): returns (history, best descriptor, best makespan, best iteration,
        device simulations issued)."""
        cfg = SolverConfigC(iterations, TASK_SELECTION[task_selection], SAMPLING[sampling], k_max, seed, min_block,
                            overhead_factor)
        hist = np.zeros(max(1, iterations), SOLVER_ITER_DTYPE)
        res = SolverResultC()
        res.cap_history = len(hist)
        res.history = hist.ctypes.data
        init = None
        if initial is not None:
            init = np.ascontiguousarray(initial, DESC_DTYPE).reshape(1)
        rc = self.lib.hesp_solve(self.h, init.ctypes.data if init is not None else None, C.byref(cfg), C.byref(res))
        if rc < 0:
            self._check(rc, "solve")
        if rc > 0:
            raise RuntimeError(f"solve: initial state fails with status {rc} ({status_name(rc)})")
        best = np.frombuffer(bytes(res.best), DESC_DTYPE)[0].copy()
        # first iteration whose candidates hit the descriptor's op budget (-1: never)
        self.last_budget_iteration = int(res.budget_iteration)
        return hist[:res.n_history].copy(), best, float(res.best_makespan), int(res.best_iteration), \
            int(res.n_simulated)

    def min_reduce(self, nccl_comm: int, best: Best) -> Best:
        """hesp_min_reduce: the exact cross-rank winner over an ncclComm_t (K3)."""
        b = Best()
        C.memmove(C.byref(b), C.byref(best), C.sizeof(Best))
        self._check(self.lib.hesp_min_reduce(self.h, C.c_void_p(nccl_comm), C.byref(b)), "min_reduce")
        return b

    def solve_batch(self, chains: list[dict]):
        """hesp_solve_batch: independent chains in lockstep (one trace launch and
        one candidate batch per iteration for all of them).  Each dict takes
        solve()'s keyword arguments (iterations, task_selection, sampling, seed,
        k_max, min_block, overhead_factor); returns one solve()-shaped tuple per chain."""
        n = len(chains)
        cfgs = (SolverConfigC * n)()
        hists, res = [], (SolverResultC * n)()
        for i, c in enumerate(chains):
            it = c.get("iterations", 50)
            cfgs[i] = SolverConfigC(it, TASK_SELECTION[c.get("task_selection", "All")],
                                    SAMPLING[c.get("sampling", "Soft")], c.get("k_max", 8), c.get("seed", 0),
                                    c.get("min_block", 64), c.get("overhead_factor", 1.1))
            h = np.zeros(max(1, it), SOLVER_ITER_DTYPE)
            hists.append(h)
            res[i].cap_history = len(h)
            res[i].history = h.ctypes.data
        rc = self.lib.hesp_solve_batch(self.h, n, None, C.cast(cfgs, C.c_void_p), C.cast(res, C.c_void_p))
        if rc < 0:
            self._check(rc, "solve_batch")
        if rc > 0:
            raise RuntimeError(f"solve_batch: an initial state fails with status {rc} ({status_name(rc)})")
        out = []
        self.last_budget_iterations = [int(res[i].budget_iteration) for i in range(n)]
        for i in range(n):
            best = np.frombuffer(bytes(res[i].best), DESC_DTYPE)[0].copy()
            out.append((hists[i][:res[i].n_history].copy(), best, float(res[i].best_makespan),
                        int(res[i].best_iteration), int(res[i].n_simulated)))
        return out

    def eval_neighbors(self, bases: np.ndarray, nbrs: np.ndarray):
        """hesp_eval_neighbors: candidate k = bases[nbrs[k].base] + nbrs[k].ops[:n_ops]."""
        bases = np.ascontiguousarray(bases, DESC_DTYPE)
        nbrs = np.ascontiguousarray(nbrs, NEIGHBOR_DTYPE)
        out = np.zeros(len(nbrs), OUTCOME_DTYPE)
        best = Best()
        self._check(self.lib.hesp_eval_neighbors(self.h, bases.ctypes.data, len(bases), nbrs.ctypes.data, len(nbrs),
                                                 out.ctypes.data, C.byref(best)), "eval_neighbors")
        return out, best

    def generate_host(self, first: int, count: int) -> np.ndarray:
        d = np.zeros(count, DESC_DTYPE)
        self._check(self.lib.hesp_generate_host(self.h, first, count, d.ctypes.data), "generate_host")
        return d


def generate_batch(workload: "Workload", n_base: int, base_b: int, first: int, count: int) -> np.ndarray:
    """Host generator (hesp_generate_batch): no engine or GPU needed."""
    lib = load_library()
    sc = (C.c_int32 * 4)(*(list(workload.s_choices) + [0] * (4 - len(workload.s_choices))))
    g = GenConfig(workload.seed, workload.k_max, workload.max_depth, workload.min_block, len(workload.s_choices), sc,
                  workload.merge_pct)
    d = np.zeros(count, DESC_DTYPE)
    rc = lib.hesp_generate_batch(C.byref(g), workload.n // base_b, n_base, base_b, first, count, d.ctypes.data)
    if rc != 0:
        raise RuntimeError("hesp_generate_batch failed")
    return d


# ---------------------------------------------------------------------------
# Fixtures

FIXTURES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fixtures")


def fixture_path(name: str) -> str:
    return os.path.join(FIXTURES, name)


def load_platform(name: str) -> Platform:
    with open(fixture_path(name)) as f:
        return Platform.from_json(f.read())


def load_model(name: str) -> PerfModel:
    with open(fixture_path(name)) as f:
        text = f.read()
    return PerfModel.from_table_csv(text) if name.endswith(".csv") else PerfModel.from_analytic_json(text)
