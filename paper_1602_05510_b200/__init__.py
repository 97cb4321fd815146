"""B200-native batched candidate-schedule engine for HeSP (arXiv:1602.05510).

The hot path — expand a candidate recursive partitioning of the tiled
Cholesky DAG, simulate its heterogeneous list schedule with transfer and
coherence costs, and reduce a batch to the best makespan — runs as
hand-written sm_100a CUDA behind the C ABI in include/hesp_engine.h.
"""
from .build import LIB, build  # noqa: F401
from .configs import CONFIGS, PARITY, make_engine  # noqa: F401
from .engine import (BatchEngine, PerfModel, Platform, SchedConfig, Workload,  # noqa: F401
                     load_library, status_name)

__all__ = ["LIB", "build", "CONFIGS", "PARITY", "make_engine", "BatchEngine", "PerfModel", "Platform",
           "SchedConfig", "Workload", "load_library", "status_name"]
