"""One rank of the two-process hesp_min_reduce test (tests/test_min_reduce_gpu.py).

argv: rank world shim_so dir first count  -> prints one JSON line with the
rank-local best and the all-rank result hesp_min_reduce returned."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    rank, world, shim, d, first, count = sys.argv[1:7]
    rank, world, first, count = int(rank), int(world), int(first), int(count)
    os.environ["HESP_NCCL_LIB"] = shim  # read by the engine's NCCL loader on first use
    lib = C.CDLL(shim, mode=C.RTLD_GLOBAL)
    lib.shim_comm_init.restype = C.c_void_p
    lib.shim_comm_init.argtypes = [C.c_int, C.c_int, C.c_char_p]
    lib.shim_calls.restype = C.c_long
    lib.shim_calls.argtypes = [C.c_void_p]
    comm = lib.shim_comm_init(rank, world, d.encode())
    from paper_1602_05510_b200.configs import PARITY, make_engine
    p, _ = PARITY["c2"]
    eng = make_engine(p)
    _, b = eng.eval_generated(first, count, outcomes=False)
    local = {"makespan": b.makespan, "index": b.index, "n_ok": b.n_ok, "n_evaluated": b.n_evaluated,
             "sum_leaves": b.sum_leaves}
    g = eng.min_reduce(comm, b)
    out = {"rank": rank, "local": local,
           "global": {"makespan": g.makespan, "index": g.index, "n_ok": g.n_ok, "n_evaluated": g.n_evaluated,
                      "sum_leaves": g.sum_leaves},
           "shim_calls": lib.shim_calls(comm), "min_reduces": eng.info().min_reduces}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
