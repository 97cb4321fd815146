"""Sharded partitioning search (BASELINE.json configs C4 / C5).

    python -m paper_1602_05510_b200.search --config C5 --candidates 10000000            # 1 GPU
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 -m paper_1602_05510_b200.search \\
        --config C5 --candidates 10000000                                                # 8 GPUs

Each rank takes a disjoint, contiguous share of the candidate index range
(`dist.shard`), generates and evaluates it on its own GPU in device batches
(no descriptors cross PCIe), and keeps its best (makespan, index).  The only
exchange is the final winner: `hesp_min_reduce` (C ABI), two 8-byte MIN all-reduces
over NCCL.  Rank 0 prints one JSON line; with --trace-winner it re-simulates
the winner with the full trace (hesp_eval_trace) and runs verify_schedule.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--candidates", type=int, default=1_000_000)
    ap.add_argument("--first", type=int, default=0)
    ap.add_argument("--batch", type=int, default=1_000_000, help="candidates per device call")
    ap.add_argument("--trace-winner", action="store_true")
    args = ap.parse_args(argv)

    import torch
    import torch.distributed as dist

    from .configs import CONFIGS, PARITY, make_engine
    from .dist import engine_global_best, shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    own_pg = not dist.is_initialized()
    if own_pg:
        from .dist import init_nccl
        init_nccl(local)  # 1-rank group at N=1: the winner still goes through hesp_min_reduce
    p = CONFIGS.get(args.config) or PARITY[args.config][0]
    eng = make_engine(p, device=local)
    begin, end = shard(args.candidates, world, rank, args.first)
    eng.eval_generated(begin, min(1024, max(1, end - begin)), outcomes=False)  # warm-up
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    best_mk, best_idx, n_ok, n_eval = float("nan"), -1, 0, 0
    for b0 in range(begin, end, args.batch):
        cnt = min(args.batch, end - b0)
        _, b = eng.eval_generated(b0, cnt, outcomes=False)
        n_ok += b.n_ok
        n_eval += b.n_evaluated
        if b.index >= 0 and (best_idx < 0 or b.makespan < best_mk or (b.makespan == best_mk and b.index < best_idx)):
            best_mk, best_idx = b.makespan, b.index
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt, float(n_ok), float(n_eval)], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t[1:].clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        t = torch.cat([tmax, tsum])
    wall, ok_all, ev_all = float(t[0]), int(t[1]), int(t[2])
    from .engine import Best
    mine = Best()
    mine.makespan, mine.index = (best_mk, best_idx) if best_idx >= 0 else (0.0, -1)
    (gmk, gidx), _ = engine_global_best(eng, mine)  # hesp_min_reduce over NCCL
    if rank == 0:
        line = {"config": args.config, "candidates": args.candidates, "n_gpus": world, "evaluated": ev_all,
                "valid": ok_all, "seconds_max_over_ranks": wall, "schedules_per_s": ev_all / wall,
                "best": {"makespan": gmk, "index": gidx}}
        if args.trace_winner and gidx >= 0:
            desc = eng.generate_host(gidx, 1)[0]
            tr = eng.eval_trace(desc)
            line["winner_trace"] = {"status": tr.status, "makespan": tr.makespan, "tasks": len(tr.assignments),
                                    "transfers": len(tr.transfers), "events": len(tr.events),
                                    "avg_load": tr.avg_load, "verify_violations": len(eng.verify_trace(tr)),
                                    "ops": [[int(o[0]), int(o[1])] for o in desc["ops"][:int(desc["n_ops"])]]}
            assert tr.makespan == gmk, (tr.makespan, gmk)
        print(json.dumps(line))
    if own_pg:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
