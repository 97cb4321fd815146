"""The cross-rank winner selection (paper_1602_05510_b200.dist) on a
world_size-2 gloo group: exact (makespan, lowest index) argmin, ties and
ranks without a valid candidate included."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = [
    # (rank0 (makespan, index), rank1 (makespan, index), expected)
    ((0.5, 10), (0.25, 7_000_000), (0.25, 7_000_000)),
    ((0.25, 99), (0.25, 12), (0.25, 12)),          # tie on makespan: lowest global index
    ((0.0, -1), (0.3, 5), (0.3, 5)),               # rank 0 found nothing valid
    ((0.0, -1), (0.0, -1), (None, -1)),            # nobody found anything
    ((1e-300, 3), (1e300, 1), (1e-300, 3)),
]


def _worker(rank, port, results):
    import torch.distributed as dist
    from paper_1602_05510_b200.dist import global_best
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    out = []
    for a, b, _ in CASES:
        mk, idx = (a, b)[rank]
        out.append(global_best(mk, idx, device="cpu"))
    results[rank] = out
    dist.destroy_process_group()


def test_global_best_gloo_world2():
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), results), nprocs=2, join=True)
    for r in range(2):
        for (a, b, want), got in zip(CASES, results[r]):
            if want[0] is None:
                assert got[1] == -1
            else:
                assert got == want, (a, b, got)
