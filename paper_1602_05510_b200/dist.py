"""Cross-GPU plumbing for candidate sharding.

Candidates are independent, so G ranks take disjoint index
ranges and the only exchange is the final winner: an exact lexicographic
argmin of (makespan, global index) over ranks, done as two 8-byte MIN
all-reduces (NCCL over NVLink on GPUs; gloo in the CPU tests):

  1. MIN over the order-preserving int64 view of each rank's best makespan
     (positive IEEE doubles order like their bit patterns);
  2. MIN over the index among ranks whose makespan equals the global one.
"""
from __future__ import annotations

import numpy as np

NONE = np.iinfo(np.int64).max


def shard(total: int, world: int, rank: int, first: int = 0) -> tuple[int, int]:
    """[begin, end) of rank's contiguous share of `total` candidates starting at `first`."""
    base, rem = divmod(total, world)
    begin = first + rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def makespan_key(makespan: float, index: int) -> int:
    """int64 order key of a rank-local best (NONE when the rank found no valid candidate)."""
    if index < 0:
        return NONE
    return int(np.float64(makespan).view(np.int64))


def global_best(makespan: float, index: int, device="cpu", group=None) -> tuple[float, int]:
    """Exact (makespan, lowest index) argmin across all ranks of `group`."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return (makespan, index) if index >= 0 else (float("nan"), -1)
    key = makespan_key(makespan, index)
    t = torch.tensor([key], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    gkey = int(t.item())
    if gkey == NONE:
        return float("nan"), -1
    mine = index if key == gkey else NONE
    u = torch.tensor([mine], dtype=torch.int64, device=device)
    dist.all_reduce(u, op=dist.ReduceOp.MIN, group=group)
    return float(np.int64(gkey).view(np.float64)), int(u.item())


def init_nccl(local_rank: int):
    """One NCCL process group per GPU process.  Under torchrun the rendezvous
    comes from the environment; a plain `python bench.py` (N=1) gets a 1-rank
    group on 127.0.0.1 so the cross-GPU winner path (hesp_min_reduce over the
    group's communicator) runs at every N."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", local_rank)
    if "WORLD_SIZE" in os.environ:  # torchrun
        dist.init_process_group("nccl", device_id=dev)
    else:
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=dev)
    dist.barrier()  # creates the communicator


def nccl_comm_ptr(group=None) -> int:
    """Raw ncclComm_t of a NCCL process group (0 if the communicator does not
    exist yet: it is created by the group's first collective)."""
    import torch
    import torch.distributed as dist
    pg = group or dist.group.WORLD
    backend = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
    return int(backend._comm_ptr())


def engine_global_best(eng, best, group=None):
    """K3 through the engine's C ABI: hesp_min_reduce over the process group's
    own NCCL communicator (NVLink/NVSwitch on one node).  Returns
    (makespan, index) like global_best, plus the all-rank hesp_best."""
    import torch.distributed as dist
    if not dist.is_initialized():
        return (best.makespan, best.index) if best.index >= 0 else (float("nan"), -1), best
    if dist.get_backend(group) != "nccl":  # gloo (CPU tests): the same two-round argmin in torch
        mk, idx = global_best(best.makespan, best.index, group=group)
        return (mk, idx), best
    # NCCL, any world size (a 1-rank group too, so N=1 runs exercise K3)
    comm = nccl_comm_ptr(group)
    if not comm:
        dist.barrier(group=group)  # creates the communicator
        comm = nccl_comm_ptr(group)
    g = eng.min_reduce(comm, best)
    return (g.makespan, g.index) if g.index >= 0 else (float("nan"), -1), g
