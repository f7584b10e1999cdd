"""Host-side multi-rank plumbing on torch.distributed (works with the nccl and gloo backends).

* ``share_unique_id``   rank 0 draws the NCCL unique id through the C ABI, every rank gets it
                        (the bootstrap of spmat_comm_create)
* ``layout``            contiguous ownership offsets from every rank's local size, in rank order
                        ("distributed row-wise across MPI processes")
* ``max_over_ranks``    the benchmark timing reduction (the slowest rank decides)

No arithmetic of the method lives here; it only moves a few host integers between ranks.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _dev():
    """Device for collectives of the current default group (nccl needs cuda tensors)."""
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def share_unique_id(make_id) -> bytes | None:
    """Rank 0 calls ``make_id()`` (e.g. comm_unique_id); the bytes are broadcast to all."""
    P, r = world()
    if P == 1:
        return None
    obj = [make_id() if r == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def layout(local_size: int) -> list[int]:
    """Ownership offsets [0, n_0, n_0+n_1, ...] from every rank's local size."""
    P, _ = world()
    if P == 1:
        return [0, int(local_size)]
    t = torch.tensor([int(local_size)], dtype=torch.int64, device=_dev())
    out = [torch.zeros_like(t) for _ in range(P)]
    dist.all_gather(out, t)
    offs = [0]
    for v in out:
        offs.append(offs[-1] + int(v.item()))
    return offs


def max_over_ranks(value: float) -> float:
    P, _ = world()
    if P == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: int) -> int:
    P, _ = world()
    if P == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=_dev())
    dist.all_reduce(t)
    return int(t.item())


def barrier():
    P, _ = world()
    if P > 1:
        dist.barrier()
