"""Multi-GPU plumbing for batched solves (one process per GPU).

Independent systems / right-hand sides shard contiguously over ranks with no
data-path collective (each rank runs the whole pipeline on its shard); the
only exchange is the final gather of solutions to one rank.
torch.distributed provides the communicator (NCCL on GPUs, gloo on CPU for
the tests).
"""

from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist

__all__ = ["shard_range", "shard_counts", "gather_solutions", "solve_sharded"]


def shard_counts(total: int, world: int) -> List[int]:
    base, extra = divmod(total, world)
    return [base + (1 if r < extra else 0) for r in range(world)]


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) block of `total` items owned by `rank`."""
    counts = shard_counts(total, world)
    lo = sum(counts[:rank])
    return lo, lo + counts[rank]


def gather_solutions(x_local: torch.Tensor, total: int, dst: int = 0, group=None):
    """Gather per-rank blocks [count_r, ...] into [total, ...] on `dst`
    (rank order = system order).  Returns the full tensor on dst, None
    elsewhere.  Blocks are padded to the largest shard for the collective."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    counts = shard_counts(total, world)
    width = max(counts)
    tail = tuple(x_local.shape[1:])
    buf = torch.zeros((width,) + tail, dtype=x_local.dtype, device=x_local.device)
    buf[: x_local.shape[0]] = x_local
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, gather_list=parts, dst=dst, group=group)
        return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
    dist.gather(buf, gather_list=None, dst=dst, group=group)
    return None


def solve_sharded(problems, solve_fn, dst: int = 0, group=None):
    """Solve a batch of independent problems split over the ranks: this rank
    runs ``solve_fn(shard) -> [count_r, n] complex`` on its contiguous shard
    (``solve_tikhonov_batch`` / ``DeviceBatch`` on a GPU), then the solutions
    are gathered to ``dst`` in problem order.  Returns the [total, n] complex
    array on ``dst``, None elsewhere."""
    import numpy as np
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(len(problems), rank, world)
    x = np.ascontiguousarray(solve_fn(problems[lo:hi]), dtype=np.complex128)
    local = torch.from_numpy(x.view(np.float64).reshape(hi - lo, -1, 2))
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    full = gather_solutions(local.to(dev), len(problems), dst=dst, group=group)
    if full is None:
        return None
    return full.cpu().numpy().reshape(len(problems), -1).view(np.complex128)
