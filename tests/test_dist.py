"""N>1 host path on CPU: world_size 2 over gloo (127.0.0.1).  Shards are
contiguous, cover every system exactly once, and the gather returns the
solutions in system order - the same logic bench.py runs over NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1302_6945_b200.dist import gather_solutions, shard_counts, shard_range


def test_shards_cover_everything():
    for total in (1, 7, 64, 4096):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(total, r, world)
                seen.extend(range(lo, hi))
            assert seen == list(range(total))
            assert max(shard_counts(total, world)) - min(shard_counts(total, world)) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(total, rank, world)
    # each "system" i's solution is a vector filled with i (complex as 2 doubles)
    x = torch.arange(lo, hi, dtype=torch.float64)[:, None, None].expand(hi - lo, 5, 2).contiguous()
    full = gather_solutions(x, total, dst=0)
    if rank == 0:
        q.put(full[:, 0, 0].tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [7, 64])
def test_gather_in_system_order_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == [float(i) for i in range(total)]
