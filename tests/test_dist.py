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


def _solve_worker(rank, world, port, q):
    import sys
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import toepreg_oracle as O  # the checker stands in for the GPU solve on CPU
    import paper_1302_6945_b200 as tb
    from paper_1302_6945_b200 import workloads as wl
    from paper_1302_6945_b200.dist import solve_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    raw = wl.c2_rect(m=96, n=48, nrhs=5, seed=4)  # config-2 shape: one T, 5 right-hand sides
    probs = [wl.to_problem(raw, tb, i) for i in range(5)]
    full = solve_sharded(probs, lambda shard: np.stack([O.solve(p)["x_hat"] for p in shard]))
    if rank == 0:
        q.put(full)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_solutions_equal_single_process_world2():
    """Solver output (not synthetic tensors) through the sharded path: each
    rank solves its contiguous shard of the right-hand sides, rank 0 gathers,
    and the result equals the one-process solves bit for bit."""
    import sys
    import numpy as np
    from conftest import ROOT
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import toepreg_oracle as O
    import paper_1302_6945_b200 as tb
    from paper_1302_6945_b200 import workloads as wl
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    raw = wl.c2_rect(m=96, n=48, nrhs=5, seed=4)
    want = np.stack([O.solve(wl.to_problem(raw, tb, i))["x_hat"] for i in range(5)])
    assert got.shape == want.shape and np.array_equal(got, want)


def test_bench_c2_shards_split_the_64_rhs():
    """bench.py's N > 1 c2 workload splits ONE instance's 64 right-hand
    sides over the ranks (strong scaling), covering each exactly once."""
    import sys
    import numpy as np
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    import bench
    full, count, _ = bench.make_workload("c2", 0, 8, 1)
    parts = [bench.make_workload("c2", r, 8, 4) for r in range(4)]
    assert count == 8 and [c for _, c, _ in parts] == [2, 2, 2, 2]
    assert np.array_equal(np.concatenate([p["b"] for p, _, _ in parts]), full["b"])
    assert all(np.array_equal(p["T_gen"], full["T_gen"]) for p, _, _ in parts)
