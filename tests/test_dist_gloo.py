"""The multi-GPU (N > 1) host path with world_size 2 over gloo on the CPU:
contiguous shards, no data exchange in the solve, results gathered to rank 0
equal the single-process result bit for bit.  The per-rank solve here is the
oracle (the CPU checker) standing in for each rank's GPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2403_16341_b200 import sharding, workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = W.c2_suite(12, 0, 1001, 0.1)  # odd size: uneven shards
    seen = []

    def fn(u0, p):
        seen.append(len(u0))
        return O.solve_batch(b.problem_id, "trust-region", u0, threads=1)

    res = sharding.solve_sharded(fn, b.u0)
    lo, hi = sharding.local_slice(len(b.u0))
    assert seen == [hi - lo]
    if rank == 0:
        np.savez(out_path, **res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_and_gather(tmp_path):
    from oracle import oracle as O
    from paper_2403_16341_b200 import workloads as W
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    b = W.c2_suite(12, 0, 1001, 0.1)
    ref = O.solve_batch(b.problem_id, "trust-region", b.u0, threads=2)
    for k in ("u", "resid", "retcode", "nsteps", "nf", "njac", "nlinsolve"):
        assert np.array_equal(got[k], ref[k]), k


def _bench_worker(rank, world, port, out_path, global_batch):
    """The bench's N > 1 data path (bench.rank_rows + jobs_for + the max /
    sum reductions), with the oracle standing in for each rank's GPU."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import bench
    from oracle import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = bench.rank_rows(7, global_batch, world, rank)
    jobs = bench.jobs_for("c4", lo, hi)
    (pid, n, alg, b), = jobs
    r = O.solve_batch(pid, alg, b.u0, threads=1)
    t = torch.tensor([float(hi - lo)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, r))
    if rank == 0:
        parts = sorted(gathered, key=lambda x: x[0])
        np.savez(out_path, total=t.item(), bounds=np.array([(p[0], p[1]) for p in parts]),
                 **{k: np.concatenate([p[2][k] for p in parts]) for k in ("u", "retcode", "nsteps")})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("global_batch", [None, 23])
def test_bench_shards_strong_and_weak(tmp_path, global_batch):
    """--global-batch G splits G rows per job evenly over the ranks (strong
    scaling; the union is exactly rows [0, G)); without it every rank takes
    its own --batch rows (weak scaling).  The SUM reduction gives the
    whole-job system count the bench's `value` divides by."""
    from oracle import oracle as O
    import bench
    world = 2
    out = str(tmp_path / "bench_shards.npz")
    mp.spawn(_bench_worker, args=(world, _free_port(), out, global_batch), nprocs=world, join=True)
    got = np.load(out)
    total = global_batch or 7 * world
    assert got["total"] == total
    assert got["bounds"][0][0] == 0 and got["bounds"][-1][1] == total
    assert all(got["bounds"][i][1] == got["bounds"][i + 1][0] for i in range(world - 1))
    (pid, n, alg, b), = bench.jobs_for("c4", 0, total)
    ref = O.solve_batch(pid, alg, b.u0, threads=2)
    for k in ("u", "retcode", "nsteps"):
        assert np.array_equal(got[k], ref[k]), k
