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
