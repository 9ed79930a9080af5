"""Even sharding of a batch across the GPUs of one box.

Every system is independent, so a batch is split into contiguous slices
(remainder to the first ranks), each rank solves its slice on its own GPU
with no inter-GPU traffic, and the per-system results are gathered to rank 0
(the reference's results land where its caller is).  The only collectives are
result gathering and timing reductions — never inside the solve.
"""

from __future__ import annotations

import numpy as np
import torch

from .workloads import shard_bounds

FIELDS = ("u", "resid", "retcode", "nsteps", "nf", "njac", "nlinsolve")


def local_slice(B, group=None):
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return shard_bounds(B, world, rank)


def gather_to_root(local, B, group=None, root=0):
    """Assemble per-rank result dicts (numpy arrays, leading dim = local
    shard) into full [B, ...] arrays on `root`; other ranks get None.
    Works over gloo (CPU tensors) and NCCL (CUDA tensors)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    sizes = [hi - lo for lo, hi in (shard_bounds(B, world, r) for r in range(world))]
    maxsz = max(sizes)
    out = {} if rank == root else None
    for k in FIELDS:
        a = np.asarray(local[k])
        pad = np.zeros((maxsz,) + a.shape[1:], dtype=a.dtype)
        pad[: len(a)] = a
        t = torch.from_numpy(pad.view(np.uint8) if a.dtype == np.int8 else pad).to(dev)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        if rank == root:
            full = [p.cpu().numpy()[: sizes[r]] for r, p in enumerate(parts)]
            full = np.concatenate(full)
            out[k] = full.view(np.int8) if a.dtype == np.int8 else full
    return out


def solve_sharded(solve_fn, u0, p=None, group=None):
    """Solve the rank's contiguous slice of a global batch with
    ``solve_fn(u0_slice, p_slice) -> dict`` and gather to rank 0."""
    B = len(u0)
    lo, hi = local_slice(B, group)
    local = solve_fn(u0[lo:hi], None if p is None else p[lo:hi])
    local = {k: np.asarray(local[k].cpu() if torch.is_tensor(local[k]) else local[k])
             for k in FIELDS}
    return gather_to_root(local, B, group)


def gpu_solve_fn(problem, algorithm="newton-raphson", options=None, dtype=torch.float64):
    """solve_fn for solve_sharded: the rank's slice on its current GPU."""
    from . import solvers

    def fn(u0, p):
        return solvers.solve_batch(problem, u0, p, algorithm, options, dtype=dtype,
                                   n=u0.shape[1]).to_numpy()
    return fn
