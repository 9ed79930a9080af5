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


def solve_batch_devices(problem, u0, p=None, algorithm="newton-raphson", options=None,
                        devices=None, dtype=torch.float64, n=None):
    """One host batch sharded over the GPUs of this process.

    ``u0`` [B, n] and ``p`` [B, m] are host arrays.  The batch is split into
    contiguous even slices (``shard_bounds``), one per entry of ``devices``
    (default: every visible GPU; a device may repeat).  Each slice is copied
    to pinned memory in SoA layout and handed to ``nlk_solve_batch_host_async``
    on a stream of its own device -- staging H2D, the solve and the D2H of the
    results, all asynchronous -- so the GPUs run side by side with no
    inter-GPU traffic and every result lands in host memory.  Returns a dict
    of host arrays with the fields of ``FIELDS`` for all B systems, in order.
    """
    import ctypes

    from . import _lib, solvers
    from .core import SolveOptions

    options = options or SolveOptions()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the batched solver has no CPU fallback")
    devices = list(range(torch.cuda.device_count())) if devices is None else list(devices)
    if not devices:
        raise ValueError("devices is empty")
    dtype = {"f64": torch.float64, "f32": torch.float32}.get(dtype, dtype)
    npdt = np.float64 if dtype == torch.float64 else np.float32
    u0 = np.ascontiguousarray(np.asarray(u0, dtype=npdt))
    if u0.ndim == 1:
        u0 = u0[None, :]
    B, nn = u0.shape
    pid, n_req = solvers.resolve_problem(problem, n or nn)
    handle, n_reg, m = _lib.problem_lookup(pid, n_req or nn)
    if nn != n_reg:
        raise ValueError(f"{pid}: u0 has {nn} columns, the problem has n={n_reg}")
    if m:
        if p is None:
            p = getattr(problem, "params", None)
        if p is None:
            raise ValueError(f"{pid} needs parameters p [B, {m}]")
        p = np.asarray(p, dtype=npdt)
        p = np.broadcast_to(p[None, :], (B, m)) if p.ndim == 1 else p
        if p.shape != (B, m):
            raise ValueError(f"p must be [{B}, {m}], got {p.shape}")
    if algorithm == "polyalgorithm" or algorithm is None:
        raise NotImplementedError("solve_batch_devices runs one algorithm; "
                                  "use solve_batch per device for the poly-algorithm")
    alg = solvers.resolve_algorithm(algorithm).kernel
    L = _lib.lib()
    code = 0 if dtype == torch.float64 else 1
    jobs = []
    for r, dev in enumerate(devices):
        lo, hi = shard_bounds(B, len(devices), r)
        if hi <= lo:
            continue
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        hu0 = pin(u0[lo:hi].T)
        hp = pin(p[lo:hi].T) if m else None
        k = hi - lo
        out = {"u": torch.empty((nn, k), dtype=dtype).pin_memory(),
               "resid": torch.empty(k, dtype=dtype).pin_memory(),
               "retcode": torch.empty(k, dtype=torch.int8).pin_memory(),
               "counters": torch.empty((4, k), dtype=torch.int32).pin_memory()}
        with torch.cuda.device(dev):
            st = torch.cuda.Stream(dev)
            c = out["counters"]
            _lib.check(L.nlk_solve_batch_host_async(
                handle, alg, code, k, hu0.data_ptr(), None if hp is None else hp.data_ptr(),
                float(options.abstol), int(options.maxiters), out["u"].data_ptr(),
                out["resid"].data_ptr(), out["retcode"].data_ptr(), c[0].data_ptr(),
                c[1].data_ptr(), c[2].data_ptr(), c[3].data_ptr(), ctypes.c_void_p(st.cuda_stream)))
        jobs.append((lo, hi, st, out, hu0, hp))
    res = {"u": np.empty((B, nn), dtype=npdt), "resid": np.empty(B, dtype=npdt),
           "retcode": np.empty(B, dtype=np.int8)}
    for f in ("nsteps", "nf", "njac", "nlinsolve"):
        res[f] = np.empty(B, dtype=np.int32)
    for lo, hi, st, out, _hu0, _hp in jobs:
        st.synchronize()
        res["u"][lo:hi] = out["u"].numpy().T
        res["resid"][lo:hi] = out["resid"].numpy()
        res["retcode"][lo:hi] = out["retcode"].numpy()
        for j, f in enumerate(("nsteps", "nf", "njac", "nlinsolve")):
            res[f][lo:hi] = out["counters"][j].numpy()
    return res
