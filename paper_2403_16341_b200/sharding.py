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
    (default: every visible GPU; a device may repeat).  Per slice, on a stream
    of its own device and all asynchronous: the row-major slice is staged in
    pinned memory and copied to the device as is, transposed to the kernels'
    SoA layout there, solved (``nlk_solve_batch``), and every output is
    transposed back on the device and copied straight into its rows of ONE
    pinned host result per field -- no host-side transposes, no inter-GPU
    traffic, no collective.  Returns a dict of host (numpy) arrays with the
    fields of ``FIELDS`` for all B systems, in order; the arrays are views
    of the pinned result buffers.
    """
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
        p = np.ascontiguousarray(p)
    if algorithm == "polyalgorithm" or algorithm is None:
        raise NotImplementedError("solve_batch_devices runs one algorithm; "
                                  "use solve_batch per device for the poly-algorithm")
    alg = solvers.resolve_algorithm(algorithm).kernel
    # pinned staging of the inputs and pinned results, row-major as the caller's
    hu0 = torch.empty((B, nn), dtype=dtype, pin_memory=True)
    hu0.copy_(torch.from_numpy(u0))
    hp = None
    if m:
        hp = torch.empty((B, m), dtype=dtype, pin_memory=True)
        hp.copy_(torch.from_numpy(p))
    res = {"u": torch.empty((B, nn), dtype=dtype, pin_memory=True),
           "resid": torch.empty(B, dtype=dtype, pin_memory=True),
           "retcode": torch.empty(B, dtype=torch.int8, pin_memory=True),
           "counters": torch.empty((B, 4), dtype=torch.int32, pin_memory=True)}
    streams = []
    keep = []  # device tensors alive until their stream is synchronised
    for r, dev in enumerate(devices):
        lo, hi = shard_bounds(B, len(devices), r)
        if hi <= lo:
            continue
        d = torch.device("cuda", dev)
        with torch.cuda.device(d):
            st = torch.cuda.Stream(d)
            with torch.cuda.stream(st):
                du0 = hu0[lo:hi].to(d, non_blocking=True).t().contiguous()
                dp = None if hp is None else hp[lo:hi].to(d, non_blocking=True).t().contiguous()
                out = solvers.solve_batch_soa(handle, alg, du0, dp, options.abstol,
                                              options.maxiters, stream=st.cuda_stream)
                res["u"][lo:hi].copy_(out["u"].t().contiguous(), non_blocking=True)
                res["resid"][lo:hi].copy_(out["resid"], non_blocking=True)
                res["retcode"][lo:hi].copy_(out["retcode"], non_blocking=True)
                res["counters"][lo:hi].copy_(out["counters"].t().contiguous(), non_blocking=True)
        streams.append(st)
        keep.append((du0, dp, out))
    for st in streams:
        st.synchronize()
    del keep
    c = res["counters"].numpy()
    return {"u": res["u"].numpy(), "resid": res["resid"].numpy(),
            "retcode": res["retcode"].numpy(), "nsteps": c[:, 0], "nf": c[:, 1],
            "njac": c[:, 2], "nlinsolve": c[:, 3]}
