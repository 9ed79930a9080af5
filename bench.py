#!/usr/bin/env python
"""Throughput benchmark of the batched Simple* solvers (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5] [--batch B | --global-batch G]

One *step* = one pass of the hot path over one batch: for the default
workload (config C2, the configuration the metric is quoted on for one B200)
that is every one of the 23 MINPACK / More-Garbow-Hillstrom problems at B
perturbed initial guesses (u0 = u0c + 0.1*max(1,|u0c|_inf)*U(-1,1)^n) solved
with SimpleNewtonRaphson and with SimpleTrustRegion: 46 library calls (52
kernel launches: the six closed-form jobs add the kernel that completes their
deferred systems), 23*2*B systems.  With N GPUs (torchrun, one process per GPU) every rank
solves its own contiguous shard: of an N*B batch per job (--batch, weak
scaling) or of a fixed G per job (--global-batch, strong scaling, e.g. C4's
10 M over 2/4/8 GPUs).  No inter-GPU traffic in the solve; time is the max
over ranks.

Reported on one JSON line (rank 0):
  value    systems solved/s, inputs resident in HBM, CUDA events on the
           launching stream, barrier + synchronize on both sides;
  e2e      same metric through the C-ABI with HOST buffers
           (nlk_solve_batch_host_async per job on 6 streams: pinned H2D,
           solve, D2H of every output inside the timing), max over ranks;
  roofline dominant kernel, bound chosen by its arithmetic intensity
           (algorithmic FLOPs / algorithmic HBM bytes, SURVEY.md §8d,
           paper_2403_16341_b200/flops.py) against the ridge point: FP64
           FLOP/s against the FP64 FMA peak measured in this run by
           nlk_fp64_peak, or HBM GB/s against MEASURED_PEAKS.json; both
           fractions are always reported;
  cpu_baseline  the unmodified reference (nlkit, oracle/_ref) on the host
           cores with a process pool, on a stratified sample of >= 20k
           systems of the same jobs (N = 1, rank 0);
  parity   those reference outputs against this arm's outputs for the same
           systems, bit for bit (u, resid, retcode, nsteps, nf, njac,
           nlinsolve), with the host fingerprint the reference's bits depend
           on (CPU, OpenBLAS core, glibc, numpy SIMD).
`--impl reference` times only the reference on the host cores: each step a
stratified sample (--cpu-sample systems per job) of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "systems solved/sec (fp64, 1M-100M batch) at 1/2/4/8 B200; % FP64 peak vs CPU ref"
ALG_ID = {"newton-raphson": 0, "trust-region": 1, "broyden": 2, "klement": 3, "dfsane": 4,
          "newton-backtracking": 5}


# ---------------------------------------------------------------- workloads
def iter_job_groups(config, lo, hi):
    """Yield, one input batch at a time, the [(problem_id, n, alg, Batch)]
    jobs that share it, for rows [lo, hi) of each stream."""
    from paper_2403_16341_b200 import workloads as W
    if config == "c2":
        for idx in range(1, 24):
            b = W.c2_suite(idx, lo, hi, 0.1)
            yield [(b.problem_id, b.n, alg, b) for alg in ("newton-raphson", "trust-region")]
    elif config == "c1":
        yield [("quadratic", 2, "newton-raphson", W.c1_quadratic(lo, hi))]
    elif config == "c3":
        for n in (8, 16):
            b = W.c3_rosenbrock(n, lo, hi)
            yield [(b.problem_id, n, alg, b) for alg in ("broyden", "klement")]
    elif config == "c4":
        yield [("test23/broyden-tridiagonal", 16, "dfsane", W.c4_tridiagonal(lo, hi))]
    elif config == "n16":
        b = W.c3_rosenbrock(16, lo, hi)
        yield [(b.problem_id, 16, alg, b) for alg in ("newton-raphson", "trust-region")]
        b = W.c4_tridiagonal(lo, hi)
        yield [(b.problem_id, 16, alg, b) for alg in ("newton-raphson", "trust-region")]
    elif config == "c5":
        b = W.c5_quadratic(lo, hi)
        algs = W.c5_algorithms(lo, hi)
        out = []
        for k, alg in enumerate(W.C5_ALGS):
            sel = np.nonzero(algs == k)[0]
            out.append(("quadratic", 4, alg, W.Batch("quadratic", 4, b.u0[sel], b.p[sel], lo)))
        yield out
    else:
        raise SystemExit(f"unknown config {config}")


def jobs_for(config, lo, hi):
    """[(problem_id, n, alg, Batch)] for rows [lo, hi) of each stream."""
    return [j for g in iter_job_groups(config, lo, hi) for j in g]


WORKLOAD = {
    "c2": "C2: 23 MINPACK/MGH problems x B perturbed starts (sigma=0.1) x {SimpleNewtonRaphson, SimpleTrustRegion}",
    "c1": "C1: u^2 - p (n=2) x B parameter sets, SimpleNewtonRaphson",
    "c3": "C3: generalized Rosenbrock n=8/16 x B, u0~U[0,1)^n, {SimpleBroyden, SimpleKlement}",
    "c4": "C4: broyden-tridiagonal n=16 x B, u0=-1+0.1U(-1,1)^16, SimpleDFSane",
    "c5": "C5: u^2 - p (n=4) x B, algorithm = i mod 5 over all Simple* solvers",
    "n16": "n=16 Newton/trust region: generalized Rosenbrock (C3 inputs) and broyden-tridiagonal "
           "(C4 inputs) x B, {SimpleNewtonRaphson, SimpleTrustRegion}",
}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU reference
def _ref_path():
    p = os.path.join(ROOT, "oracle", "_ref")
    return p if os.path.isdir(os.path.join(p, "nlkit")) else None


def _nlkit_residual(nlp, problem_id, n):
    if problem_id.startswith("test23/"):
        name = problem_id.split("/", 1)[1]
        for nm, fun, *_r in nlp._SUITE:
            if nm == name:
                return fun
    if problem_id == "generalized_rosenbrock":
        return nlp.generalized_rosenbrock(n).problem.residual
    if problem_id == "quadratic":
        return nlp.quadratic(tuple([1.0] * n)).problem.residual
    raise KeyError(problem_id)


def _ref_solve(args):
    """One system through the unmodified reference's public preset entry
    point (nlkit.solvers.run_preset, solvers.py:640-655).  Returns every
    per-system output the GPU arm returns: (retcode index, u bytes, resid,
    nsteps, nf, njac, nlinsolve)."""
    problem_id, n, alg, u0, p = args
    import nlkit
    from nlkit import problems as nlp
    fun = _nlkit_residual(nlp, problem_id, n)
    prob = nlkit.Problem(fun, u0, params=p if p is not None else np.zeros(0))
    with np.errstate(all="ignore"):
        if alg == "dfsane":  # no reference algorithm: builder-authored statement
            from oracle import dfsane_ref
            res = dfsane_ref.run_dfsane(prob, nlkit.SolveOptions(), nlkit)
        else:
            res = nlkit.solvers.run_preset(alg, prob, nlkit.SolveOptions())
    st = res.stats
    return (list(nlkit.RetCode).index(res.retcode),
            np.asarray(res.u_star, dtype=np.float64).tobytes(), float(res.resid_norm),
            int(st.nsteps), int(st.nf), int(st.njac), int(st.nlinsolve))


def stratified_rows(Bj, k, offset=0):
    """Systematic sample of k of Bj rows (every Bj/k-th, shifted by offset):
    the heavy-tailed iteration counts of a job are sampled in proportion."""
    k = max(1, min(k, Bj))
    idx = (np.arange(k, dtype=np.int64) * Bj) // k + offset
    return idx[idx < Bj]


def host_fingerprint():
    """What the reference's bits depend on: CPU, the
    OpenBLAS kernel family numpy/scipy dispatch to (getrf/getrs/gemv/dot
    orders), glibc (libm FMA ifunc variants) and numpy's SIMD dispatch
    (SVML exp/arctan)."""
    fp = {"cores": os.cpu_count()}
    try:
        info = {}
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k = k.strip()
            if k in ("model name", "cpu family", "model", "stepping") and k not in info:
                info[k] = v.strip()
        fp["cpu"] = info
    except OSError:
        pass
    try:
        fp["glibc"] = os.confstr("CS_GNU_LIBC_VERSION")
    except (ValueError, OSError):
        pass
    fp["numpy"] = np.__version__
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as F
        fp["numpy_simd"] = sorted(k for k, v in F.items() if v and k.startswith("AVX512"))
    except ImportError:
        pass
    try:
        import scipy
        import scipy.linalg  # noqa: F401  (loads scipy's OpenBLAS)
        import threadpoolctl
        fp["scipy"] = scipy.__version__
        fp["blas"] = [{"lib": os.path.basename(x.get("filepath", "")),
                       "version": x.get("version"), "core": x.get("architecture")}
                      for x in threadpoolctl.threadpool_info() if x.get("user_api") == "blas"]
    except ImportError:
        pass
    return fp


def cpu_reference_run(tasks, cores=None):
    """Run the unmodified reference (oracle/_ref) on `tasks` in a fork pool
    over the host cores, one run_preset per system; returns (outputs, seconds,
    kind).  Without oracle/_ref the C++ port of the path stands in."""
    cores = cores or os.cpu_count() or 1
    ref = _ref_path()
    if ref is not None:
        import multiprocessing as mp
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        if ref not in sys.path:
            sys.path.insert(0, ref)
        with mp.get_context("fork").Pool(cores) as pool:
            pool.map(_ref_solve, tasks[: max(cores * 2, 16)], chunksize=1)  # warm-up
            t0 = time.perf_counter()
            outs = pool.map(_ref_solve, tasks, chunksize=4)
            dt = time.perf_counter() - t0
        return outs, dt, "reference", cores
    from oracle import oracle as O
    outs = []
    t0 = time.perf_counter()
    for pid, n, alg, u0, p in tasks:
        r = O.solve_batch(pid, alg, u0[None, :], None if p is None else p[None, :], threads=1)
        outs.append((int(r["retcode"][0]), r["u"][0].tobytes(), float(r["resid"][0]),
                     int(r["nsteps"][0]), int(r["nf"][0]), int(r["njac"][0]),
                     int(r["nlinsolve"][0])))
    return outs, time.perf_counter() - t0, "port", 1


PARITY_FIELDS = ("retcode", "u", "resid", "nsteps", "nf", "njac", "nlinsolve")


def cpu_baseline_and_parity(prepared, per_job, compare=True):
    """The CPU leg of the GPU arm: the reference on a stratified sample of
    every job (per_job systems each), timed, and compared bit for bit with
    the GPU arm's outputs for the same systems (u and resid as bit patterns,
    retcode and the four counters exactly)."""
    tasks, gpu = [], []
    for pid, n, m, alg, h, u0, p, out, b in prepared:
        Bj = int(u0.shape[1])
        idx = stratified_rows(Bj, per_job)
        it = torch_index(idx, out["u"].device)
        gu = out["u"][:, it].t().contiguous().cpu().numpy()
        gr = out["resid"][it].cpu().numpy()
        grc = out["retcode"][it].cpu().numpy()
        gc = out["counters"][:, it].cpu().numpy()
        for j, i in enumerate(idx):
            tasks.append((pid, n, alg, b.u0[i], None if b.p is None else b.p[i]))
            gpu.append((int(grc[j]), gu[j].astype(np.float64).tobytes(),
                        float(gr[j]), int(gc[0, j]), int(gc[1, j]), int(gc[2, j]),
                        int(gc[3, j]), pid, alg, int(i)))
    outs, dt, kind, cores = cpu_reference_run(tasks)
    cb = {"value": len(tasks) / dt, "unit": "systems/s", "cores": cores, "kind": kind,
          "sample": f"stratified: every (B/{per_job})-th system of each of {len(prepared)} "
                    f"(problem, algorithm) jobs = {len(tasks)} solves, one run_preset per "
                    f"system, fork pool over {cores} host cores",
          "seconds": dt}
    if not compare:
        return cb, {"skipped": "fp32 arm: the reference computes in fp64 (fp32 is checked "
                               "against the fp64 oracle at 1e-4 in tests/test_gpu_fp32.py)"}
    by_field = {f: 0 for f in PARITY_FIELDS}
    mism, examples = 0, []
    pinned = unpinned = 0
    for g, r in zip(gpu, outs):
        bad = [f for k, f in enumerate(PARITY_FIELDS)
               if (g[k] != r[k] if f != "resid" else
                   np.float64(g[k]).tobytes() != np.float64(r[k]).tobytes())]
        if g[8] == "dfsane":
            unpinned += 1
        else:
            pinned += 1
        if bad:
            mism += 1
            for f in bad:
                by_field[f] += 1
            if len(examples) < 8:
                examples.append({"problem": g[7], "alg": g[8], "index": g[9], "fields": bad})
    parity = {"systems": len(tasks), "mismatches": mism, "fields": list(PARITY_FIELDS),
              "mismatches_by_field": by_field, "examples": examples,
              "against": kind + (" (nlkit, unmodified)" if kind == "reference" else ""),
              "systems_unpinned_dfsane": unpinned, "host": host_fingerprint()}
    return cb, parity


def torch_index(idx, device):
    import torch
    return torch.from_numpy(np.asarray(idx, dtype=np.int64)).to(device)


def reference_arm_samples(config, B, per_job, steps):
    """For each of `steps` steps, the (problem, algorithm) jobs of `config`
    at batch B per job, each reduced to a stratified sample of per_job
    systems shifted by one row per step (the steps cover different systems
    of the same workload).  Batches are generated one at a time."""
    from paper_2403_16341_b200 import workloads as W
    out = [[] for _ in range(steps)]
    for group in iter_job_groups(config, 0, B):
        for pid, n, alg, b in group:
            for s in range(steps):
                idx = stratified_rows(len(b.u0), per_job, s)
                out[s].append((pid, n, alg, W.Batch(b.problem_id, b.n, b.u0[idx].copy(),
                                                    None if b.p is None else b.p[idx].copy(), 0)))
        del group
    return out


def tasks_of(jobs):
    return [(pid, n, alg, b.u0[i], None if b.p is None else b.p[i])
            for pid, n, alg, b in jobs for i in range(len(b.u0))]


def e2e_via_devices(args, prepared, dist, dev, total_systems, world):
    """The e2e leg through the user-facing one-process sharder
    (sharding.solve_batch_devices): each job's host batch (numpy [B, n]) is
    split over the listed devices (--e2e-devices, e.g. "0,1,2,3"; under
    torchrun each rank lists its own GPU), pinned, solved and gathered into
    one host result buffer per job -- everything a user's call does, inside
    the timed region."""
    import torch
    from paper_2403_16341_b200 import sharding
    devices = [int(d) for d in args.e2e_devices.split(",")]
    host = [(pid, n, alg, np.ascontiguousarray(b.u0), None if b.p is None else np.ascontiguousarray(b.p))
            for pid, n, m, alg, h, u0, p, out, b in prepared]
    f32 = args.dtype == "f32"

    def step():
        for pid, n, alg, u0, p in host:
            sharding.solve_batch_devices(pid, u0, p, alg, devices=devices, n=n,
                                         dtype=torch.float32 if f32 else torch.float64)

    step()  # warm-up
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        step()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    esz = 4 if f32 else 8
    bi = sum((u0.size + (0 if p is None else p.size)) * esz for _, _, _, u0, p in host)
    bo = sum(len(u0) * ((n + 1) * esz + 1 + 16) for _, n, _, u0, _ in host)
    return {"value": total_systems * args.e2e_steps / float(te.item()), "unit": "systems/s",
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "steps": args.e2e_steps,
            "api": f"sharding.solve_batch_devices(devices={devices}) per job, numpy in/out"}


def rank_rows(batch, global_batch, world, rank):
    """Rows [lo, hi) of every job that this rank solves: a fixed global batch
    split evenly (strong scaling, workloads.shard_bounds) or `batch` rows per
    rank (weak scaling, rank r takes [r*batch, (r+1)*batch))."""
    if global_batch:
        from paper_2403_16341_b200.workloads import shard_bounds
        return shard_bounds(global_batch, world, rank)
    return rank * batch, (rank + 1) * batch


def _hbm_peak():
    """HBM GB/s denominator: the driver-measured copy bandwidth of this pool
    (MEASURED_PEAKS.json), else the profiling recipe's stated fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return float(json.load(open(p))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
        except (KeyError, ValueError):
            pass
    return 6650.0, "of fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local_rank, dist):
    import torch
    from paper_2403_16341_b200 import _lib, flops, solvers, workloads as W

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = _lib.lib()
    lo, hi = rank_rows(args.batch, args.global_batch, world, rank)
    B = hi - lo
    f32 = args.dtype == "f32"
    tdt = torch.float32 if f32 else torch.float64
    esz = 4 if f32 else 8
    # fp32 cannot reach 1e-8 on the parametrised quadratics (SURVEY.md §7:
    # MaxIters on ~95 %); their fp32 runs use 1e-6.  Generalized Rosenbrock's
    # root is exactly representable, so C3 keeps 1e-8 in fp32.
    abstol = args.abstol or (1e-6 if f32 and args.config in ("c1", "c5") else 1e-8)
    jobs = jobs_for(args.config, lo, hi)
    if args.only:
        keys = args.only.split(",")
        jobs = [j for j in jobs if any(k in f"{j[0]}:{j[2]}:n={j[1]}" for k in keys)]

    # device-resident SoA inputs (shared by the jobs of one problem) and outputs
    inputs, prepared = {}, []
    for pid, n, alg, b in jobs:
        key = id(b)
        if key not in inputs:
            u0 = torch.from_numpy(np.ascontiguousarray(b.u0.T)).to(dev, tdt)
            p = None if b.p is None else torch.from_numpy(np.ascontiguousarray(b.p.T)).to(dev, tdt)
            inputs[key] = (u0, p)
        u0, p = inputs[key]
        h, nn, m = _lib.problem_lookup(pid, n)
        Bj = u0.shape[1]
        out = {"u": torch.empty((n, Bj), dtype=tdt, device=dev),
               "resid": torch.empty(Bj, dtype=tdt, device=dev),
               "retcode": torch.empty(Bj, dtype=torch.int8, device=dev),
               "counters": torch.empty((4, Bj), dtype=torch.int32, device=dev)}
        prepared.append((pid, n, m, alg, h, u0, p, out, b))

    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    # --streams K: jobs round-robin over K streams (K = 1: one stream), so the
    # heavy-tailed end of one persistent launch overlaps the next launch
    side = [torch.cuda.Stream(dev) for _ in range(max(args.streams, 1) - 1)]
    lanes = [stream] + side

    launches = [1] * len(prepared)  # kernels per call (nlk_last_launches, read in warm-up)

    def one_step(events=None, count=False):
        if side:
            fork = torch.cuda.Event()
            fork.record(stream)
            for st_ in side:
                st_.wait_event(fork)
        for j, (pid, n, m, alg, h, u0, p, out, b) in enumerate(prepared):
            st_ = lanes[j % len(lanes)]
            if events is not None:
                events[j][0].record(st_)
            solvers.solve_batch_soa(h, ALG_ID[alg], u0, p, abstol, 1000, out=out,
                                    stream=st_.cuda_stream)
            if count:
                launches[j] = int(L.nlk_last_launches())
            if events is not None:
                events[j][1].record(st_)
        for st_ in side:
            join = torch.cuda.Event()
            join.record(st_)
            stream.wait_event(join)

    peak = ctypes.c_double()
    _lib.check((L.nlk_fp32_peak if f32 else L.nlk_fp64_peak)(
        1 << 16, ctypes.byref(peak), ctypes.c_void_p(sptr)))
    fp64_peak = peak.value

    for w in range(args.warmup):
        one_step(count=(w == 0))
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in prepared] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        start.record(stream)
        for s in range(args.steps):
            one_step(ev[s])
        end.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    elapsed = start.elapsed_time(end) / 1e3
    t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    per_step_systems = sum(int(x[5].shape[1]) for x in prepared)
    total_systems = per_step_systems
    if dist:
        ts_ = torch.tensor([float(per_step_systems)], dtype=torch.float64, device=dev)
        dist.all_reduce(ts_, op=dist.ReduceOp.SUM)
        total_systems = int(ts_.item())
    value = total_systems * args.steps / elapsed

    # per-launch durations (mean over steps) and the dominant kernel's roofline
    launch_ms = [statistics.mean(ev[s][j][0].elapsed_time(ev[s][j][1]) for s in range(args.steps))
                 for j in range(len(prepared))]
    jdom = int(np.argmax(launch_ms))
    pid, n, m, alg, h, u0, p, out, b = prepared[jdom]
    c = out["counters"]
    F = float(flops.system_flops(pid, n, alg, c[0], c[1], c[2], c[3]).sum())
    dom_s = launch_ms[jdom] / 1e3
    achieved = F / dom_s / 1e12
    total_flops = 0.0
    for (pid_, n_, m_, alg_, _h, _u0, _p, out_, _b) in prepared:
        cc = out_["counters"]
        total_flops += float(flops.system_flops(pid_, n_, alg_, cc[0], cc[1], cc[2], cc[3]).sum())
    kernel_names = [f"solve_kernel<{x[0]},n={x[1]},{x[3]}{',f32' if f32 else ''}>" for x in prepared]
    stats = {"per_launch_ms": dict(zip(kernel_names, [round(v, 4) for v in launch_ms])),
             "retcodes": {kernel_names[j]: np.bincount(prepared[j][7]["retcode"].cpu().numpy(),
                                                       minlength=6).tolist()
                          for j in range(len(prepared))},
             "step_fp64_tflops": total_flops / (elapsed / args.steps) / 1e12}
    hbm_bytes = sum(flops.system_bytes(x[1], x[2], elem=esz) * x[5].shape[1] for x in prepared)

    # ---- e2e through the C-ABI with host buffers
    e2e = None
    if args.e2e_steps > 0 and args.e2e_devices:
        e2e = e2e_via_devices(args, prepared, dist, dev, total_systems, world)
    elif args.e2e_steps > 0:
        # a job is handed to the library as `pieces` contiguous column chunks
        # (each its own asynchronous call) when there are fewer jobs than
        # streams, so that the copies of one chunk overlap the solve of another
        nst = int(os.environ.get("NLK_E2E_STREAMS", "6"))
        pieces = max(1, -(-nst // len(prepared)))
        host = []
        for pid_, n_, m_, alg_, h_, u0_, p_, out_, b_ in prepared:
            Bj = u0_.shape[1]
            bounds = np.linspace(0, Bj, pieces + 1).astype(int)
            for lo_, hi_ in zip(bounds[:-1], bounds[1:]):
                if hi_ <= lo_:
                    continue
                hu0 = u0_[:, lo_:hi_].contiguous().cpu().pin_memory()
                hp = None if p_ is None else p_[:, lo_:hi_].contiguous().cpu().pin_memory()
                Bc = int(hi_ - lo_)
                hout = (torch.empty((n_, Bc), dtype=tdt).pin_memory(),
                        torch.empty(Bc, dtype=tdt).pin_memory(),
                        torch.empty(Bc, dtype=torch.int8).pin_memory(),
                        torch.empty((4, Bc), dtype=torch.int32).pin_memory())
                host.append((h_, ALG_ID[alg_], Bc, hu0, hp, hout))

        # every job (chunk) enqueued through the asynchronous host-buffer entry
        # point, round-robin over the streams (copies of one overlap the solves
        # of others), one synchronisation per step
        e2e_streams = [torch.cuda.Stream(dev) for _ in range(nst)]

        def e2e_step():
            for j, (h_, a_, Bj, hu0, hp, (uo, ro, rc, cn)) in enumerate(host):
                _lib.check(L.nlk_solve_batch_host_async(
                    h_, a_, 1 if f32 else 0, Bj, hu0.data_ptr(), None if hp is None else hp.data_ptr(), abstol,
                    1000, uo.data_ptr(), ro.data_ptr(), rc.data_ptr(), cn[0].data_ptr(),
                    cn[1].data_ptr(), cn[2].data_ptr(), cn[3].data_ptr(),
                    e2e_streams[j % nst].cuda_stream))
            for st_ in e2e_streams:
                st_.synchronize()

        for _ in range(2):  # warm-up (allocations, first-touch, clocks after the idle setup)
            e2e_step()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        step_t = []
        for _ in range(args.e2e_steps):
            ts = time.perf_counter()
            e2e_step()
            step_t.append(time.perf_counter() - ts)
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        bi = sum((x[3].numel() + (0 if x[4] is None else x[4].numel())) * esz for x in host)
        bo = sum(x[5][0].numel() * esz + x[5][1].numel() * esz + x[5][2].numel() + x[5][3].numel() * 4
                 for x in host)
        # value: median step (robust to a one-off host hiccup); value_mean: all steps
        # value: all steps, max over ranks; value_median: the median step (rank 0)
        e2e = {"value": total_systems * args.e2e_steps / float(te.item()),
               "value_median": total_systems / statistics.median(step_t),
               "unit": "systems/s", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
               "steps": args.e2e_steps, "step_ms": [round(1e3 * t, 1) for t in step_t],
               "streams": nst, "calls_per_step": len(host)}

    # roofline.traffic: DRAM bytes of the dominant kernel from a committed ncu --set full
    # capture (profiles/ncu_traffic.json), scaled to this run's batch; null if none matches
    traffic = None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        t = json.load(open(tpath)).get(kernel_names[jdom])
        if t:
            traffic = t["dram_bytes"] * (prepared[jdom][5].shape[1] / t["batch"])

    # The bound follows the dominant kernel's arithmetic intensity: algorithmic
    # FLOPs per algorithmic HBM byte against the ridge point peak_flops /
    # peak_bytes.  Below the ridge (the n = 2/4 quadratics) the kernel is
    # HBM-bound and `achieved` is algorithmic GB/s; above it (every C2 job)
    # the FP64 (FP32) pipe bounds it.  Both fractions are reported.
    alg_bytes = flops.system_bytes(n, m, elem=esz) * prepared[jdom][5].shape[1]
    hbm_peak, hbm_src = _hbm_peak()
    ai = F / alg_bytes
    ridge = fp64_peak * 1e12 / (hbm_peak * 1e9)
    gbs = alg_bytes / dom_s / 1e9
    pipe = "fp32" if f32 else "fp64"
    hbm_bound = ai < ridge
    ncu = None
    npath = os.path.join(ROOT, "profiles", "ncu_pipe.json")
    if os.path.exists(npath):
        ncu = json.load(open(npath)).get(kernel_names[jdom])
    roofline = {
        "bound": "hbm" if hbm_bound else pipe,
        "achieved": gbs if hbm_bound else achieved,
        "peak": hbm_peak if hbm_bound else fp64_peak,
        "unit": "GB/s" if hbm_bound else "TFLOP/s",
        "frac": gbs / hbm_peak if hbm_bound else achieved / fp64_peak,
        "traffic": traffic,
        "traffic_unit": "DRAM bytes per launch (ncu, profiles/ncu_traffic.json)",
        "kernel": kernel_names[jdom], "launch_ms": launch_ms[jdom],
        "flops_per_launch": F, "algorithmic_bytes": alg_bytes,
        "arithmetic_intensity": ai, "ridge_flop_per_byte": ridge,
        f"frac_{pipe}": achieved / fp64_peak, "frac_hbm": gbs / hbm_peak,
        f"achieved_{pipe}_tflops": achieved, "achieved_hbm_gbs": gbs,
        f"peak_{pipe}_tflops": fp64_peak,
        f"peak_{pipe}_source": ("nlk_fp32_peak (FFMA chains" if f32 else "nlk_fp64_peak (DFMA chains")
                               + ", measured in this run)",
        "peak_hbm_gbs": hbm_peak, "peak_hbm_source": hbm_src,
        "ncu": ncu,
        "step_hbm_gbs": hbm_bytes / (elapsed / args.steps) / 1e9,
    }

    result = {
        "metric": METRIC, "value": value, "unit": "systems/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.global_batch else "weak", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "batch_per_job_per_gpu": B,
                   "global_batch_per_job": args.global_batch or args.batch * world,
                   "jobs": len(prepared), "systems_per_step_per_gpu": per_step_systems,
                   "abstol": abstol, "maxiters": 1000,
                   "l2": f"inputs+outputs {hbm_bytes / 1e9:.2f} GB/step/GPU > 126 MB L2 (no flush needed)",
                   "parallelism": f"shard{world} (independent systems, no collective)"},
        "gpu_launches": sum(launches) * args.steps,
        "roofline": roofline,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    # CPU leg (rank 0, N = 1): the unmodified reference on a stratified sample
    # of every job, timed, and compared bit for bit with this arm's outputs
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        per_job = max(1, -(-args.parity_systems // len(prepared)))
        cb, parity = cpu_baseline_and_parity(prepared, per_job, compare=not f32)
        cb.pop("seconds", None)
        result["cpu_baseline"] = cb
        result["parity"] = parity
    return result, stats, jobs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "n16"])
    ap.add_argument("--batch", type=int, default=1 << 20, help="systems per job per GPU")
    ap.add_argument("--abstol", type=float, default=None,
                    help="default 1e-8 (f32 on the quadratics: 1e-6)")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="arithmetic type (f32: registered fp32 instances, C1/C3/C4/C5)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-devices", default=None,
                    help="e2e leg through sharding.solve_batch_devices over these devices "
                         "(comma-separated ids; default: the C-ABI async host-buffer path)")
    ap.add_argument("--streams", type=int, default=1,
                    help="device-resident step: jobs round-robin over this many streams")
    ap.add_argument("--global-batch", type=int, default=None,
                    help="strong scaling: systems per job over ALL GPUs, split evenly "
                         "(default: --batch per job per GPU, weak scaling)")
    ap.add_argument("--parity-systems", type=int, default=20000,
                    help="GPU arm: reference systems (stratified over the jobs) timed on the "
                         "host and compared bit for bit with the GPU outputs")
    ap.add_argument("--cpu-sample", type=int, default=60,
                    help="reference arm: stratified systems per job per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stats", default=None, help="write per-launch stats JSON here")
    ap.add_argument("--only", default=None,
                    help="comma-separated substrings: keep only matching (problem, algorithm) jobs "
                         "(profiling aid; the default runs the whole workload)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # functional test of the N > 1 path on a one-GPU box (tests/ and DESIGN §5):
    # NLK_BENCH_DEVICE pins every rank to one device, NLK_BENCH_BACKEND=gloo
    # replaces NCCL (which refuses two ranks on one GPU).  Never a measurement.
    if os.environ.get("NLK_BENCH_DEVICE") is not None:
        local_rank = int(os.environ["NLK_BENCH_DEVICE"])

    if args.impl == "reference":
        if rank != 0:
            return 0
        steps = args.warmup + args.steps
        B = args.global_batch or args.batch
        samples = reference_arm_samples(args.config, B, args.cpu_sample, steps)
        rates = []
        for s in range(steps):
            tasks = tasks_of(samples[s])
            _outs, dt, kind, cores = cpu_reference_run(tasks)
            if s >= args.warmup:
                rates.append((len(tasks) / dt, dt, len(tasks)))
        v = statistics.median(x[0] for x in rates)
        sample = (f"stratified: {args.cpu_sample} systems (every B/{args.cpu_sample}-th, shifted "
                  f"one row per step) of each of {len(samples[0])} (problem, algorithm) jobs at "
                  f"B = {B} = {rates[0][2]} solves per step, one run_preset per system, fork pool")
        line = {"metric": METRIC, "value": v, "unit": "systems/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * statistics.median(x[1] for x in rates),
                "higher_is_better": True, "scaling": "strong" if args.global_batch else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": WORKLOAD[args.config], "batch_per_job": B,
                           "abstol": 1e-8, "maxiters": 1000,
                           "parallelism": f"host process pool ({cores} processes)"},
                "cpu_baseline": {"kind": kind, "cores": cores, "sample": sample, "value": v,
                                 "unit": "systems/s", "host": host_fingerprint()},
                "e2e": {"value": v, "unit": "systems/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        backend = os.environ.get("NLK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            tdist.init_process_group(backend)
        dist = tdist
    result, stats, jobs = run_ours(args, rank, world, local_rank, dist)
    if rank == 0:
        if args.stats:
            with open(args.stats, "w") as fh:
                json.dump({"result": result, "stats": stats}, fh, indent=1)
        print(json.dumps(result), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
