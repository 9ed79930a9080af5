#!/usr/bin/env python
"""Throughput benchmark of the batched Simple* solvers (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5] [--batch B]

One *step* = one pass of the hot path over one batch: for the default
workload (config C2, the configuration the metric is quoted on for one B200)
that is every one of the 23 MINPACK / More-Garbow-Hillstrom problems at B
perturbed initial guesses (u0 = u0c + 0.1*max(1,|u0c|_inf)*U(-1,1)^n) solved
with SimpleNewtonRaphson and with SimpleTrustRegion: 46 kernel launches,
23*2*B systems.  With N GPUs (torchrun, one process per GPU) every rank
solves its own contiguous shard of an N*B global batch (weak scaling, no
inter-GPU traffic in the solve); time is the max over ranks.

Reported on one JSON line (rank 0):
  value    systems solved/s, inputs resident in HBM, CUDA events on the
           launching stream, barrier + synchronize on both sides;
  e2e      same metric through the C-ABI with HOST buffers
           (nlk_solve_batch_host_async per job on 6 streams: pinned H2D,
           solve, D2H of every output inside the timing);
  roofline dominant kernel: algorithmic FP64 FLOPs (SURVEY.md §8d,
           paper_2403_16341_b200/flops.py) / its CUDA-event duration, against
           the FP64 FMA peak measured on this GPU by nlk_fp64_peak;
  cpu_baseline  the unmodified reference (nlkit, oracle/_ref) on the host
           cores with a process pool, on a bounded sample of the same inputs.
`--impl reference` times only the reference on the host cores.
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
def jobs_for(config, lo, hi):
    """[(problem_id, n, alg, Batch)] for rows [lo, hi) of each stream."""
    from paper_2403_16341_b200 import workloads as W
    out = []
    if config == "c2":
        for idx in range(1, 24):
            b = W.c2_suite(idx, lo, hi, 0.1)
            for alg in ("newton-raphson", "trust-region"):
                out.append((b.problem_id, b.n, alg, b))
    elif config == "c1":
        out.append(("quadratic", 2, "newton-raphson", W.c1_quadratic(lo, hi)))
    elif config == "c3":
        for n in (8, 16):
            b = W.c3_rosenbrock(n, lo, hi)
            for alg in ("broyden", "klement"):
                out.append((b.problem_id, n, alg, b))
    elif config == "c4":
        out.append(("test23/broyden-tridiagonal", 16, "dfsane", W.c4_tridiagonal(lo, hi)))
    elif config == "c5":
        b = W.c5_quadratic(lo, hi)
        algs = W.c5_algorithms(lo, hi)
        for k, alg in enumerate(W.C5_ALGS):
            sel = np.nonzero(algs == k)[0]
            out.append(("quadratic", 4, alg, W.Batch("quadratic", 4, b.u0[sel], b.p[sel], lo)))
    else:
        raise SystemExit(f"unknown config {config}")
    return out


WORKLOAD = {
    "c2": "C2: 23 MINPACK/MGH problems x B perturbed starts (sigma=0.1) x {SimpleNewtonRaphson, SimpleTrustRegion}",
    "c1": "C1: u^2 - p (n=2) x B parameter sets, SimpleNewtonRaphson",
    "c3": "C3: generalized Rosenbrock n=8/16 x B, u0~U[0,1)^n, {SimpleBroyden, SimpleKlement}",
    "c4": "C4: broyden-tridiagonal n=16 x B, u0=-1+0.1U(-1,1)^16, SimpleDFSane",
    "c5": "C5: u^2 - p (n=4) x B, algorithm = i mod 5 over all Simple* solvers",
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
    problem_id, n, alg, u0, p = args
    import nlkit
    from nlkit import problems as nlp
    fun = _nlkit_residual(nlp, problem_id, n)
    prob = nlkit.Problem(fun, u0, params=p if p is not None else np.zeros(0))
    with np.errstate(all="ignore"):
        if alg == "dfsane":
            from oracle import dfsane_ref
            res = dfsane_ref.run_dfsane(prob, nlkit.SolveOptions(), nlkit)
        else:
            res = nlkit.solvers.run_preset(alg, prob, nlkit.SolveOptions())
    return res.retcode.value


def cpu_reference_rate(jobs, per_job, cores=None):
    """Time the unmodified reference (process pool, one solve per task) on the
    first `per_job` systems of every job; falls back to the C++ oracle port."""
    cores = cores or os.cpu_count() or 1
    tasks = []
    for pid, n, alg, b in jobs:
        for i in range(min(per_job, len(b.u0))):
            tasks.append((pid, n, alg, b.u0[i], None if b.p is None else b.p[i]))
    ref = _ref_path()
    if ref is not None:
        import multiprocessing as mp
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        if ref not in sys.path:
            sys.path.insert(0, ref)
        with mp.get_context("fork").Pool(cores) as pool:
            pool.map(_ref_solve, tasks[: max(cores * 2, 16)], chunksize=1)  # warm-up
            t0 = time.perf_counter()
            pool.map(_ref_solve, tasks, chunksize=4)
            dt = time.perf_counter() - t0
        kind = "reference"
    else:
        from oracle import oracle as O
        t0 = time.perf_counter()
        for pid, n, alg, b in jobs:
            k = min(per_job, len(b.u0))
            O.solve_batch(pid, alg, b.u0[:k], None if b.p is None else b.p[:k], threads=cores)
        dt = time.perf_counter() - t0
        kind = "port"
    return {"value": len(tasks) / dt, "unit": "systems/s", "cores": cores, "kind": kind,
            "sample": f"first {per_job} systems of each of {len(jobs)} (problem, algorithm) "
                      f"jobs = {len(tasks)} solves, one Problem per system, fork pool",
            "seconds": dt}


# ---------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local_rank, dist):
    import torch
    from paper_2403_16341_b200 import _lib, flops, solvers, workloads as W

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = _lib.lib()
    B = args.batch
    lo, hi = rank * B, (rank + 1) * B
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
        jobs = [j for j in jobs if any(k in f"{j[0]}:{j[2]}" for k in keys)]

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

    def one_step(events=None):
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

    for _ in range(args.warmup):
        one_step()
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
    value = world * per_step_systems * args.steps / elapsed

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
    if args.e2e_steps > 0:
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
        e2e = {"value": world * per_step_systems / statistics.median(step_t),
               "value_mean": world * per_step_systems * args.e2e_steps / float(te.item()),
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

    result = {
        "metric": METRIC, "value": value, "unit": "systems/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "batch_per_job_per_gpu": B,
                   "jobs": len(prepared), "systems_per_step_per_gpu": per_step_systems,
                   "abstol": abstol, "maxiters": 1000,
                   "l2": f"inputs+outputs {hbm_bytes / 1e9:.2f} GB/step/GPU > 126 MB L2 (no flush needed)",
                   "parallelism": f"shard{world} (independent systems, no collective)"},
        "gpu_launches": len(prepared) * args.steps,
        "roofline": {"bound": "fp32" if f32 else "fp64", "achieved": achieved, "peak": fp64_peak,
                     "unit": "TFLOP/s", "frac": achieved / fp64_peak, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu, profiles/ncu_traffic.json)",
                     "algorithmic_bytes": flops.system_bytes(n, m, elem=esz) * prepared[jdom][5].shape[1],
                     "kernel": kernel_names[jdom], "launch_ms": launch_ms[jdom],
                     "flops_per_launch": F,
                     "peak_source": ("nlk_fp32_peak (FFMA chains" if f32 else "nlk_fp64_peak (DFMA chains")
                                    + ", measured in this run)",
                     "hbm_gbs": hbm_bytes / (elapsed / args.steps) / 1e9},
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    return result, stats, jobs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--batch", type=int, default=1 << 20, help="systems per job per GPU")
    ap.add_argument("--abstol", type=float, default=None,
                    help="default 1e-8 (f32 on the quadratics: 1e-6)")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="arithmetic type (f32: registered fp32 instances, C1/C3/C4/C5)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--streams", type=int, default=1,
                    help="device-resident step: jobs round-robin over this many streams")
    ap.add_argument("--cpu-sample", type=int, default=60, help="systems per job for the CPU leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stats", default=None, help="write per-launch stats JSON here")
    ap.add_argument("--only", default=None,
                    help="comma-separated substrings: keep only matching (problem, algorithm) jobs "
                         "(profiling aid; the default runs the whole workload)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        jobs = jobs_for(args.config, 0, max(args.cpu_sample, 1))
        rates = []
        for s in range(args.warmup + args.steps):
            r = cpu_reference_rate(jobs, args.cpu_sample)
            if s >= args.warmup:
                rates.append(r)
        v = statistics.median(x["value"] for x in rates)
        line = {"metric": METRIC, "value": v, "unit": "systems/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * statistics.median(x["seconds"] for x in rates),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": WORKLOAD[args.config], "abstol": 1e-8, "maxiters": 1000,
                           "parallelism": "host process pool"},
                "cpu_baseline": {k: rates[0][k] for k in ("kind", "cores", "sample")} | {"value": v,
                                                                                       "unit": "systems/s"},
                "e2e": {"value": v, "unit": "systems/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist = tdist
    result, stats, jobs = run_ours(args, rank, world, local_rank, dist)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_reference_rate(jobs, args.cpu_sample)
            cb.pop("seconds", None)
            result["cpu_baseline"] = cb
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
