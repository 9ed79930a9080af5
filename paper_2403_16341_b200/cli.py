"""Benchmark command line with the reference's commands and CSV contract
(nlkit/cli.py), every solve on the B200.

    python -m paper_2403_16341_b200.cli solve <problem> <algorithm> [--abstol F] [--maxiters N]
    python -m paper_2403_16341_b200.cli wp --problems ... --algorithms ... --tols 1e-2..1e-10
                                          --reps K --out FILE [--batch B]
    python -m paper_2403_16341_b200.cli scaling --family generalized_rosenbrock --sizes 2,4,8
                                          --algorithms ... --out FILE [--batch B]
    python -m paper_2403_16341_b200.cli list problems|algorithms

Same headers (cli.py:33-35), same tolerance grammar (`_parse_tols`,
cli.py:88-108), same warm-up + median-of-reps timing (cli.py:111-131), same
exit codes (solve: 0 success / 1 not success / 2 unknown problem).
``--backend b200`` is accepted for scripts written against a reference with
a backend switch; it is the only backend.  ``--batch B`` (default 1) times one
launch of B copies of the cell's system and reports runtime_ns per system —
the batched throughput the GPU exists for; B = 1 is the reference's per-solve
latency.  ``resid_inf`` is ‖f(u*)‖∞ at the returned iterate, evaluated on the
device by the solve kernel (the reference re-evaluates the same float
residual at the same point, cli.py:62-64: the same value).
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import os
import statistics
import sys
import time
from dataclasses import dataclass

import numpy as np

from . import problems, solvers
from .core import RetCode, SolveOptions, result_to_json

WP_HEADER = ["problem", "algorithm", "abstol", "runtime_ns", "resid_inf",
             "retcode", "nf", "njac", "nlinsolve"]
SCALING_HEADER = ["size", "algorithm", "runtime_ns", "resid_inf", "retcode"]


@dataclass(frozen=True)
class BenchConfig:
    """cli.py:38-56: problems x algorithms x tolerances."""

    problems: tuple
    algorithms: tuple
    tols: tuple
    reps: int = 5
    maxiters: int = 1000
    seed: int = 0
    jobs: int = 1
    out: str = "-"
    batch: int = 1

    def __post_init__(self):
        if any(b >= a for a, b in zip(self.tols, self.tols[1:])) or not self.tols:
            raise ValueError("tolerance grid must be strictly decreasing")
        if self.reps < 1:
            raise ValueError("reps must be >= 1")
        if self.batch < 1:
            raise ValueError("batch must be >= 1")


def _seed(config_seed):
    env = os.environ.get("NLKIT_SEED")
    return int(env) if env is not None else config_seed


def _parse_tols(spec):
    """Comma list, or a decade range 'hi..lo' (cli.py:88-108)."""
    if ".." in spec:
        lo_s, hi_s = spec.split("..")
        start, stop = float(lo_s), float(hi_s)
        if not stop < start:
            raise ValueError("tolerance range must be strictly decreasing")
        e0, e1 = math.log10(start), math.log10(stop)
        if abs(e0 - round(e0)) < 1e-9 and abs(e1 - round(e1)) < 1e-9:
            return [10.0 ** e for e in range(round(e0), round(e1) - 1, -1)]
        tols, t = [], start
        while t >= stop * (1 - 1e-12):
            tols.append(t)
            t /= 10.0
        return tols
    tols = [float(t) for t in spec.split(",")]
    if any(b >= a for a, b in zip(tols, tols[1:])):
        raise ValueError("tolerance grid must be strictly decreasing")
    return tols


def _timed_batch(problem, algorithm, options, batch):
    """One solve of `batch` copies of `problem`; returns (ns, BatchResult)."""
    import torch
    u0 = np.broadcast_to(problem.u0, (batch, problem.n))
    p = None if problem.params.size == 0 else np.broadcast_to(problem.params,
                                                              (batch, problem.params.size))
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    r = solvers.solve_batch(problem, u0, p, algorithm, options, n=problem.n)
    torch.cuda.synchronize()
    return time.perf_counter_ns() - t0, r


def _cell(problem, algorithm, abstol, maxiters, reps, seed, batch):
    options = SolveOptions(abstol=abstol, maxiters=maxiters)
    if batch == 1:
        solvers.run_preset(algorithm, problem, options, seed)  # warm-up (cli.py:114)
        times, result = [], None
        for _ in range(reps):
            t0 = time.perf_counter_ns()
            result = solvers.run_preset(algorithm, problem, options, seed)
            times.append(time.perf_counter_ns() - t0)
        return int(statistics.median(times)), result
    _timed_batch(problem, algorithm, options, batch)  # warm-up
    times, r = [], None
    for _ in range(reps):
        ns, r = _timed_batch(problem, algorithm, options, batch)
        times.append(ns / batch)
    return int(statistics.median(times)), r.result(0)


def run_wp(config):
    """cli.py:134-147; returns the CSV rows."""
    rows = []
    for pid in config.problems:
        desc = problems.get_problem(pid)
        for alg in config.algorithms:
            for tol in config.tols:
                ns, res = _cell(desc.problem, alg, tol, config.maxiters, config.reps,
                                config.seed, config.batch)
                rows.append({"problem": desc.id, "algorithm": alg, "abstol": repr(tol),
                             "runtime_ns": ns, "resid_inf": repr(float(res.resid_norm)),
                             "retcode": res.retcode.value, "nf": res.stats.nf,
                             "njac": res.stats.njac, "nlinsolve": res.stats.nlinsolve})
    return rows


def _write_csv(path, header, rows):
    fh = open(path, "w", newline="") if path != "-" else sys.stdout
    try:
        w = csv.DictWriter(fh, fieldnames=header)
        w.writeheader()
        w.writerows(rows)
    finally:
        if path != "-":
            fh.close()


# Reference presets and problems that exist in nlkit (solvers.py:610-637,
# 640-655; problems.py:390-474) but deliberately have no batched kernel: they
# are not "unknown" (exit 2) but "not ported" (exit 3, EXIT_NOT_PORTED).
EXIT_NOT_PORTED = 3
REFERENCE_ONLY_PRESETS = ("newton-fd", "newton-sparse", "newton-sparse-fd", "newton-krylov",
                          "newton-krylov-ilu0", "trust-region-nw", "levenberg-marquardt",
                          "lm-cholesky", "lm-geodesic", "halley", "potra-ptak",
                          "broyden-true-jac", "lbroyden", "pseudo-transient")
REFERENCE_ONLY_PROBLEMS = ("brusselator2d",)


def cmd_solve(args):
    if args.problem.split("?", 1)[0] in REFERENCE_ONLY_PROBLEMS:
        print(f"error: reference problem {args.problem!r} has no device residual "
              "(n = 2N^2 is outside the batched small-system path; not ported)", file=sys.stderr)
        return EXIT_NOT_PORTED
    if args.algorithm in REFERENCE_ONLY_PRESETS:
        print(f"error: reference preset {args.algorithm!r} has no batched GPU kernel "
              "(not ported)", file=sys.stderr)
        return EXIT_NOT_PORTED
    try:
        desc = problems.get_problem(args.problem)
    except KeyError as exc:
        print(f"error: {exc.args[0]}", file=sys.stderr)
        return 2
    options = SolveOptions(abstol=args.abstol, maxiters=args.maxiters)
    try:
        t0 = time.perf_counter_ns()
        result = solvers.run_preset(args.algorithm, desc.problem, options)
    except KeyError as exc:
        print(f"error: {exc.args[0]}", file=sys.stderr)
        return 2
    result.stats.wall_time = (time.perf_counter_ns() - t0) / 1e9
    payload = json.loads(result_to_json(result))
    payload["problem"] = desc.id
    payload["algorithm"] = args.algorithm
    payload["resid_inf_measured"] = float(result.resid_norm)
    print(json.dumps(payload))
    return 0 if result.retcode == RetCode.SUCCESS else 1


def cmd_wp(args):
    config = BenchConfig(problems=tuple(args.problems.split(",")),
                         algorithms=tuple(args.algorithms.split(",")),
                         tols=tuple(_parse_tols(args.tols)), reps=args.reps,
                         maxiters=args.maxiters, seed=_seed(args.seed), jobs=args.jobs,
                         out=args.out, batch=args.batch)
    _write_csv(config.out, WP_HEADER, run_wp(config))
    return 0


def cmd_scaling(args):
    if args.family != "generalized_rosenbrock":
        # brusselator2d (n = 2N^2) is outside the batched small-system kernels
        print(f"error: unknown or unsupported family {args.family!r}", file=sys.stderr)
        return 2
    rows = []
    for size in (int(s) for s in args.sizes.split(",")):
        desc = problems.generalized_rosenbrock(size)
        for alg in args.algorithms.split(","):
            ns, res = _cell(desc.problem, alg, args.abstol, args.maxiters, 1, None, args.batch)
            rows.append({"size": size, "algorithm": alg, "runtime_ns": ns,
                         "resid_inf": repr(float(res.resid_norm)),
                         "retcode": res.retcode.value})
    _write_csv(args.out, SCALING_HEADER, rows)
    return 0


def cmd_list(args):
    if args.what == "problems":
        for desc in problems.list_problems():
            print(f"{desc.id}\tn={desc.n}\t[{','.join(sorted(desc.tags))}]")
    else:
        for name in solvers.list_algorithms():
            print(name)
    return 0


def build_parser():
    parser = argparse.ArgumentParser(prog="nlk-b200", description="batched B200 solver benchmarks")
    parser.add_argument("--backend", choices=["b200"], default="b200")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("solve", help="run one solve, print JSON result")
    p.add_argument("problem")
    p.add_argument("algorithm")
    p.add_argument("--abstol", type=float, default=1e-8)
    p.add_argument("--maxiters", type=int, default=1000)
    p.set_defaults(func=cmd_solve)

    p = sub.add_parser("wp", help="work-precision sweep to CSV")
    p.add_argument("--problems", required=True)
    p.add_argument("--algorithms", required=True)
    p.add_argument("--tols", default="1e-2..1e-10")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--maxiters", type=int, default=1000)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--jobs", type=int, default=1)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--backend", choices=["b200"], default="b200")
    p.add_argument("--out", default="-")
    p.set_defaults(func=cmd_wp)

    p = sub.add_parser("scaling", help="problem-size scaling runs to CSV")
    p.add_argument("--family", required=True)
    p.add_argument("--sizes", required=True)
    p.add_argument("--algorithms", required=True)
    p.add_argument("--abstol", type=float, default=1e-6)
    p.add_argument("--maxiters", type=int, default=1000)
    p.add_argument("--timeout-s", type=float, default=600.0)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--backend", choices=["b200"], default="b200")
    p.add_argument("--out", default="-")
    p.set_defaults(func=cmd_scaling)

    p = sub.add_parser("list", help="list problems or algorithms")
    p.add_argument("what", choices=["problems", "algorithms"])
    p.set_defaults(func=cmd_list)
    return parser


def main(argv=None):
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
