"""Generate the golden parity fixtures from the UNMODIFIED reference (nlkit).

Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

For every case it solves a bounded sample of a BASELINE.json configuration
with ``nlkit.solvers.run_preset`` (one Problem per system, exactly as a
reference user would) and stores inputs and outputs bit-exactly:

  <case>/u0, <case>/p, <case>/u, <case>/resid, <case>/retcode, <case>/nsteps,
  <case>/nf, <case>/njac, <case>/nlinsolve, <case>/sensitive

``sensitive`` marks systems whose (retcode, nsteps) change when the float
residual is nudged by one ulp in either direction: their
outcome is decided by roundoff, so parity gates exact retcode/nsteps only
outside this mask.  DFSane has no reference implementation; its fixtures come
from the builder-authored oracle/dfsane_ref.py run on nlkit's own types.

Residual fixtures (``residuals.npz``) hold the reference's float residual and
dual-number Jacobian at random points for every registered problem.
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
NLKIT_REF = os.environ.get("NLKIT_REF", "/root/reference/pkg/src")
sys.path.insert(0, NLKIT_REF)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import nlkit  # noqa: E402
from nlkit import problems as nlp  # noqa: E402
from nlkit import autodiff  # noqa: E402
from nlkit.errors import NonFiniteValue  # noqa: E402

from oracle import dfsane_ref  # noqa: E402
from paper_2403_16341_b200 import workloads as W  # noqa: E402

RC_INDEX = {rc: i for i, rc in enumerate(nlkit.RetCode)}


def nlkit_residual(problem_id, n):
    if problem_id.startswith("test23/"):
        name = problem_id.split("/", 1)[1]
        for (nm, fun, *_r) in nlp._SUITE:
            if nm == name:
                return fun
        raise KeyError(name)
    if problem_id == "generalized_rosenbrock":
        return nlp.generalized_rosenbrock(n).problem.residual
    if problem_id == "quadratic":
        return nlp.quadratic(tuple([1.0] * n)).problem.residual
    raise KeyError(problem_id)


def _nudge(fun, direction):
    def wrapped(u, theta):
        out = fun(u, theta)
        arr = np.asarray(out)
        if arr.dtype == np.float64:
            return np.nextafter(arr, direction)
        return out
    return wrapped


def _solve(args):
    problem_id, n, alg, u0, p, abstol, maxiters, nudge = args
    fun = nlkit_residual(problem_id, n)
    if nudge:
        fun = _nudge(fun, nudge)
    prob = nlkit.Problem(fun, u0, params=p if p is not None else np.zeros(0))
    opts = nlkit.SolveOptions(abstol=abstol, maxiters=maxiters)
    with np.errstate(all="ignore"):
        if alg == "dfsane":
            res = dfsane_ref.run_dfsane(prob, opts, nlkit)
        else:
            res = nlkit.solvers.run_preset(alg, prob, opts)
    st = res.stats
    return (np.asarray(res.u_star, dtype=float), float(res.resid_norm), RC_INDEX[res.retcode],
            st.nsteps, st.nf, st.njac, st.nlinsolve)


def run_case(pool, batch, alg, abstol=1e-8, maxiters=1000, mask=True):
    B = batch.u0.shape[0]
    p = batch.p
    jobs = [(batch.problem_id, batch.n, alg, batch.u0[i], None if p is None else p[i],
             abstol, maxiters, 0.0) for i in range(B)]
    res = pool.map(_solve, jobs, chunksize=4)
    out = {
        "u0": batch.u0, "p": p if p is not None else np.zeros((B, 0)),
        "u": np.stack([r[0] for r in res]),
        "resid": np.array([r[1] for r in res]),
        "retcode": np.array([r[2] for r in res], np.int8),
        "nsteps": np.array([r[3] for r in res], np.int32),
        "nf": np.array([r[4] for r in res], np.int32),
        "njac": np.array([r[5] for r in res], np.int32),
        "nlinsolve": np.array([r[6] for r in res], np.int32),
    }
    sens = np.zeros(B, bool)
    if mask:
        for direction in (np.inf, -np.inf):
            jobs2 = [j[:7] + (direction,) for j in jobs]
            res2 = pool.map(_solve, jobs2, chunksize=4)
            for i, r in enumerate(res2):
                if r[2] != out["retcode"][i] or r[3] != out["nsteps"][i]:
                    sens[i] = True
    out["sensitive"] = sens
    return out


def cases():
    """(file, case name, batch, alg) — bounded samples of configs C1-C5."""
    yield "c1", "c1/newton-raphson", W.c1_quadratic(0, 1024), "newton-raphson"
    for alg in ("trust-region", "broyden", "klement", "dfsane", "newton-backtracking"):
        yield "c1", f"c1/{alg}", W.c1_quadratic(0, 256), alg
    for idx in range(1, 24):
        name = W.problems.SUITE[idx - 1][0]
        for alg in ("newton-raphson", "trust-region"):
            yield "c2", f"c2/{name}/{alg}/s0.1", W.c2_suite(idx, 0, 48, 0.1), alg
            yield "c2", f"c2/{name}/{alg}/s1.0", W.c2_suite(idx, 0, 16, 1.0), alg
        for alg in ("broyden", "klement", "dfsane", "newton-backtracking"):
            yield "c2", f"c2/{name}/{alg}/s0.1", W.c2_suite(idx, 0, 12, 0.1), alg
    for n in (8, 16):
        for alg in ("broyden", "klement", "newton-raphson", "trust-region", "dfsane"):
            yield "c3", f"c3/n{n}/{alg}", W.c3_rosenbrock(n, 0, 96), alg
    for alg in ("dfsane", "newton-raphson", "trust-region", "broyden", "klement"):
        B = 256 if alg == "dfsane" else 48
        yield "c4", f"c4/{alg}", W.c4_tridiagonal(0, B), alg
    b = W.c5_quadratic(0, 1000)
    algs = W.c5_algorithms(0, 1000)
    for k, alg in enumerate(W.C5_ALGS):
        sel = np.nonzero(algs == k)[0]
        sub = W.Batch(b.problem_id, b.n, b.u0[sel], b.p[sel], 0)
        yield "c5", f"c5/{alg}", sub, alg


def residual_fixtures():
    rng = np.random.default_rng(77)
    ids = [(f"test23/{s[0]}", s[1], s[2]) for s in W.problems.SUITE]
    ids += [("generalized_rosenbrock", 8, None), ("generalized_rosenbrock", 16, None),
            ("quadratic", 2, None), ("quadratic", 4, None),
            ("test23/broyden-tridiagonal", 16, -np.ones(16))]
    out, manifest = {}, []
    for pid, n, start in ids:
        fun = nlkit_residual(pid, n)
        K = 48
        if start is None:
            X = rng.uniform(-2, 2, (K, n))
        else:
            sc = max(1.0, float(np.max(np.abs(start))))
            X = np.concatenate([start + 0.1 * sc * rng.uniform(-1, 1, (K // 2, n)),
                                start + 1.0 * sc * rng.uniform(-1, 1, (K // 2, n))])
        P = rng.uniform(0.5, 10, (K, n)) if pid == "quadratic" else np.zeros((K, 0))
        F = np.empty((K, n))
        J = np.full((K, n, n), np.nan)
        ok = np.zeros(K, bool)
        for k in range(K):
            with np.errstate(all="ignore"):
                F[k] = np.asarray(fun(X[k], P[k]), dtype=float)
                try:
                    J[k] = autodiff.dense_jacobian(fun, X[k], P[k])
                    ok[k] = True
                except NonFiniteValue:
                    ok[k] = False
        key = f"{pid}|{n}"
        out[key + "/x"], out[key + "/p"], out[key + "/f"] = X, P, F
        out[key + "/J"], out[key + "/ok"] = J, ok
        manifest.append({"key": key, "problem_id": pid, "n": n})
    return out, manifest


def main():
    t0 = time.time()
    files, manifest = {}, []
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for fname, case, batch, alg in cases():
            t1 = time.time()
            r = run_case(pool, batch, alg)
            d = files.setdefault(fname, {})
            for k, v in r.items():
                d[f"{case}/{k}"] = v
            manifest.append({"file": fname, "case": case, "problem_id": batch.problem_id,
                             "n": batch.n, "alg": alg, "B": int(batch.u0.shape[0]),
                             "sensitive": int(r["sensitive"].sum()),
                             "retcodes": np.bincount(r["retcode"], minlength=6).tolist()})
            print(f"{case:55s} B={batch.u0.shape[0]:5d} {time.time() - t1:6.1f}s "
                  f"rc={np.bincount(r['retcode'], minlength=6).tolist()} "
                  f"sens={int(r['sensitive'].sum())}", flush=True)
    for fname, d in files.items():
        np.savez_compressed(os.path.join(HERE, f"{fname}.npz"), **d)
    res, rman = residual_fixtures()
    np.savez_compressed(os.path.join(HERE, "residuals.npz"), **res)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump({"generated_by": "tests/golden/make_golden.py",
                   "reference": "nlkit 0.1.0 (unmodified, imported from NLKIT_REF)",
                   "numpy": np.__version__, "cases": manifest, "residuals": rman},
                  fh, indent=1)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
