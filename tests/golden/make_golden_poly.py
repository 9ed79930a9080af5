"""Golden fixtures for the default poly-algorithm from the UNMODIFIED reference.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_poly.py

Every system is solved with ``nlkit.solve(problem)`` (algorithm=None ->
run_polyalgorithm, /root/reference/pkg/src/nlkit/core.py:158-169,
solvers.py:570-599), one Problem per system, on inputs where the first stage
(newton-raphson) often fails, so newton-backtracking and the trust region
run: generalized Rosenbrock n = 10 (the reference's own rescue case,
pkg/tests/test_globalize.py:153-159 and test_solvers.py:166-173) at its
canonical start and at u0 ~ U[0,1)^10, the C3 inputs (n = 8, 16), every suite
problem at its canonical start (acceptance criterion #4,
pkg/tests/test_acceptance.py:66-80) and at sigma = 1.0 perturbed starts,
trigonometric sigma = 0.1 (37 % of Newton runs end in MaxIters), boggs
sigma = 1.0, and quadratic.  Stored per case: u0, p, u, resid, retcode,
nsteps, nf, njac, nlinsolve, stage_retcodes (int8 [B, 3], -1 = stage not
run) and the reference's result_to_json payload with wall_time removed.
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("NLKIT_REF", "/root/reference/pkg/src"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import nlkit  # noqa: E402
from nlkit import problems as nlp  # noqa: E402

from paper_2403_16341_b200 import workloads as W  # noqa: E402
sys.path.insert(0, HERE)
from make_golden import nlkit_residual  # noqa: E402

RC_INDEX = {rc: i for i, rc in enumerate(nlkit.RetCode)}


def _solve(args):
    problem_id, n, u0, p = args
    prob = nlkit.Problem(nlkit_residual(problem_id, n), u0,
                         params=p if p is not None else np.zeros(0))
    with np.errstate(all="ignore"):
        res = nlkit.solve(prob)
    st = res.stats
    codes = [RC_INDEX[c] for c in res.stage_retcodes] + [-1] * (3 - len(res.stage_retcodes))
    payload = json.loads(nlkit.core.result_to_json(res))
    payload["stats"].pop("wall_time")
    return (np.asarray(res.u_star, dtype=float), float(res.resid_norm), RC_INDEX[res.retcode],
            st.nsteps, st.nf, st.njac, st.nlinsolve, codes, json.dumps(payload))


def cases():
    rng = np.random.default_rng(2024)
    out = {}
    d = nlp.generalized_rosenbrock(10)
    out["rosen10_canon"] = W.Batch("generalized_rosenbrock", 10, np.asarray(d.problem.u0)[None, :], None)
    out["rosen10"] = W.Batch("generalized_rosenbrock", 10, rng.random((160, 10)), None)
    out["rosen10_wide"] = W.Batch("generalized_rosenbrock", 10, rng.uniform(-2.0, 2.0, (160, 10)), None)
    out["rosen8"] = W.c3_rosenbrock(8, 0, 96)
    out["rosen16"] = W.c3_rosenbrock(16, 0, 64)
    for i in range(1, 24):
        b = W.c2_suite(i, 0, 24, 1.0)
        canon = np.asarray(nlp.test23(i).problem.u0, dtype=float)[None, :]
        out[f"suite{i:02d}"] = W.Batch(b.problem_id, b.n, np.concatenate([canon, b.u0]), None)
    out["trig_s01"] = W.c2_suite(11, 0, 160, 0.1)
    out["boggs_s1"] = W.c2_suite(22, 24, 184, 1.0)
    q = nlp.quadratic()
    out["quad"] = W.Batch("quadratic", q.problem.u0.shape[0], np.asarray(q.problem.u0)[None, :],
                          np.asarray(q.problem.params)[None, :])
    out["quad4"] = W.c5_quadratic(0, 64)
    return out


def main():
    data, meta = {}, {}
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for name, b in cases().items():
            jobs = [(b.problem_id, b.n, b.u0[i], None if b.p is None else b.p[i])
                    for i in range(len(b.u0))]
            res = pool.map(_solve, jobs, chunksize=1)
            B = len(jobs)
            data[f"{name}/u0"] = b.u0
            data[f"{name}/p"] = b.p if b.p is not None else np.zeros((B, 0))
            data[f"{name}/u"] = np.stack([r[0] for r in res])
            data[f"{name}/resid"] = np.array([r[1] for r in res])
            for k, f in enumerate(("retcode", "nsteps", "nf", "njac", "nlinsolve")):
                data[f"{name}/{f}"] = np.array([r[2 + k] for r in res],
                                               np.int8 if f == "retcode" else np.int32)
            data[f"{name}/stage_retcodes"] = np.array([r[7] for r in res], np.int8)
            data[f"{name}/json"] = np.array([r[8] for r in res])
            sr = data[f"{name}/stage_retcodes"]
            meta[name] = {"problem": b.problem_id, "n": b.n, "B": B,
                          "stages_run": np.bincount((sr >= 0).sum(1), minlength=4).tolist(),
                          "retcodes": np.bincount(data[f"{name}/retcode"], minlength=6).tolist()}
            print(name, meta[name], flush=True)
    np.savez_compressed(os.path.join(HERE, "poly.npz"), **data)
    with open(os.path.join(HERE, "poly_manifest.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
