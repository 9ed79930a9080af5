"""Trigonometric starts with exact +0.0 / -0.0 components, from the UNMODIFIED
reference: a zero component makes its Jacobian column all zeros with
row-dependent zero signs -- the case the trust region's compressed
rank-one-plus-diagonal Jacobian (RDJac, nlk_solvers.cuh) stores separately.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_trig_zero.py

Writes tests/golden/trig_zero.npz with keys <alg>/{u0,u,resid,retcode,nsteps,
nf,njac,nlinsolve}.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as G  # noqa: E402

ALGS = ["trust-region", "newton-raphson"]


def starts(count=40, seed=11):
    rng = np.random.default_rng(seed)
    base = np.asarray(G.W.problems.suite_start("trigonometric"), dtype=float)
    U = base[None, :] + 0.1 * rng.uniform(-1, 1, (count, 10))
    for i in range(count):
        k = 1 + i % 4  # 1..4 zero components, alternating signs
        cols = rng.choice(10, k, replace=False)
        U[i, cols] = np.where(np.arange(k) % 2 == 0, 0.0, -0.0)
    U[-2] = 0.0
    U[-1] = -0.0
    return U


def main():
    import multiprocessing as mp
    out = {}
    U = starts()
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for alg in ALGS:
            r = G.run_case(pool, G.W.Batch("test23/trigonometric", 10, U, None, 0), alg,
                           1e-8, 1000, mask=False)
            for k in ("u0", "u", "resid", "retcode", "nsteps", "nf", "njac", "nlinsolve"):
                out[f"{alg}/{k}"] = r[k]
    np.savez_compressed(os.path.join(HERE, "trig_zero.npz"), **out)
    print({a: np.bincount(out[f"{a}/retcode"], minlength=6).tolist() for a in ALGS})


if __name__ == "__main__":
    main()
