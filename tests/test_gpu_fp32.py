"""fp32 instantiations on the configurations that ask for them (BASELINE
config C3: generalized Rosenbrock n = 8/16, SimpleBroyden and SimpleKlement,
fp64 and fp32; C4/C5 fp32 arms; north_star: "1e-4 in fp32").

The reference computes in fp64 only, so fp32 has no bit-level oracle
(SURVEY.md §7).  Each fp32 run is compared with the fp64 oracle on the same
inputs (the bench's seeds):
  * systems with the same retcode and the same step count, where the run
    succeeded or took at most 3 steps (Broyden's Stalled-after-2, short
    NonFinite runs): ||u32 - u64||_inf <= 1e-4 ||u64||_inf -- the same
    trajectory, computed in fp32;
  * every fp32 success is a root: the fp64 residual (oracle) at u32 is within
    10x the fp32 abstol (u32 is a rounded root; u^2 = p has two roots, and an
    fp32 run may legitimately land on the other one after a different
    trajectory);
  * no retcode gate elsewhere: fp32 trajectories of the chaotic Klement
    runs legitimately diverge from fp64 ones.
The comparisons must cover a real share of each batch (non-vacuous).
"""

import numpy as np
import pytest
import torch

from paper_2403_16341_b200 import solvers, workloads as W

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def rel_err(u32, u64):
    num = np.max(np.abs(u32.astype(np.float64) - u64), axis=1)
    den = np.max(np.abs(u64), axis=1)
    with np.errstate(all="ignore"):
        return np.where(den > 0, num / den, num)


def check(pid, alg, u0, p=None, abstol=1e-8, min_compared=4000, maxiters=1000):
    from oracle import oracle as O
    ref = O.solve_batch(pid, alg, u0, p, abstol=abstol, maxiters=maxiters)
    got = solvers.solve_batch(pid, u0, p, alg, solvers.SolveOptions(abstol, maxiters),
                              dtype=torch.float32, n=u0.shape[1]).to_numpy()
    assert got["u"].dtype == np.float32
    same = (ref["retcode"] == got["retcode"]) & (ref["nsteps"] == got["nsteps"])
    cmp_ = same & ((ref["retcode"] == 0) | (ref["nsteps"] <= 3))
    err = rel_err(got["u"], ref["u"])
    bad = np.nonzero(cmp_ & ~(err <= RTOL))[0]
    assert len(bad) == 0, f"{pid} {alg}: {len(bad)} systems beyond 1e-4 (e.g. {bad[:5]}, " \
                          f"err {err[bad[:5]]})"
    assert cmp_.sum() >= min_compared, f"only {cmp_.sum()} systems comparable"
    succ = np.nonzero(got["retcode"] == 0)[0]
    assert np.all(got["resid"][succ] <= abstol)
    for i in succ[:: max(1, len(succ) // 500)]:  # fp64 residual at the fp32 root
        r = O.residual(pid, got["u"][i].astype(np.float64), None if p is None else p[i],
                       u0.shape[1])
        assert np.max(np.abs(r)) <= 10 * abstol, f"{pid} {alg}[{i}]: not a root"
    return ref, got


@pytest.mark.parametrize("alg", ["broyden", "klement"])
@pytest.mark.parametrize("n", [8, 16])
def test_c3_fp32_vs_fp64(n, alg):
    b = W.c3_rosenbrock(n, 0, 20000)  # the bench's C3 inputs (seed 0)
    # Klement n = 16 ends NonFinite on 87 % of these starts in fp64 (SURVEY.md
    # App. B), after chaotic trajectories: few full runs are comparable there
    check(b.problem_id, alg, b.u0, min_compared=10 if (n, alg) == (16, "klement") else 4000)
    if alg == "broyden":
        # the first three iterations of every system (maxiters = 3): the same
        # trajectory in fp32 and fp64 wherever both run all three steps.  Not
        # for Klement: its diagonal secant t_i / s_i divides by differences of
        # nearby iterates, so fp32 rounding is amplified along the trajectory
        # (1e-4..2e-3 relative after 3 steps on ~1 % of the C3 starts) -- a
        # property of the fp32 iteration, compared only at its roots
        check(b.problem_id, alg, b.u0, maxiters=3, min_compared=4000)


@pytest.mark.parametrize("alg", ["newton-raphson", "trust-region", "broyden", "klement", "dfsane"])
def test_c5_fp32_vs_fp64(alg):
    """C5's n = 4 quadratics in fp32 (abstol 1e-6: fp32 cannot reach 1e-8 on
    u^2 = p) against fp64 at the same abstol."""
    b = W.c5_quadratic(0, 20000)
    check("quadratic", alg, b.u0, b.p, abstol=1e-6)


def test_c4_fp32_dfsane():
    b = W.c4_tridiagonal(0, 5000)
    check(b.problem_id, "dfsane", b.u0, abstol=1e-5, min_compared=1000)
