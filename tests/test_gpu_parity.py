"""Parity of the CUDA kernels (through the C-ABI) with the reference.

Three layers, all on identical inputs:
  1. golden fixtures produced by the unmodified reference (small samples of
     every BASELINE.json config, all five algorithms + newton-backtracking);
  2. the oracle restatement at larger samples (20k systems per C2 problem,
     5k per C3/C4 case);
  3. size-independent properties at full size (1M systems): known roots,
     determinism, permutation invariance, host-buffer path == device path.

Gate: bit-identical u and resid, and identical retcode, nsteps, nf, njac,
nlinsolve, on every system — including the roundoff-sensitive ones (the
survey's one-ulp probe flips up to 60 % of test23/trigonometric starts).
This holds because the kernels reproduce the reference host's arithmetic:
unfused residuals, the OpenBLAS/LAPACK operation orders, glibc's exp / pow /
sin / cos / atan and numpy's SVML exp (nlk_glibc.cuh).
"""

import numpy as np
import pytest
import torch

from conftest import close, golden_case, load_manifest
from paper_2403_16341_b200 import _lib, solvers, workloads as W

pytestmark = pytest.mark.gpu

CASES = load_manifest()["cases"]


def gpu_solve(pid, alg, u0, p=None, abstol=1e-8, maxiters=1000, dtype=torch.float64):
    r = solvers.solve_batch(pid, u0, p, alg, solvers.SolveOptions(abstol, maxiters),
                            dtype=dtype, n=u0.shape[1])
    return r.to_numpy()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def check_against(ref, got, what, problem_id=None):
    """Every field of every system bit-identical (no exemptions: sin/cos of
    huge arguments go through the port of glibc's __branred)."""
    same = np.ones(len(ref["retcode"]), bool)
    for k in ("retcode", "nsteps", "nf", "njac", "nlinsolve"):
        same &= got[k] == ref[k]
    same &= (bits(got["u"]) == bits(ref["u"])).all(axis=1)
    same &= bits(got["resid"]) == bits(ref["resid"])
    bad = np.nonzero(~same)[0]
    assert len(bad) == 0, f"{what}: {len(bad)} systems differ (e.g. {bad[:8]})"


@pytest.mark.parametrize("case", CASES, ids=[c["case"] for c in CASES])
def test_golden(case):
    g = golden_case(case)
    p = g["p"] if g["p"].shape[1] else None
    got = gpu_solve(case["problem_id"], case["alg"], g["u0"], p)
    check_against(g, got, case["case"], case["problem_id"])


@pytest.mark.parametrize("sigma", [0.1, 1.0])
@pytest.mark.parametrize("alg", ["newton-raphson", "trust-region"])
@pytest.mark.parametrize("index", range(1, 24))
def test_oracle_c2_sample(index, alg, sigma):
    """C2's 20k-system samples at the primary sigma = 0.1 and the stress
    sigma = 1.0."""
    from oracle import oracle as O
    b = W.c2_suite(index, 0, 20000, sigma)
    ref = O.solve_batch(b.problem_id, alg, b.u0)
    got = gpu_solve(b.problem_id, alg, b.u0)
    check_against(ref, got, f"C2 #{index} {alg} sigma={sigma}", b.problem_id)


@pytest.mark.parametrize("alg", ["broyden", "klement", "dfsane", "newton-raphson", "trust-region"])
@pytest.mark.parametrize("n", [8, 16])
def test_oracle_c3_c4_sample(n, alg):
    from oracle import oracle as O
    batches = [W.c3_rosenbrock(n, 0, 5000)] + ([W.c4_tridiagonal(0, 5000)] if n == 16 else [])
    for b in batches:
        ref = O.solve_batch(b.problem_id, alg, b.u0)
        got = gpu_solve(b.problem_id, alg, b.u0)
        check_against(ref, got, f"{b.problem_id} {alg}", b.problem_id)


def test_c1_full_size_known_roots():
    """1M parameter sets of u^2 - p: every solve succeeds and u = sqrt(p) to
    rounding; the first 1024 are the reference's golden C1 systems."""
    b = W.c1_quadratic(0, 1 << 20)
    got = gpu_solve("quadratic", "newton-raphson", b.u0, b.p)
    assert (got["retcode"] == 0).all()
    assert (got["resid"] <= 1e-8).all()
    # |u^2 - p| <= 1e-8 and u >= 0.7  =>  |u - sqrt(p)| <= 1e-8 / (2 * 0.7)
    assert (np.abs(got["u"] - np.sqrt(b.p)) <= 1e-8).all()
    g = golden_case(next(c for c in CASES if c["case"] == "c1/newton-raphson"))
    assert np.array_equal(bits(got["u"][:1024]), bits(g["u"]))
    assert np.array_equal(got["nsteps"][:1024], g["nsteps"])


def test_determinism_and_permutation_invariance():
    b = W.c2_suite(23, 0, 200_000, 0.1)
    a1 = gpu_solve(b.problem_id, "trust-region", b.u0)
    a2 = gpu_solve(b.problem_id, "trust-region", b.u0)
    for k in a1:
        assert np.array_equal(a1[k], a2[k]), k
    perm = np.random.default_rng(1).permutation(len(b.u0))
    a3 = gpu_solve(b.problem_id, "trust-region", b.u0[perm])
    assert np.array_equal(bits(a3["u"]), bits(a1["u"][perm]))
    assert np.array_equal(a3["nsteps"], a1["nsteps"][perm])


def test_host_buffer_path_equals_device_path():
    import ctypes
    b = W.c2_suite(13, 0, 300_001, 0.1)
    dev = gpu_solve(b.problem_id, "newton-raphson", b.u0)
    h, n, m = _lib.problem_lookup(b.problem_id, 10)
    B = len(b.u0)
    u0 = np.ascontiguousarray(b.u0.T)
    uo = np.empty((n, B))
    ro = np.empty(B)
    rc = np.empty(B, np.int8)
    cnt = np.empty((4, B), np.int32)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _lib.check(_lib.lib().nlk_solve_batch_host(h, 0, 0, B, ptr(u0), None, 1e-8, 1000, ptr(uo),
                                               ptr(ro), ptr(rc), ptr(cnt[0]), ptr(cnt[1]),
                                               ptr(cnt[2]), ptr(cnt[3]), 100_000, 3))
    assert np.array_equal(bits(uo.T), bits(dev["u"]))
    assert np.array_equal(rc, dev["retcode"])
    assert np.array_equal(cnt[0], dev["nsteps"]) and np.array_equal(cnt[1], dev["nf"])


def test_async_host_path_equals_device_path():
    """nlk_solve_batch_host_async: two batches in flight on two streams from
    pinned buffers, results identical to the device-buffer path."""
    import ctypes
    outs = []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    jobs = [W.c2_suite(13, 0, 200_003, 0.1), W.c2_suite(11, 0, 150_001, 0.1)]
    for j, b in enumerate(jobs):
        h, n, m = _lib.problem_lookup(b.problem_id, b.u0.shape[1])
        B = len(b.u0)
        u0 = torch.from_numpy(np.ascontiguousarray(b.u0.T)).pin_memory()
        o = (torch.empty((n, B), dtype=torch.float64).pin_memory(),
             torch.empty(B, dtype=torch.float64).pin_memory(),
             torch.empty(B, dtype=torch.int8).pin_memory(),
             torch.empty((4, B), dtype=torch.int32).pin_memory())
        _lib.check(_lib.lib().nlk_solve_batch_host_async(
            h, 0, 0, B, u0.data_ptr(), None, 1e-8, 1000, o[0].data_ptr(), o[1].data_ptr(),
            o[2].data_ptr(), o[3][0].data_ptr(), o[3][1].data_ptr(), o[3][2].data_ptr(),
            o[3][3].data_ptr(), streams[j].cuda_stream))
        outs.append((b, u0, o))
    for st in streams:
        st.synchronize()
    for b, _u0, (uo, ro, rc, cn) in outs:
        dev = gpu_solve(b.problem_id, "newton-raphson", b.u0)
        assert np.array_equal(bits(uo.numpy().T), bits(dev["u"]))
        assert np.array_equal(bits(ro.numpy()), bits(dev["resid"]))
        assert np.array_equal(rc.numpy(), dev["retcode"])
        assert np.array_equal(cn.numpy()[0], dev["nsteps"]) and np.array_equal(cn.numpy()[3], dev["nlinsolve"])


@pytest.mark.parametrize("alg", ["newton-raphson", "trust-region", "klement", "dfsane"])
def test_fp32_against_fp64(alg):
    """fp32 has no reference; where fp32 and fp64 both succeed, u agrees to
    1e-4 relative (north star), with abstol 1e-5 for fp32."""
    b = W.c1_quadratic(0, 100_000, n=4, seed=5)
    r64 = gpu_solve("quadratic", alg, b.u0, b.p)
    r32 = gpu_solve("quadratic", alg, b.u0, b.p, abstol=1e-5, dtype=torch.float32)
    both = (r64["retcode"] == 0) & (r32["retcode"] == 0)
    assert both.mean() > 0.99
    # u^2 = p has roots +-sqrt(p); a solver may pick either, so compare |u|
    assert close(np.abs(r32["u"][both]), np.abs(r64["u"][both]), 1e-4).all()


def test_drop_in_single_solve_and_polyalgorithm():
    import paper_2403_16341_b200 as nlk
    d = nlk.get_problem("test23/rosenbrock")
    r = nlk.solve(d.problem, nlk.SimpleNewtonRaphson)
    assert r.retcode is nlk.RetCode.SUCCESS and r.stats.nsteps == 2
    r = nlk.run_preset("trust-region", d.problem)
    assert r.success and r.stats.nsteps == 13
    r = nlk.solve(d.problem)  # default poly-algorithm: NR succeeds first
    assert r.success and r.stats.nsteps == 2
    g = nlk.get_problem("generalized_rosenbrock?N=8")
    r = nlk.run_preset("klement", g.problem)
    assert r.retcode is nlk.RetCode.NONFINITE and r.stats.nsteps == 12


@pytest.mark.parametrize("maxiters", [150, 400, 1000, 3000])
@pytest.mark.parametrize("index,sigma", [(11, 0.1), (11, 1.0), (16, 1.0), (17, 1.0), (21, 1.0), (8, 1.0), (15, 1.0), (4, 1.0)])
def test_trust_region_fast_forward(index, sigma, maxiters):
    """The trust region's radius-exhaustion fast-forward (nlk_solvers.cuh,
    TrustRegion::step) replays the counters and the radius halving of a tail
    of bit-identical rejections.  Both ways out of that tail are exercised:
    maxiters (150..1000) and the radius underflow break (globalize.py:211-212,
    reached before maxiters = 3000 by the trigonometric, dennis-schnabel and
    freudenstein-roth MaxIters runs)."""
    from oracle import oracle as O
    b = W.c2_suite(index, 20000, 24000, sigma)
    ref = O.solve_batch(b.problem_id, "trust-region", b.u0, maxiters=maxiters)
    got = gpu_solve(b.problem_id, "trust-region", b.u0, maxiters=maxiters)
    check_against(ref, got, f"C2 #{index} TR sigma={sigma} maxiters={maxiters}", b.problem_id)
    if index in (11, 17, 21) and maxiters == 3000:
        early = (got["retcode"] == 1) & (got["nlinsolve"] < maxiters)
        assert early.any(), "radius-underflow exit not exercised"
