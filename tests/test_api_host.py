"""Host-side logic of the drop-in API that needs no GPU: problem identity
mapping (including nlkit's own Problem objects), presets, options, workload
generation and sharding."""

import os
import sys

import numpy as np
import pytest

from paper_2403_16341_b200 import core, problems, solvers, workloads as W

NLKIT_SRC = os.environ.get("NLKIT_REF", "/root/reference/pkg/src")


def test_presets_and_aliases():
    assert solvers.SimpleNewtonRaphson.kernel == 0
    assert solvers.SimpleDFSane.name == "dfsane"
    assert solvers.resolve_algorithm("klement") is solvers.SimpleKlement
    with pytest.raises(KeyError):
        solvers.resolve_algorithm("nope")
    assert "polyalgorithm" in solvers.list_algorithms()


def test_options_validation():
    with pytest.raises(ValueError):
        core.SolveOptions(abstol=0)
    with pytest.raises(ValueError):
        core.SolveOptions(maxiters=0)


def test_problem_catalogue():
    for i in range(1, 24):
        d = problems.test23(i)
        assert d.problem.n == d.n
        assert solvers.resolve_problem(d.problem) == (d.id, d.n)
    d = problems.get_problem("generalized_rosenbrock?N=8")
    assert d.problem.u0[0] == -1.2 and solvers.resolve_problem(d.problem) == ("generalized_rosenbrock", 8)
    q = problems.quadratic((2.0, 5.0))
    assert np.allclose(q.reference_solution, np.sqrt([2, 5]))
    with pytest.raises(RuntimeError):
        q.problem.residual(q.problem.u0, q.problem.params)  # no CPU evaluation
    with pytest.raises(KeyError):
        problems.get_problem("brusselator2d?N=8")


@pytest.mark.skipif(not os.path.isdir(NLKIT_SRC), reason="reference not present")
def test_nlkit_problems_map_to_registry():
    sys.path.insert(0, NLKIT_SRC)
    import nlkit
    from nlkit import problems as nlp
    for i in range(1, 24):
        d = nlp.test23(i)
        assert solvers.resolve_problem(d.problem) == (d.id, d.n)
    assert solvers.resolve_problem(nlp.generalized_rosenbrock(16).problem) == \
        ("generalized_rosenbrock", 16)
    assert solvers.resolve_problem(nlp.quadratic((1.0, 2.0, 3.0)).problem) == ("quadratic", 3)
    for name in ("newton-raphson", "trust-region", "broyden", "klement"):
        assert solvers.resolve_algorithm(nlkit.ALGORITHM_PRESETS[name]).name == name
    with pytest.raises(NotImplementedError):
        solvers.resolve_problem(nlkit.Problem(lambda u, p: u, np.ones(2)))


def test_workload_chunks_are_shard_invariant():
    full = W.c2_suite(4, 0, 3 * W.CHUNK + 17).u0
    for world in (1, 2, 3, 8):
        parts = [W.c2_suite(4, *W.shard_bounds(len(full), world, r)).u0 for r in range(world)]
        assert np.array_equal(np.concatenate(parts), full)
    # chunk 0 is the plain default_rng(seed) stream (what the golden fixtures hold)
    p = W.c1_quadratic(0, 1024).p
    assert np.array_equal(p, np.random.default_rng(0).uniform(0.5, 10.0, (1024, 2)))


def test_shard_bounds():
    for B in (0, 1, 7, 1000, 10**8 + 3):
        for world in (1, 2, 4, 8):
            b = [W.shard_bounds(B, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == B
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1


def test_result_json_roundtrip():
    r = core.SolveResult(np.array([1.0, 2.0]), 1e-9, core.RetCode.SUCCESS,
                         core.Stats(nf=3, njac=1, nlinsolve=1, nsteps=1))
    s = core.result_to_json(r)
    assert '"retcode": "Success"' in s and '"nf": 3' in s


@pytest.mark.skipif(not os.path.isdir(NLKIT_SRC), reason="reference not present")
def test_assemble_matches_reference():
    """solvers.assemble raises IncompatibleSpec (same message) exactly where
    nlkit.solvers.assemble does (solvers.py:76-103), over every combination
    of Jacobian strategy x descent x globalization x linear solver; a valid
    specification without a batched kernel is NotImplementedError, and the
    presets map to their kernels."""
    sys.path.insert(0, NLKIT_SRC)
    import itertools

    import nlkit
    from nlkit import descent as nd, jacobians as nj, linalg as nl, quasinewton as nq
    from nlkit import solvers as ns

    from paper_2403_16341_b200.errors import IncompatibleSpec
    jacs = [nj.ANALYTIC, nj.DUAL_DENSE, nj.FD_DENSE, nj.COLORED_SPARSE, nj.MATRIX_FREE,
            nj.JacobianSpec("quasi_newton", qn=nq.QuasiNewtonConfig())]
    descs = [nd.NEWTON, nd.STEEPEST, nd.DOGLEG, nd.HALLEY, nd.POTRA_PTAK, nd.DampedNewton()]
    globs = [ns.NO_GLOBALIZATION, ns.LineSearch(), ns.TrustRegion()]
    lins = [nl.AUTO, nl.LU, nl.QR, nl.GMRES()]
    n_bad = 0
    for j, d, g, li in itertools.product(jacs, descs, globs, lins):
        spec = ns.AlgorithmSpec(jacobian=j, descent=d, globalization=g, linear=li)
        try:
            ns.assemble(spec)
            ref = None
        except nlkit.errors.IncompatibleSpec as e:
            ref = str(e)
        if ref is None:
            assert solvers.assemble(spec) is spec
        else:
            n_bad += 1
            with pytest.raises(IncompatibleSpec) as ei:
                solvers.resolve_algorithm(spec)
            assert str(ei.value) == ref
    assert n_bad > 100
    for name in ("newton-raphson", "trust-region", "broyden", "klement", "newton-backtracking"):
        assert solvers.resolve_algorithm(ns.ALGORITHM_PRESETS[name]).name == name
    with pytest.raises(NotImplementedError):
        solvers.resolve_algorithm(ns.ALGORITHM_PRESETS["levenberg-marquardt"])
