"""The C-ABI library loads, exports exactly the symbols include/nlk_b200.h
declares, and validates arguments before touching the GPU (the error
conventions of the reference: KeyError for unknown problems / presets
(problems.py:459,474; solvers.py:649-650), ValueError for bad options
(core.py:61-65)).  Runs on the CPU: no call here launches a kernel."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2403_16341_b200 import _lib

HEADER = os.path.join(ROOT, "include", "nlk_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return set(re.findall(r"NLK_API\s+[\w\s\*]+?\b(nlk_\w+)\s*\(", text))


def test_exports_match_header():
    L = _lib.lib()
    declared = header_symbols()
    assert declared == set(_lib.SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name


def test_problem_registry():
    h, n, m = _lib.problem_lookup("test23/wood")
    assert (n, m) == (4, 0)
    assert _lib.problem_lookup("quadratic", 2)[1:] == (2, 2)
    assert _lib.problem_lookup("generalized_rosenbrock", 16)[1] == 16
    assert _lib.problem_lookup("test23/broyden-tridiagonal", 16)[1] == 16
    ids = {p[0] for p in _lib.problems()}
    assert len([i for i in ids if i.startswith("test23/")]) == 23
    with pytest.raises(KeyError):
        _lib.problem_lookup("test23/nope")
    with pytest.raises(ValueError):
        _lib.problem_lookup("test23/wood", 5)


def test_alg_lookup():
    names = ["newton-raphson", "trust-region", "broyden", "klement", "dfsane",
             "newton-backtracking"]
    assert [_lib.alg_lookup(n) for n in names] == list(range(6))
    with pytest.raises(KeyError):
        _lib.alg_lookup("levenberg-marquardt")


def _call(handle=0, alg=0, dtype=0, B=0, u0=None, p=None, abstol=1e-8, maxiters=1000,
          uo=None, ro=None, rc=None):
    return _lib.lib().nlk_solve_batch(handle, alg, dtype, B, u0, p, abstol, maxiters, uo, ro,
                                      rc, None, None, None, None, None)


def test_validation_before_launch():
    L = _lib.lib()
    fake = ctypes.c_void_p(0x1000)  # never dereferenced: validation fails first
    assert _call(B=0) == 0
    assert _call(handle=10_000) == -1
    assert _call(alg=42) == -3
    assert _call(abstol=0.0) == -4
    assert _call(maxiters=0) == -4
    assert _call(B=-1) == -5
    assert _call(B=5) == -5  # null buffers
    hq = _lib.problem_lookup("quadratic", 2)[0]
    assert _call(handle=hq, B=5, u0=fake, uo=fake, ro=fake, rc=fake) == -5  # params missing
    hw = _lib.problem_lookup("test23/wood")[0]
    assert _call(handle=hw, dtype=1, B=5, u0=fake, uo=fake, ro=fake, rc=fake) == -6
    assert b"no compiled kernel" in L.nlk_last_error()
