"""Shared fixtures.  ``-m gpu`` tests need a CUDA device; everything else runs
on the CPU (oracle, host logic, C-ABI loading/validation)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


_NPZ = {}


def golden_case(case):
    """Arrays of one golden case: u0, p, u, resid, retcode, nsteps, nf, njac,
    nlinsolve, sensitive."""
    fname = case["file"]
    if fname not in _NPZ:
        _NPZ[fname] = np.load(os.path.join(GOLDEN, f"{fname}.npz"))
    f = _NPZ[fname]
    k = case["case"]
    return {x: f[f"{k}/{x}"] for x in ("u0", "p", "u", "resid", "retcode", "nsteps", "nf",
                                       "njac", "nlinsolve", "sensitive")}


def load_manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


# Problems whose float path calls numpy's SIMD exp (not glibc's; SURVEY.md
# App. A.3): u/resid agree to rounding, not bit for bit.
EXP_PROBLEMS = {"test23/powell-badly-scaled", "test23/dennis-schnabel",
                "test23/product-exponential"}


def close(a, b, rtol):
    """|a - b| <= rtol * max(|a|, |b|), elementwise; NaN == NaN, inf == inf."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    with np.errstate(all="ignore"):
        ok = np.abs(a - b) <= rtol * np.maximum(np.abs(a), np.abs(b))
    return same | ok
