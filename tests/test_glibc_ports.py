"""The device ports of glibc's exp / pow / sin / cos / atan
(paper_2403_16341_b200/csrc/nlk_glibc.cuh) compiled for the host with g++
are bit-identical to the libm the reference calls, on random inputs across
every branch (the same source is what the kernels run)."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CSRC = os.path.join(ROOT, "paper_2403_16341_b200", "csrc")
SHIM = r'''
#include "nlk_glibc.cuh"
extern "C" {
void g_exp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::glibc::exp(x[i]); }
void g_sincos_s(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) { double c; nlk::glibc::sincos(x[i], &y[i], &c); } }
void g_sincos_c(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) { double s; nlk::glibc::sincos(x[i], &s, &y[i]); } }
void g_sincosn(const double* x, double* s, double* c, long n) {  // n % 10 == 0
  for (long i = 0; i < n; i += 10)
    if (nlk::glibc::sincos_n<10>(x + i, s + i, c + i))
      for (long j = i; j < i + 10; ++j)
        if (nlk::glibc::sincos_slow(x[j])) nlk::glibc::sincos(x[j], &s[j], &c[j]);
}
void g_npexp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::svml::exp(x[i]); }
void g_npatan(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::svml::atan(x[i]); }
void g_sin(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::glibc::sin(x[i]); }
void g_cos(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::glibc::cos(x[i]); }
void g_atan(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::glibc::atan(x[i]); }
void g_pow2(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::glibc::pow_int<2>(x[i]); }
void g_pow3(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = nlk::glibc::pow_int<3>(x[i]); }
void l_exp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = ::exp(x[i]); }
void l_sin(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = ::sin(x[i]); }
void l_cos(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = ::cos(x[i]); }
void l_atan(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = ::atan(x[i]); }
void l_pow2(const double* x, double* y, long n) { double (*volatile p)(double, double) = ::pow; for (long i = 0; i < n; ++i) y[i] = p(x[i], 2.0); }
void l_pow3(const double* x, double* y, long n) { double (*volatile p)(double, double) = ::pow; for (long i = 0; i < n; ++i) y[i] = p(x[i], 3.0); }
}
'''


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    d = tmp_path_factory.mktemp("glibc")
    src, so = d / "shim.cpp", d / "shim.so"
    src.write_text(SHIM)
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-builtin", "-shared",
                    "-fPIC", "-I", CSRC, str(src), "-o", str(so), "-lm"], check=True)
    L = ctypes.CDLL(str(so))
    return L


def inputs(kind, n, rng):
    u = rng.uniform(-1, 1, n)
    if kind == "exp":
        parts = [u * 20, u * 745, u * 1e-3, rng.uniform(-1, 1, n) * 700]
    elif kind in ("sin", "cos"):
        parts = [u * 10, u * 3, u * 1e5, u * 1e-3, u * np.exp(rng.uniform(-18, 18, n)),
                 u * np.exp(rng.uniform(18.4, 709, n)),  # >= 105414350: __branred
                 np.round(u * 1e12) * 1.0]
    elif kind == "atan":
        parts = [u, u * 20, u * 0.07, u * np.exp(rng.uniform(-40, 40, n))]
    else:
        parts = [u * 10, u * np.exp(rng.uniform(-300, 300, n)), u * 1e-310, 1 + u * 1e-6]
    x = np.concatenate(parts + [np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.0])])
    return np.ascontiguousarray(x)


@pytest.mark.parametrize("fn", ["exp", "sin", "cos", "atan", "pow2", "pow3", "sincos_s", "sincos_c"])
def test_port_is_bit_exact(lib, fn):
    rng = np.random.default_rng({"exp": 1, "sin": 2, "cos": 3, "atan": 4, "pow2": 5, "pow3": 6, "sincos_s": 7, "sincos_c": 8}[fn])
    kind = {"sincos_s": "sin", "sincos_c": "cos"}.get(fn, fn.rstrip("23"))
    x = inputs(kind, 250_000, rng)
    a, b = np.empty_like(x), np.empty_like(x)
    ptr = lambda v: v.ctypes.data_as(ctypes.c_void_p)
    getattr(lib, "g_" + fn)(ptr(x), ptr(a), ctypes.c_long(len(x)))
    ref = {"sincos_s": "sin", "sincos_c": "cos"}.get(fn, fn)
    getattr(lib, "l_" + ref)(ptr(x), ptr(b), ctypes.c_long(len(x)))
    same = (a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))
    assert same.all(), f"{fn}: {np.count_nonzero(~same)} mismatches, e.g. x={x[~same][:3]}"


def _numpy_uses_svml_exp():
    try:
        from numpy._core._multiarray_umath import __cpu_features__ as f
    except ImportError:
        return False
    return bool(f.get("AVX512_SKX"))


@pytest.mark.skipif(not _numpy_uses_svml_exp(), reason="numpy dispatches exp to SVML only on AVX512_SKX")
def test_numpy_exp_port_is_bit_exact(lib):
    """np.exp on this host is Intel SVML (__svml_exp8_ha), not glibc."""
    rng = np.random.default_rng(7)
    x = np.ascontiguousarray(np.concatenate([rng.uniform(-20, 20, 200_000),
                                             rng.uniform(-707, 707, 200_000),
                                             rng.uniform(-1e-6, 1e-6, 50_000)]))
    a = np.empty_like(x)
    lib.g_npexp(x.ctypes.data_as(ctypes.c_void_p), a.ctypes.data_as(ctypes.c_void_p),
                ctypes.c_long(len(x)))
    assert np.array_equal(a.view(np.int64), np.exp(x).view(np.int64))


@pytest.mark.skipif(not _numpy_uses_svml_exp(), reason="numpy dispatches to SVML only on AVX512_SKX")
def test_numpy_arctan_port_is_bit_exact(lib):
    """np.arctan on float64 is Intel SVML (__svml_atan8_ha, with a VRCP14PD
    seed), not glibc: ~0.17 % of results differ from math.atan."""
    rng = np.random.default_rng(8)
    u = rng.uniform(-1, 1, 200_000)
    x = np.ascontiguousarray(np.concatenate([
        u, u * 4, u * 7.875, u * 8, u * 100, u * np.exp(rng.uniform(-40, 40, 200_000)),
        u * 1e-300, np.round(u * 64) / 8,
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 7.875, -7.875, 1e300, 5e-324])]))
    a = np.empty_like(x)
    lib.g_npatan(x.ctypes.data_as(ctypes.c_void_p), a.ctypes.data_as(ctypes.c_void_p),
                 ctypes.c_long(len(x)))
    ref = np.arctan(x)
    same = (a.view(np.int64) == ref.view(np.int64)) | (np.isnan(a) & np.isnan(ref))
    assert same.all(), f"{np.count_nonzero(~same)} mismatches, e.g. x={x[~same][:4]}"


def test_grouped_sincos_is_bit_exact(lib):
    """glibc::sincos_n (the branch-free G-argument form the fp64 residuals
    use) equals libm sin and cos on every branch, arguments mixed per group."""
    rng = np.random.default_rng(9)
    x = np.concatenate([inputs("sin", 100_000, rng), inputs("cos", 100_000, rng)])
    x = rng.permutation(x)
    x = np.ascontiguousarray(np.concatenate([x, np.zeros((-len(x)) % 10)]))
    s, c, rs, rc = (np.empty_like(x) for _ in range(4))
    ptr = lambda v: v.ctypes.data_as(ctypes.c_void_p)
    lib.g_sincosn(ptr(x), ptr(s), ptr(c), ctypes.c_long(len(x)))
    lib.l_sin(ptr(x), ptr(rs), ctypes.c_long(len(x)))
    lib.l_cos(ptr(x), ptr(rc), ctypes.c_long(len(x)))
    for a, b in ((s, rs), (c, rc)):
        same = (a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))
        assert same.all(), f"{np.count_nonzero(~same)} mismatches, e.g. x={x[~same][:3]}"
