"""ctypes binding of the in-tree CUDA library (include/nlk_b200.h).

There is no fallback: if ``libnlk_b200.so`` is missing or cannot be loaded,
every solve raises.  The library is built in-tree by
``python -m paper_2403_16341_b200.build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# NLK_LIB_PATH selects a variant build (python -m paper_2403_16341_b200.build --tag)
LIB_PATH = os.environ.get("NLK_LIB_PATH") or os.path.join(_PKG, "libnlk_b200.so")

NLK_OK = 0
ERRORS = {
    -1: KeyError,            # unknown problem (problems.py:459,474)
    -2: ValueError,          # size not compiled
    -3: KeyError,            # unknown algorithm (solvers.py:649-650)
    -4: ValueError,          # bad options (core.py:61-65)
    -5: ValueError,          # bad argument
    -6: NotImplementedError,  # combination not compiled
    -7: RuntimeError,        # CUDA error
}

# exported symbols, exactly those declared in include/nlk_b200.h
SYMBOLS = ("nlk_version", "nlk_build_id", "nlk_last_error", "nlk_alg_lookup", "nlk_num_problems",
           "nlk_problem_info", "nlk_problem_lookup", "nlk_solve_batch",
           "nlk_solve_batch_host", "nlk_solve_batch_host_async", "nlk_solve_batch_poly", "nlk_last_grid", "nlk_last_launches",
           "nlk_fp64_peak", "nlk_fp32_peak", "nlk_ift_forward_batch", "nlk_ift_adjoint_batch")

_lib = None


class LibraryMissing(ImportError):
    pass


def lib():
    """Load and type the library (once)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built; run `python -m paper_2403_16341_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i32, i64, vp, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
    pi32 = ctypes.POINTER(i32)
    L.nlk_version.restype = ctypes.c_int
    L.nlk_last_error.restype = ctypes.c_char_p
    L.nlk_build_id.restype = ctypes.c_char_p
    L.nlk_alg_lookup.argtypes = [ctypes.c_char_p]
    L.nlk_num_problems.restype = ctypes.c_int
    L.nlk_problem_info.argtypes = [i32, ctypes.POINTER(ctypes.c_char_p), pi32, pi32]
    L.nlk_problem_lookup.argtypes = [ctypes.c_char_p, i32, pi32, pi32, pi32]
    L.nlk_solve_batch.argtypes = [i32, i32, i32, i64, vp, vp, dbl, i32, vp, vp, vp, vp, vp, vp,
                                  vp, vp]
    L.nlk_solve_batch_host.argtypes = [i32, i32, i32, i64, vp, vp, dbl, i32, vp, vp, vp, vp,
                                       vp, vp, vp, i64, i32]
    L.nlk_solve_batch_host_async.argtypes = [i32, i32, i32, i64, vp, vp, dbl, i32, vp, vp, vp,
                                             vp, vp, vp, vp, vp]
    L.nlk_solve_batch_poly.argtypes = [i32, i32, i64, vp, vp, dbl, i32, vp, vp, vp, vp, vp, vp,
                                       vp, vp, vp]
    L.nlk_last_grid.restype = ctypes.c_int
    L.nlk_last_launches.restype = ctypes.c_int
    L.nlk_fp64_peak.argtypes = [i64, ctypes.POINTER(dbl), vp]
    L.nlk_fp32_peak.argtypes = [i64, ctypes.POINTER(dbl), vp]
    L.nlk_ift_forward_batch.argtypes = [i32, i32, i64, vp, vp, dbl, vp, vp, vp, vp]
    L.nlk_ift_adjoint_batch.argtypes = [i32, i32, i64, vp, vp, vp, dbl, vp, vp, vp, vp]
    _lib = L
    return L


def build_id():
    """nlk_build_id() of the loaded library."""
    return lib().nlk_build_id().decode()


def source_build_id():
    """The build id of the sources in this tree (build.source_build_id)."""
    from .build import source_build_id as sbi
    return sbi()


def check(rc):
    if rc != NLK_OK:
        msg = lib().nlk_last_error().decode(errors="replace")
        raise ERRORS.get(rc, RuntimeError)(msg)
    return rc


def problem_lookup(problem_id, n=0):
    h, nn, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    check(lib().nlk_problem_lookup(problem_id.encode(), int(n), ctypes.byref(h),
                                   ctypes.byref(nn), ctypes.byref(m)))
    return h.value, nn.value, m.value


def alg_lookup(name):
    rc = lib().nlk_alg_lookup(name.encode())
    if rc < 0:
        check(rc)
    return rc


def problems():
    out = []
    L = lib()
    for h in range(L.nlk_num_problems()):
        pid, n, m = ctypes.c_char_p(), ctypes.c_int32(), ctypes.c_int32()
        check(L.nlk_problem_info(h, ctypes.byref(pid), ctypes.byref(n), ctypes.byref(m)))
        out.append((pid.value.decode(), n.value, m.value))
    return out
