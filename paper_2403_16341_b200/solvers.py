"""Drop-in solve API over the batched CUDA kernels.

Mirrors the reference entry points
  ``nlkit.solve(problem, algorithm=None, options=None)``      (core.py:158-169)
  ``nlkit.solvers.run_preset(name, problem, options, seed)``  (solvers.py:640-655)
  ``nlkit.solvers.run_algorithm(problem, spec, options)``     (solvers.py:106-116)
  ``nlkit.ALGORITHM_PRESETS``                                 (solvers.py:610-637)
  ``nlkit.solvers.run_polyalgorithm(problem, options)``       (solvers.py:570-599)
with identical signatures and result types, and adds the batched call the
reference cannot express: ``solve_batch(problem, u0[B, n], p[B, m], ...)``.
Every solve runs in ``libnlk_b200.so``; there is no CPU path.  PyTorch only
provides device memory and the current CUDA stream.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import (Problem, RetCode, SolveOptions, SolveResult, Stats, retcode_from_int)
from .errors import IncompatibleSpec
from .problems import DeviceResidual


@dataclass(frozen=True)
class AlgorithmSpec:
    """A batched-kernel algorithm; ``name`` is the nlkit preset name
    (solvers.py:610-637) and ``kernel`` the C-ABI algorithm id."""

    name: str
    kernel: int


ALGORITHM_PRESETS = {
    "newton-raphson": AlgorithmSpec("newton-raphson", 0),
    "trust-region": AlgorithmSpec("trust-region", 1),
    "broyden": AlgorithmSpec("broyden", 2),
    "klement": AlgorithmSpec("klement", 3),
    "dfsane": AlgorithmSpec("dfsane", 4),
    "newton-backtracking": AlgorithmSpec("newton-backtracking", 5),
}

# the paper's names for the same presets
SimpleNewtonRaphson = ALGORITHM_PRESETS["newton-raphson"]
SimpleTrustRegion = ALGORITHM_PRESETS["trust-region"]
SimpleBroyden = ALGORITHM_PRESETS["broyden"]
SimpleKlement = ALGORITHM_PRESETS["klement"]
SimpleDFSane = ALGORITHM_PRESETS["dfsane"]

# default poly-algorithm for n <= QN_SKIP_THRESHOLD (solvers.py:553-567): the
# quasi-Newton stages are skipped, so every small system runs NR -> NR+LS -> TR
POLY_STAGES = ("newton-raphson", "newton-backtracking", "trust-region")
QN_SKIP_THRESHOLD = 25

# nlkit's built-in residual functions (problems.py:36-292), by __name__
_NLKIT_SUITE_FUNCS = {
    "_rosenbrock": "rosenbrock", "_powell_singular": "powell-singular",
    "_powell_badly_scaled": "powell-badly-scaled", "_wood": "wood",
    "_helical_valley": "helical-valley", "_watson": "watson", "_chebyquad": "chebyquad",
    "_brown_almost_linear": "brown-almost-linear",
    "_discrete_boundary_value": "discrete-boundary-value",
    "_discrete_integral": "discrete-integral", "_trigonometric": "trigonometric",
    "_variably_dimensioned": "variably-dimensioned",
    "_broyden_tridiagonal": "broyden-tridiagonal", "_broyden_banded": "broyden-banded",
    "_matrix_sqrt_2x2": "matrix-sqrt-2x2", "_matrix_sqrt_3x3": "matrix-sqrt-3x3",
    "_dennis_schnabel": "dennis-schnabel", "_product_exponential": "product-exponential",
    "_cubic_radial": "cubic-radial", "_double_root_scalar": "double-root-scalar",
    "_freudenstein_roth": "freudenstein-roth", "_boggs": "boggs",
    "_chandrasekhar": "chandrasekhar",
}


def resolve_problem(problem, n=None):
    """Map a problem description to (registry id, n).

    Accepts an id string, a DeviceResidual, one of our Problems, or an
    nlkit Problem whose residual is an nlkit built-in (matched by function
    identity: suite functions by name, the ``generalized_rosenbrock`` and
    ``quadratic`` closures by qualname).  Anything else raises — an arbitrary
    Python callable has no device code, and there is no CPU fallback.
    """
    if isinstance(problem, str):
        name, _, query = problem.partition("?")
        if query.startswith("N=") or query.startswith("n="):
            n = int(query[2:])
        return name, int(n or 0)
    res = getattr(problem, "residual", problem)
    if isinstance(res, DeviceResidual):
        return res.problem_id, res.n
    mod = getattr(res, "__module__", "") or ""
    qual = getattr(res, "__qualname__", "") or ""
    u0 = getattr(problem, "u0", None)
    size = int(np.asarray(u0).shape[0]) if u0 is not None else int(n or 0)
    if mod.endswith("nlkit.problems"):
        name = getattr(res, "__name__", "")
        if name in _NLKIT_SUITE_FUNCS:
            return "test23/" + _NLKIT_SUITE_FUNCS[name], size
        if qual.startswith("generalized_rosenbrock."):
            return "generalized_rosenbrock", size
        if qual.startswith("quadratic."):
            return "quadratic", size
    raise NotImplementedError(
        f"residual {mod}.{qual} has no device implementation; only the built-in "
        "problems of the registry run on the GPU (no CPU fallback)")


def resolve_algorithm(algorithm):
    """str preset name, our AlgorithmSpec, or an nlkit AlgorithmSpec equal to
    one of nlkit's presets."""
    if isinstance(algorithm, AlgorithmSpec):
        return algorithm
    if isinstance(algorithm, str):
        if algorithm not in ALGORITHM_PRESETS:
            raise KeyError(f"unknown algorithm {algorithm!r}")
        return ALGORITHM_PRESETS[algorithm]
    mod = type(algorithm).__module__ or ""
    if mod.startswith("nlkit"):
        assemble(algorithm)  # IncompatibleSpec exactly where nlkit raises it
        import importlib
        nl_solvers = importlib.import_module(mod.rsplit(".", 1)[0] + ".solvers")
        for name, spec in nl_solvers.ALGORITHM_PRESETS.items():
            if spec == algorithm and name in ALGORITHM_PRESETS:
                return ALGORITHM_PRESETS[name]
        raise NotImplementedError(f"nlkit algorithm {algorithm!r} is a valid specification "
                                  "without a batched kernel")
    raise TypeError(f"cannot interpret {algorithm!r} as an algorithm")


def assemble(spec):
    """nlkit's block-compatibility validation (solvers.py:76-103), restated
    on the attributes of an nlkit AlgorithmSpec: raises IncompatibleSpec with
    the reference's message wherever ``nlkit.solvers.assemble`` would, so an
    invalid specification fails the same way before any kernel is looked up
    (run_algorithm calls it first, solvers.py:106-109)."""
    jac, des, glob, lin = spec.jacobian, spec.descent, spec.globalization, spec.linear
    materializes = jac.kind in ("analytic", "dual_dense", "fd_dense", "colored_sparse")
    if jac.kind == "matrix_free" and lin.kind not in ("gmres", "auto"):
        raise IncompatibleSpec("matrix-free Jacobians require an iterative "
                               "Krylov linear solver (gmres or auto)")
    if glob.kind == "trust_region":
        if des.kind != "dogleg":
            raise IncompatibleSpec("trust-region globalization requires the dogleg descent")
        if not materializes:
            raise IncompatibleSpec("trust region needs a materialized Jacobian "
                                   "for the dogleg/steepest directions")
    if des.kind == "dogleg" and glob.kind != "trust_region":
        raise IncompatibleSpec("dogleg descent only runs inside a trust region")
    if des.kind in ("halley", "potra_ptak") and glob.kind != "none":
        raise IncompatibleSpec(f"{des.kind} manages its own steps; globalization must be none")
    if jac.kind == "quasi_newton":
        if des.kind != "newton":
            raise IncompatibleSpec("quasi-Newton strategies provide only the "
                                   "Newton-type inverse application")
        if glob.kind == "trust_region":
            raise IncompatibleSpec("quasi-Newton strategies cannot drive a "
                                   "trust region (no explicit matrix)")
    if des.kind in ("damped_newton", "steepest") and not materializes:
        raise IncompatibleSpec(f"{des.kind} needs a materialized Jacobian")
    return spec


@dataclass
class BatchResult:
    """Per-system outputs of a batched solve (device tensors).

    ``u`` is [B, n] (a transposed view of the SoA [n, B] buffer); retcode
    codes are RetCode in declaration order (core.py:17-24)."""

    u: torch.Tensor
    resid: torch.Tensor
    retcode: torch.Tensor
    nsteps: torch.Tensor
    nf: torch.Tensor
    njac: torch.Tensor
    nlinsolve: torch.Tensor
    wall_time: float = 0.0
    stage_retcodes: torch.Tensor = None  # poly-algorithm: int8 [B, 3], -1 = stage not run

    def to_numpy(self):
        out = {k: getattr(self, k).cpu().numpy() for k in
               ("u", "resid", "retcode", "nsteps", "nf", "njac", "nlinsolve")}
        if self.stage_retcodes is not None:
            out["stage_retcodes"] = self.stage_retcodes.cpu().numpy()
        return out

    def result(self, i):
        """SolveResult of system i (core.py:80-91)."""
        st = Stats(nf=int(self.nf[i]), njac=int(self.njac[i]), njvp=0,
                   nlinsolve=int(self.nlinsolve[i]), nsteps=int(self.nsteps[i]),
                   wall_time=self.wall_time)
        stages = None
        if self.stage_retcodes is not None:
            stages = [retcode_from_int(c) for c in self.stage_retcodes[i].cpu().tolist() if c >= 0]
        return SolveResult(self.u[i].detach().cpu().numpy().astype(float),
                           float(self.resid[i]), retcode_from_int(int(self.retcode[i])), st,
                           stage_retcodes=stages)


_DTYPES = {torch.float64: 0, torch.float32: 1, "f64": 0, "f32": 1, np.float64: 0,
           np.float32: 1}


def solve_batch_soa(handle, alg, u0_soa, p_soa, abstol=1e-8, maxiters=1000, out=None,
                    stream=None):
    """Lowest-level call: SoA device tensors in, SoA device tensors out
    (nlk_solve_batch).  ``out`` may pre-allocate (u [n,B], resid [B],
    retcode [B], counters [4,B]); returns that dict."""
    n, B = u0_soa.shape
    dt = u0_soa.dtype
    dev = u0_soa.device
    if out is None:
        out = {"u": torch.empty((n, B), dtype=dt, device=dev),
               "resid": torch.empty(B, dtype=dt, device=dev),
               "retcode": torch.empty(B, dtype=torch.int8, device=dev),
               "counters": torch.empty((4, B), dtype=torch.int32, device=dev)}
    c = out["counters"]
    # the library runs on the stream's device; the legacy default stream (0)
    # means the current device, so make it u0's
    with torch.cuda.device(dev):
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().nlk_solve_batch(
            handle, alg, _DTYPES[dt], B, u0_soa.data_ptr(),
            None if p_soa is None else p_soa.data_ptr(), float(abstol), int(maxiters),
            out["u"].data_ptr(), out["resid"].data_ptr(), out["retcode"].data_ptr(),
            c[0].data_ptr(), c[1].data_ptr(), c[2].data_ptr(), c[3].data_ptr(), stream))
    return out


def solve_batch_poly_soa(handle, u0_soa, p_soa, abstol=1e-8, maxiters=1000, out=None,
                         stream=None):
    """The batched default poly-algorithm (nlk_solve_batch_poly): SoA device
    tensors in; the dict of solve_batch_soa plus ``stage_retcodes`` int8
    [3, B] (-1 = stage not run)."""
    n, B = u0_soa.shape
    dt = u0_soa.dtype
    dev = u0_soa.device
    if out is None:
        out = {"u": torch.empty((n, B), dtype=dt, device=dev),
               "resid": torch.empty(B, dtype=dt, device=dev),
               "retcode": torch.empty(B, dtype=torch.int8, device=dev),
               "counters": torch.empty((4, B), dtype=torch.int32, device=dev),
               "stage_retcodes": torch.empty((3, B), dtype=torch.int8, device=dev)}
    c = out["counters"]
    with torch.cuda.device(dev):
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().nlk_solve_batch_poly(
            handle, _DTYPES[dt], B, u0_soa.data_ptr(),
            None if p_soa is None else p_soa.data_ptr(), float(abstol), int(maxiters),
            out["u"].data_ptr(), out["resid"].data_ptr(), out["retcode"].data_ptr(),
            c[0].data_ptr(), c[1].data_ptr(), c[2].data_ptr(), c[3].data_ptr(),
            out["stage_retcodes"].data_ptr(), stream))
    return out


def _as_device(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype)
    a = np.asarray(x)
    if not a.flags.writeable:  # e.g. np.broadcast_to views: torch wants writable memory
        a = np.array(a)
    return torch.as_tensor(a, dtype=dtype, device=device)


def solve_batch(problem, u0, p=None, algorithm="newton-raphson", options=None,
                dtype=torch.float64, device=None, n=None):
    """Solve B independent systems of one registered problem.

    ``u0`` is [B, n] (or [n] for one system), ``p`` is [B, m] (or [m],
    broadcast); host (numpy / CPU tensor) or CUDA inputs.  Returns a
    BatchResult of CUDA tensors.  ``algorithm`` is a preset name, an
    AlgorithmSpec, an nlkit AlgorithmSpec, or "polyalgorithm".
    """
    options = options or SolveOptions()
    if getattr(options, "store_trace", False):
        raise NotImplementedError("store_trace is not supported on the batched GPU path")
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the batched solver has no CPU fallback")
    device = torch.device(device or "cuda")
    dtype = {"f64": torch.float64, "f32": torch.float32}.get(dtype, dtype)
    u0 = _as_device(u0, dtype, device)
    if u0.dim() == 1:
        u0 = u0[None, :]
    B, nn = u0.shape
    pid, n_req = resolve_problem(problem, n or nn)
    handle, n_reg, m = _lib.problem_lookup(pid, n_req or nn)
    if nn != n_reg:
        raise ValueError(f"{pid}: u0 has {nn} columns, the problem has n={n_reg}")
    if m:
        if p is None:
            p = getattr(problem, "params", None)
        if p is None:
            raise ValueError(f"{pid} needs parameters p [B, {m}]")
        p = _as_device(p, dtype, device)
        if p.dim() == 1:
            p = p[None, :].expand(B, m)
        if p.shape != (B, m):
            raise ValueError(f"p must be [{B}, {m}], got {tuple(p.shape)}")
        p_soa = p.t().contiguous()
    else:
        p_soa = None
    u0_soa = u0.t().contiguous()
    t0 = time.perf_counter()
    if algorithm == "polyalgorithm" or algorithm is None:
        out = solve_batch_poly_soa(handle, u0_soa, p_soa, options.abstol, options.maxiters)
    else:
        spec = resolve_algorithm(algorithm)
        out = solve_batch_soa(handle, spec.kernel, u0_soa, p_soa, options.abstol,
                              options.maxiters)
    torch.cuda.current_stream(device).synchronize()
    wall = time.perf_counter() - t0
    c = out["counters"]
    sr = out.get("stage_retcodes")
    return BatchResult(out["u"].t(), out["resid"], out["retcode"], c[0], c[1], c[2], c[3],
                       wall, None if sr is None else sr.t())


def run_algorithm(problem, spec, options=None):
    """solvers.py:106-116 for one system (a batch of one on the GPU)."""
    options = options or SolveOptions()
    r = solve_batch(problem, problem.u0, getattr(problem, "params", None), spec, options)
    res = r.result(0)
    res.stats.wall_time = r.wall_time
    return res


def run_polyalgorithm(problem, options=None):
    """solvers.py:570-599 (small systems: QN stages are skipped)."""
    options = options or SolveOptions()
    if problem.n > QN_SKIP_THRESHOLD:
        raise NotImplementedError("systems with n > 25 are outside the batched small-system path")
    r = solve_batch(problem, problem.u0, getattr(problem, "params", None), "polyalgorithm",
                    options)
    return r.result(0)


def run_preset(name, problem, options=None, seed=None):
    """solvers.py:640-655."""
    options = options or SolveOptions()
    if name == "polyalgorithm":
        return run_polyalgorithm(problem, options)
    if name not in ALGORITHM_PRESETS:
        raise KeyError(f"unknown algorithm {name!r}")
    return run_algorithm(problem, ALGORITHM_PRESETS[name], options)


def solve(problem, algorithm=None, options=None):
    """core.py:158-169: the default poly-algorithm when algorithm is None."""
    options = options or SolveOptions()
    if algorithm is None:
        return run_polyalgorithm(problem, options)
    return run_algorithm(problem, algorithm, options)


def list_algorithms():
    return sorted(list(ALGORITHM_PRESETS) + ["polyalgorithm"])
