"""Implicit-function-theorem sensitivities of roots, batched on the GPU.

Mirrors nlkit/sensitivity.py (ift_forward 40-57, ift_adjoint 60-80,
SensitivityResult 20-23): at a root u*(θ) of f(u, θ) = 0,

    forward   du*/dθ = S  solves  (∂f/∂u) S = -(∂f/∂θ)      (one LU, m solves)
    adjoint   ∇_θ g   = -(∂f/∂θ)ᵀ λ  with  (∂f/∂u)ᵀ λ = ∂g/∂u

The work runs in the CUDA library (nlk_ift_forward_batch /
nlk_ift_adjoint_batch, csrc/nlk_ift.cuh) with the reference's operation
order: dual Jacobians over u and θ, strict partial-pivoting LU, LAPACK
getrs (and getrs with trans=1) for one right-hand side at a time.
Parametrised registry problems only (m > 0); there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import NonFiniteValue, SingularMatrix
from .solvers import resolve_problem

OK, NOT_A_ROOT, SINGULAR, NONFINITE = 0, 1, 2, 3


@dataclass
class SensitivityResult:
    """sensitivity.py:20-23."""

    value: np.ndarray
    solve_residual: float


@dataclass
class BatchSensitivity:
    """Per-system outputs of a batched IFT call (CUDA tensors).

    ``value`` is [B, n, m] (forward) or [B, m] (adjoint); ``status`` holds
    OK / NOT_A_ROOT / SINGULAR / NONFINITE; ``solve_residual`` is [B] (the
    reference's ``full=True`` diagnostic) or None."""

    value: torch.Tensor
    status: torch.Tensor
    solve_residual: torch.Tensor | None


def _handle(problem, n):
    # the reference differentiates problem.analytic_jacobian when one is set
    # (sensitivity.py:26-28); the device only has the dual-sweep Jacobian of
    # its registered residuals, so such a problem is refused, not silently
    # given a different Jacobian
    if getattr(problem, "analytic_jacobian", None) is not None:
        raise NotImplementedError("problems with an analytic_jacobian are not supported on the "
                                  "GPU sensitivity path (the device differentiates the "
                                  "registered residual with dual sweeps)")
    pid, nn = resolve_problem(problem, n)
    h, n_out, m = _lib.problem_lookup(pid, nn)
    if m == 0:
        raise NotImplementedError(f"{pid} has no parameters: nothing to differentiate")
    return h, n_out, m


def _soa(x, B, k, dev):
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float64))
    t = t.to(device=dev, dtype=torch.float64)
    if t.dim() == 1:
        t = t.reshape(1, k).expand(B, k)
    if tuple(t.shape) != (B, k):
        raise ValueError(f"expected [B, {k}] values, got {tuple(t.shape)}")
    return t.t().contiguous()


def ift_forward_batch(problem, u_star, theta, abstol=1e-8, full=False, n=None, device=None):
    """Batched ift_forward: u_star [B, n], theta [B, m] (or [m], broadcast)."""
    dev = torch.device(device or "cuda")
    u = u_star if isinstance(u_star, torch.Tensor) else torch.as_tensor(np.asarray(u_star, float))
    if u.dim() == 1:
        u = u.reshape(1, -1)
    B = int(u.shape[0])
    h, n, m = _handle(problem, n or int(u.shape[1]))
    us, ts = _soa(u, B, n, dev), _soa(theta, B, m, dev)
    S = torch.empty((n * m, B), dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int8, device=dev)
    res = torch.empty(B, dtype=torch.float64, device=dev) if full else None
    with torch.cuda.device(dev):  # the legacy stream (0) means the current device
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().nlk_ift_forward_batch(
            h, 0, B, us.data_ptr(), ts.data_ptr(), float(abstol), S.data_ptr(),
            None if res is None else res.data_ptr(), st.data_ptr(), stream))
    return BatchSensitivity(S.t().reshape(B, n, m), st, res)


def ift_adjoint_batch(problem, u_star, theta, gbar, abstol=1e-8, full=False, n=None, device=None):
    """Batched ift_adjoint: gbar [B, n] = dg/du at each root."""
    dev = torch.device(device or "cuda")
    u = u_star if isinstance(u_star, torch.Tensor) else torch.as_tensor(np.asarray(u_star, float))
    if u.dim() == 1:
        u = u.reshape(1, -1)
    B = int(u.shape[0])
    h, n, m = _handle(problem, n or int(u.shape[1]))
    us, ts, gs = _soa(u, B, n, dev), _soa(theta, B, m, dev), _soa(gbar, B, n, dev)
    G = torch.empty((m, B), dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int8, device=dev)
    res = torch.empty(B, dtype=torch.float64, device=dev) if full else None
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().nlk_ift_adjoint_batch(
            h, 0, B, us.data_ptr(), ts.data_ptr(), gs.data_ptr(), float(abstol), G.data_ptr(),
            None if res is None else res.data_ptr(), st.data_ptr(), stream))
    return BatchSensitivity(G.t(), st, res)


def _raise_for(code, what):
    if code == NOT_A_ROOT:
        raise ValueError(f"u_star is not a root to the required accuracy ({what})")
    if code == SINGULAR:
        raise SingularMatrix(f"state Jacobian is singular ({what})")
    if code == NONFINITE:
        raise NonFiniteValue(f"dual evaluation failed ({what})")


def ift_forward(problem, u_star, theta, abstol=1e-8, mode=None, full=False):
    """sensitivity.ift_forward (sensitivity.py:40-57) for one system."""
    if mode is not None and getattr(mode, "is_dual", True) is not True:
        raise NotImplementedError("only the dual-number (DUAL_FORWARD) mode runs on the GPU")
    r = ift_forward_batch(problem, np.asarray(u_star, float)[None], np.asarray(theta, float)[None],
                          abstol, full)
    code = int(r.status[0])
    _raise_for(code, "ift_forward")
    S = r.value[0].cpu().numpy()
    return SensitivityResult(S, float(r.solve_residual[0])) if full else S


def ift_adjoint(problem, u_star, theta, gbar, abstol=1e-8, mode=None, full=False):
    """sensitivity.ift_adjoint (sensitivity.py:60-80) for one system."""
    if mode is not None and getattr(mode, "is_dual", True) is not True:
        raise NotImplementedError("only the dual-number (DUAL_FORWARD) mode runs on the GPU")
    r = ift_adjoint_batch(problem, np.asarray(u_star, float)[None], np.asarray(theta, float)[None],
                          np.asarray(gbar, float)[None], abstol, full)
    code = int(r.status[0])
    _raise_for(code, "ift_adjoint")
    g = r.value[0].cpu().numpy()
    return SensitivityResult(g, float(r.solve_residual[0])) if full else g
