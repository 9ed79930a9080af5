"""Synthetic batches for the five BASELINE.json configurations.

Inputs are generated on the host with numpy's PCG64 so the GPU path, the CPU
oracle and the unmodified reference see identical arrays.  A batch is a
sequence of fixed-size chunks; chunk ``c`` of a stream with seed ``s`` is
drawn from ``default_rng(s)`` when ``c == 0`` and ``default_rng([s, c])``
otherwise, so any contiguous shard (one per GPU) or any sample can be
regenerated without materialising the whole 1M-100M batch.

  C1  quadratic n=2, u0 = 1, p ~ U(0.5, 10)^2, seed 0          (NR)
  C2  the 23 suite members, u0 = u0c + s*max(1,|u0c|_inf)*U(-1,1)^n,
      s = 0.1 (stress 1.0), seed 1000 + index                 (NR, TR)
  C3  generalized Rosenbrock n=8/16, u0 ~ U[0,1)^n, seed 0     (Broyden, Klement)
  C4  broyden-tridiagonal n=16, u0 = -1 + 0.1*U(-1,1)^16, seed 4 (DFSane)
  C5  quadratic n=4, u0 = 1, p ~ U(0.5,10)^4, seed 5, alg = i mod 5
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import problems

CHUNK = 1 << 16

C5_ALGS = ("newton-raphson", "trust-region", "broyden", "klement", "dfsane")


def _chunk_rng(seed, c):
    return np.random.default_rng(seed if c == 0 else [seed, c])


def _draw(seed, lo, hi, width, kind, a=0.0, b=1.0):
    """Rows [lo, hi) of the chunked stream; kind 'uniform' draws U(a, b),
    'random' draws U[0, 1)."""
    out = np.empty((hi - lo, width))
    c0, c1 = lo // CHUNK, (hi - 1) // CHUNK
    for c in range(c0, c1 + 1):
        rng = _chunk_rng(seed, c)
        base = c * CHUNK
        s, e = max(lo, base), min(hi, base + CHUNK)
        if kind == "uniform":
            block = rng.uniform(a, b, (e - base, width))
        else:
            block = rng.random((e - base, width))
        out[s - lo:e - lo] = block[s - base:e - base]
    return out


@dataclass
class Batch:
    problem_id: str
    n: int
    u0: np.ndarray          # [B, n]
    p: np.ndarray | None    # [B, m] or None
    lo: int = 0             # global index of row 0


def c1_quadratic(lo, hi, n=2, seed=0):
    p = _draw(seed, lo, hi, n, "uniform", 0.5, 10.0)
    return Batch("quadratic", n, np.ones((hi - lo, n)), p, lo)


def c2_suite(index, lo, hi, sigma=0.1, seed=None):
    name, n, start, _ref, _tags = problems.SUITE[index - 1]
    seed = 1000 + index if seed is None else seed
    scale = sigma * max(1.0, float(np.max(np.abs(start))))
    u0 = start[None, :] + scale * _draw(seed, lo, hi, n, "uniform", -1.0, 1.0)
    return Batch(f"test23/{name}", n, u0, None, lo)


def c3_rosenbrock(n, lo, hi, seed=0):
    return Batch("generalized_rosenbrock", n, _draw(seed, lo, hi, n, "random"), None, lo)


def c4_tridiagonal(lo, hi, n=16, seed=4):
    u0 = -1.0 + 0.1 * _draw(seed, lo, hi, n, "uniform", -1.0, 1.0)
    return Batch("test23/broyden-tridiagonal", n, u0, None, lo)


def c5_quadratic(lo, hi, seed=5):
    b = c1_quadratic(lo, hi, n=4, seed=seed)
    return b


def c5_algorithms(lo, hi):
    return (np.arange(lo, hi) % 5).astype(np.int8)


def shard_bounds(B, world, rank):
    """Contiguous even split, remainder to the first ranks."""
    base, rem = divmod(B, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)
