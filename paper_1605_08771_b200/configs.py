"""The five BASELINE.json configurations.

Seeded synthetic stand-ins for the reference's benchmark matrices; the
reference ships no data files. Decisions recorded in DESIGN.md:
  Q seed 1000+cfg (Householder QR of a mt19937_64 N(0,1) block, column signs
  normalised as proj/src/matmodel.cpp:93-104), Lambda seed 2000+cfg
  (std::uniform_real_distribution on mt19937_64), X0 = make_initial_guess(seed 42).
  cfg1: s = 2 for XFEAST/RFEAST; cfg2: Lambda gap (-0.31,-0.3) by
  reject-resample; cfg3: the better-conditioned endpoints of Appendix A and
  tol = 1e-12 * lambda_max; tol 1e-10 elsewhere.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    index: int
    name: str
    n: int
    lo: float
    hi: float
    n_c: int
    tol: float
    max_iter: int
    s: int = 2
    m0: int | None = None  # None: 1.5 x true count (cfg1)


CONFIGS = {
    0: Config(0, "cfg0-n1000-uniform", 1000, -0.1, 0.1, 8, 1e-10, 20, m0=150),
    1: Config(1, "cfg1-n2000-hard-edge", 2000, -0.1, 0.1, 8, 1e-10, 20, s=2, m0=None),
    2: Config(2, "cfg2-n4096-gap", 4096, -0.3, 0.2, 16, 1e-10, 20, m0=768),
    3: Config(3, "cfg3-laplace96", 9216, 0.0, 0.0, 8, 0.0, 20, m0=300),
    4: Config(4, "cfg4-n16384-uniform", 16384, -0.02, 0.02, 32, 1e-10, 20, m0=512),
}


def laplacian_eigenvalues(m: int = 96):
    h = 1.0 / (m + 1)
    j = np.arange(1, m + 1)
    s = np.sin(j * math.pi * h / 2.0) ** 2
    return np.sort((4.0 / h ** 2) * (s[:, None] + s[None, :]).ravel())


def cfg3_interval():
    """Appendix A, better-conditioned choice: 200 inside, no split pair."""
    lam = laplacian_eigenvalues()
    lo = 0.5 * (lam[919] + lam[920])
    hi = 0.5 * (lam[1119] + lam[1120])
    return lo, hi, 1e-12 * lam[-1]


def spectrum(index: int, uniform_fill) -> np.ndarray:
    """Eigenvalues (ascending) of config `index`; uniform_fill(count, lo, hi, seed)."""
    seed = 2000 + index
    if index in (0, 4):
        n = CONFIGS[index].n
        return np.sort(uniform_fill(n, -1.0, 1.0, seed))
    if index == 1:
        a = uniform_fill(1400, -1.0, 1.0, seed)
        b = uniform_fill(300, 0.098, 0.102, seed + 100)
        c = uniform_fill(300, -0.102, -0.098, seed + 200)
        return np.sort(np.concatenate([a, b, c]))
    if index == 2:
        out = []
        k = 0
        while len(out) < 4096:
            batch = uniform_fill(8192, -2.0, 2.0, seed + k)
            out.extend(v for v in batch if not (-0.31 < v < -0.3))
            k += 1
        return np.sort(np.array(out[:4096]))
    if index == 3:
        return laplacian_eigenvalues()
    raise ValueError(index)


def resolved(index: int, values: np.ndarray) -> dict:
    """lo/hi/tol/m0 with the data-dependent choices filled in."""
    c = CONFIGS[index]
    lo, hi, tol = c.lo, c.hi, c.tol
    if index == 3:
        lo, hi, tol = cfg3_interval()
    inside = int(np.count_nonzero((values > lo) & (values < hi)))
    m0 = c.m0 if c.m0 is not None else int(round(1.5 * inside))
    return dict(n=c.n, lo=lo, hi=hi, tol=tol, m0=m0, n_c=c.n_c, max_iter=c.max_iter, s=c.s,
                inside=inside)


def laplacian_2d(m: int = 96) -> np.ndarray:
    """Dense 5-point Dirichlet Laplacian (1/h^2)(4, -1 neighbours), n = m^2."""
    h = 1.0 / (m + 1)
    n = m * m
    A = np.zeros((n, n), order="F")
    idx = np.arange(n)
    A[idx, idx] = 4.0
    r = idx % m
    right = idx[r < m - 1]
    A[right, right + 1] = -1.0
    A[right + 1, right] = -1.0
    down = idx[idx < n - m]
    A[down, down + m] = -1.0
    A[down + m, down] = -1.0
    return A / (h * h)
