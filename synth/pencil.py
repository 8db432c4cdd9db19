"""Seeded synthetic r-Hessenberg-triangular pencils (the paper's workload shape).

This module holds NO arithmetic of the method: it only draws random inputs.
It is the one module shared by the oracle tests and the CUDA-path tests/bench.

Recipe (BASELINE.json ``configs``; the paper's own workload
is "randomly generated pencils", fed to stage two as an
r-HT pencil):

* H: N(0,1) entries on and above the diagonal and on the r subdiagonals
  (``H(i,j) = 0`` for ``i > j + r``); complex: Re, Im i.i.d. N(0, 1/2).
* T: upper triangular, N(0,1) strictly-upper entries (complex: N(0,1/2) parts);
  diagonal ``1+|N(0,1)|`` ("abs"), complex ``(1+|N(0,1)|)·e^{iθ}``, θ~U(0,2π),
  or graded ``10^{U(-3,0)}`` ("graded", config 5), or "singular25": ``1+|N(0,1)|`` with a seeded
  quarter of the entries exactly 0 (the paper's saddle-point pencils have 25% infinite
  eigenvalues).
* Q = Z = I.

Generator: numpy's counter-based Philox bit generator, one stream per
(seed, matrix id, column panel) so any column panel can be regenerated alone.
All arrays are Fortran-ordered (column-major), matching the C ABI.
"""
from __future__ import annotations

import numpy as np

PANEL = 512

# BASELINE.json configs[0..4]; seeds fixed a priori.
CONFIGS = {
    1: dict(n=256, r=8, complex=False, tdiag="abs", seed=1001),
    2: dict(n=4096, r=16, complex=False, tdiag="abs", seed=1002),
    3: dict(n=8192, r=32, complex=True, tdiag="abs", seed=1003),
    4: dict(n=16384, r=64, complex=False, tdiag="abs", seed=1004),
    5: dict(n=32768, r=128, complex=False, tdiag="graded", seed=1005),
}

_MID_H, _MID_T, _MID_TD, _MID_TH, _MID_TZ = 1, 2, 3, 4, 5


def _rng(seed: int, mid: int, panel: int) -> np.random.Generator:
    key = (int(seed) << 48) | (mid << 40) | int(panel)
    return np.random.Generator(np.random.Philox(key=key))


def _normal(rng, shape, cplx):
    if cplx:
        s = np.sqrt(0.5)
        return s * rng.standard_normal(shape) + 1j * (s * rng.standard_normal(shape))
    return rng.standard_normal(shape)


def make_pencil(n: int, r: int, complex: bool = False, tdiag: str = "abs", seed: int = 0):
    """Return (H, T): an n x n r-HT pencil, Fortran order, float64 or complex128."""
    dt = np.complex128 if complex else np.float64
    H = np.zeros((n, n), dt, order="F")
    T = np.zeros((n, n), dt, order="F")
    rows = np.arange(n)[:, None]
    for p0 in range(0, n, PANEL):
        p1 = min(n, p0 + PANEL)
        cols = np.arange(p0, p1)[None, :]
        g = _normal(_rng(seed, _MID_H, p0 // PANEL), (n, p1 - p0), complex)
        g[rows > cols + r] = 0.0
        H[:, p0:p1] = g
        g = _normal(_rng(seed, _MID_T, p0 // PANEL), (n, p1 - p0), complex)
        g[rows >= cols] = 0.0
        T[:, p0:p1] = g
    rd = _rng(seed, _MID_TD, 0)
    if tdiag == "graded":
        d = 10.0 ** rd.uniform(-3.0, 0.0, n)
    else:
        d = 1.0 + np.abs(rd.standard_normal(n))
    if tdiag == "singular25":
        # saddle-point-like pencil (25% infinite eigenvalues): a seeded quarter of
        # T's diagonal is exactly zero, so T is singular and the pencil has n/4 infinite eigenvalues
        zero = _rng(seed, _MID_TZ, 0).permutation(n)[: n // 4]
        d[zero] = 0.0
    if complex:
        theta = _rng(seed, _MID_TH, 0).uniform(0.0, 2.0 * np.pi, n)
        d = d * np.exp(1j * theta)
    T[np.arange(n), np.arange(n)] = d
    return H, T


def config_pencil(cfg: int, n: int | None = None):
    """Pencil of BASELINE config ``cfg`` (optionally at a reduced n, same r/field/seed)."""
    c = CONFIGS[cfg]
    return make_pencil(n or c["n"], c["r"], c["complex"], c["tdiag"], c["seed"])
