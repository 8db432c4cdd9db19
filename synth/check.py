"""Result checks for HT reductions (test/bench infrastructure; not the method).

* ``invariants`` -- north_star's bounds (BASELINE.json): relative backward errors
  ||A - Q H Z^*||_F/||A||_F and ||B - Q T Z^*||_F/||B||_F, orthogonality
  ||Q^*Q - I||_F, ||Z^*Z - I||_F, and exact-zero structure of (H, T).
* ``normalize_phase`` -- reading c10: the diagonal
  sign/phase scaling that makes T_ii > 0 (i >= 2) and H_{i+1,i} > 0, used to
  compare two correct reductions (unique up to that scaling, reading c9).
"""
from __future__ import annotations

import numpy as np

U = 2.0 ** -53  # unit roundoff (reading c11)


def structure_violations(H, T) -> int:
    """Number of entries that must be exactly 0 but are not (below H's first
    subdiagonal, below T's diagonal)."""
    H = np.asarray(H)
    T = np.asarray(T)
    n = H.shape[0]
    i, j = np.indices((n, n))
    return int(np.count_nonzero(H[i > j + 1]) + np.count_nonzero(T[i > j]))


def invariants(A, B, H, T, Q, Z):
    """Return dict(eA, eB, oQ, oZ, zeros_bad, bound) -- numpy, fp64."""
    n = A.shape[0]
    eA = np.linalg.norm(A - Q @ H @ Z.conj().T) / max(np.linalg.norm(A), 1e-300)
    eB = np.linalg.norm(B - Q @ T @ Z.conj().T) / max(np.linalg.norm(B), 1e-300)
    I = np.eye(n)
    oQ = np.linalg.norm(Q.conj().T @ Q - I)
    oZ = np.linalg.norm(Z.conj().T @ Z - I)
    return dict(eA=float(eA), eB=float(eB), oQ=float(oQ), oZ=float(oZ),
                zeros_bad=structure_violations(H, T), bound=10.0 * n * U)


def phase_factors(H, T):
    """Reading c10: dq_1 = dz_1 = 1; for i = 1..n: if i>=2 and T_ii != 0,
    dz_i = dq_i |T_ii|/T_ii; if i<n and H_{i+1,i} != 0,
    dq_{i+1} = H_{i+1,i} dz_i / |H_{i+1,i} dz_i|.  Zero entries keep d = 1."""
    H = np.asarray(H)
    T = np.asarray(T)
    return phase_factors_diag(np.diagonal(H, -1), np.diagonal(T))


def phase_factors_diag(hsub, tdiag):
    """phase_factors from H's first subdiagonal (n-1) and T's diagonal (n) alone."""
    hsub = np.asarray(hsub)
    tdiag = np.asarray(tdiag)
    n = tdiag.shape[0]
    cplx = np.iscomplexobj(hsub) or np.iscomplexobj(tdiag)
    dt = np.complex128 if cplx else np.float64
    dq = np.ones(n, dt)
    dz = np.ones(n, dt)
    for i in range(n):
        if i >= 1 and tdiag[i] != 0:
            dz[i] = dq[i] * abs(tdiag[i]) / tdiag[i]
        if i < n - 1 and hsub[i] != 0:
            h = hsub[i] * dz[i]
            dq[i + 1] = h / abs(h)
    return dq, dz


def normalize_phase(H, T, Q=None, Z=None):
    """Apply reading c10: H' = D_Q^* H D_Z, T' = D_Q^* T D_Z, Q' = Q D_Q, Z' = Z D_Z."""
    dq, dz = phase_factors(H, T)
    Hn = (dq.conj()[:, None] * np.asarray(H)) * dz[None, :]
    Tn = (dq.conj()[:, None] * np.asarray(T)) * dz[None, :]
    Qn = None if Q is None else np.asarray(Q) * dq[None, :]
    Zn = None if Z is None else np.asarray(Z) * dz[None, :]
    return Hn, Tn, Qn, Zn


def rel_diff(X, Y) -> float:
    """||X - Y||_F / ||Y||_F."""
    return float(np.linalg.norm(np.asarray(X) - np.asarray(Y)) / max(np.linalg.norm(Y), 1e-300))


def forward_gap(H1, T1, H2, T2):
    """Max of the relative Frobenius differences of the c10-normalised H and T."""
    a = normalize_phase(H1, T1)
    b = normalize_phase(H2, T2)
    return max(rel_diff(a[0], b[0]), rel_diff(a[1], b[1]))


def normalise_samples(raw: dict, dq, dz, cols, rows) -> dict:
    """Reading c10 applied to sampled columns / rows only (full-size comparisons).

    raw[name] = (X[:, cols], X[rows, :]) for name in H, T, Q, Z (raw, un-normalised);
    returns {name_cols, name_rows} of H' = D_Q^* H D_Z, T' = D_Q^* T D_Z, Q' = Q D_Q, Z' = Z D_Z."""
    cols = np.asarray(cols)
    rows = np.asarray(rows)
    out = {}
    for nm, dl, dr in (("H", dq, dz), ("T", dq, dz), ("Q", None, dq), ("Z", None, dz)):
        c, rr = raw[nm]
        c = np.asarray(c) * dr[cols][None, :]
        rr = np.asarray(rr) * dr[None, :]
        if dl is not None:
            c = dl.conj()[:, None] * c
            rr = dl.conj()[rows][:, None] * rr
        out[nm + "_cols"] = c
        out[nm + "_rows"] = rr
    return out


def sample_rel_diff(a: dict, b: dict, nm: str) -> float:
    """Relative Frobenius difference of the sampled entries of matrix nm (b is the reference)."""
    num = np.linalg.norm(a[nm + "_cols"] - b[nm + "_cols"]) ** 2 + np.linalg.norm(a[nm + "_rows"] - b[nm + "_rows"]) ** 2
    den = np.linalg.norm(b[nm + "_cols"]) ** 2 + np.linalg.norm(b[nm + "_rows"]) ** 2
    return float(np.sqrt(num / max(den, 1e-300)))
