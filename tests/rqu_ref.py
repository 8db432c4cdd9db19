"""Unblocked stage two on the CPU (numpy) with the opposite reflector from an UPDATED RQ
factorisation -- TEST-ONLY model of the CUDA chase's "RQ update" path.

Alg. 2 computes the opposite reflector Z_k^j from an RQ factorisation of
the m x m block B' = Q^* B0 (B0 = B(i1:i2, i1:i2) before the left reflector Q = I - tau v v^*,
reading c3/c4), which costs O(m^3) on the chase's critical path.  The block's leading
(m-1) x (m-1) part B1 = B0(1:m-1, 1:m-1) is the trailing part of the PREVIOUS sweep's reduced
block at the same step k: B'_prev Z_prev = R~ (Q~ Z_prev), whose rows/columns 2..m are
R~(2:m, 2:m) W with W = (Q~ Z_prev)(2:m, 2:m) -- an RQ factorisation handed from sweep j-1 to
sweep j.  With it, B0 = [[R1, b'], [0, beta]] diag(W, 1) (the last row of B1's columns is zero,
the last column b is the caught-up column i2), and

    Q^* B0 = (R0 - v w^*) Q0,   w = tau^* R0^* v   (rank-one update of the triangular R0),

whose RQ follows from 2(m-1) Givens column rotations (reduce w to a multiple of e_m, which turns
R0 into upper Hessenberg; subtract the rank-one part from the last column; restore the
triangle bottom-up).  Q~ = G^T Q0 (rows rotated), Z_k^j = larfg(conj(Q~(1,:))^T) as in c3.
O(m^2) per step instead of O(m^3).

The first sweep of every group starts from a fresh Householder RQ of B1 (`fresh`), like the
CUDA path's per-group prologue.  Shares no code with oracle/.
"""
from __future__ import annotations

import numpy as np


def house(x):
    """xLARFG convention (reading c1): v (v[0]=1), tau, beta."""
    x = np.asarray(x, dtype=np.float64)
    m = x.shape[0]
    alpha = x[0]
    xn2 = float(np.sum(x[1:] ** 2)) if m > 1 else 0.0
    v = np.zeros(m)
    v[0] = 1.0
    if xn2 == 0.0:
        return v, 0.0, alpha
    nrm = np.sqrt(alpha * alpha + xn2)
    beta = -nrm if alpha >= 0 else nrm
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def rq_full(C):
    """Householder RQ (rows bottom-up) with Q formed explicitly: C = R Q."""
    C = np.array(C, dtype=np.float64, copy=True)
    m = C.shape[0]
    P = np.eye(m)  # accumulates the right factors: C P = R  ->  Q = P^T
    for i in range(m - 1, 0, -1):
        x = np.concatenate(([C[i, i]], C[i, :i]))
        vv, tau, beta = house(x)
        h = np.concatenate((vv[1:], [1.0]))  # over columns 0..i (pivot last)
        C[:, :i + 1] -= tau * np.outer(C[:, :i + 1] @ h, h)
        P[:, :i + 1] -= tau * np.outer(P[:, :i + 1] @ h, h)
        C[i, :i] = 0.0
    return np.triu(C), P.T


def rot(a, b):
    """(c, s) with [a, b] [[c, s], [-s, c]] = [0, rho], rho = hypot(a, b) >= 0."""
    rho = np.hypot(a, b)
    if rho == 0.0:
        return 1.0, 0.0, 0.0
    return b / rho, a / rho, rho


def rq_update(R0, Q0, v, tau):
    """RQ of (I - tau v v^T)^T R0 Q0 = (R0 - v w^T) Q0 by 2(m-1) Givens column rotations.
    Returns (R~, Q~) with Q^T B0 = R~ Q~."""
    m = R0.shape[0]
    w = tau * (R0.T @ v)
    Hs = np.array(R0, copy=True)
    Qt = np.array(Q0, copy=True)
    # (1) reduce w^T to rho e_m^T: rotation i on columns (i, i+1), ascending
    p = w[0]
    cs = []
    for i in range(m - 1):
        c, s, rho = rot(p, w[i + 1])
        cs.append((c, s))
        p = rho
        xi, xj = Hs[:, i].copy(), Hs[:, i + 1].copy()
        Hs[:, i], Hs[:, i + 1] = xi * c - xj * s, xi * s + xj * c
        yi, yj = Qt[i].copy(), Qt[i + 1].copy()  # G^T on the rows of Q0
        Qt[i], Qt[i + 1] = c * yi - s * yj, s * yi + c * yj
    Hs[:, m - 1] -= v * p
    # (2) upper Hessenberg -> triangular, bottom-up
    for i in range(m - 2, -1, -1):
        c, s, rho = rot(Hs[i + 1, i], Hs[i + 1, i + 1])
        xi, xj = Hs[:, i].copy(), Hs[:, i + 1].copy()
        Hs[:, i], Hs[:, i + 1] = xi * c - xj * s, xi * s + xj * c
        Hs[i + 1, i] = 0.0
        yi, yj = Qt[i].copy(), Qt[i + 1].copy()
        Qt[i], Qt[i + 1] = c * yi - s * yj, s * yi + c * yj
    return Hs, Qt


def stage2_rqu(A, B, r, q=None, check=False):
    """Alg. 2 with the opposite reflector from the handed-over RQ factorisation.
    q: sweeps per group (fresh RQ for the first sweep of each group; None = only sweep 1).
    Returns H, T, Q, Z and the largest relative mismatch ||B1 - R1 W|| / ||B1|| seen (check)."""
    A = np.array(A, dtype=np.float64, order="F", copy=True)
    B = np.array(B, dtype=np.float64, order="F", copy=True)
    n = A.shape[0]
    Q = np.eye(n)
    Z = np.eye(n)
    F = {}  # step k -> (R1, W): RQ of the next sweep's leading block
    worst = 0.0
    for j in range(1, n - 1):
        fresh = (j == 1) if q is None else ((j - 1) % q == 0)
        Fn = {}
        for k in range(0, (n - j - 2) // r + 1):
            jb = j + max(0, (k - 1) * r + 1)
            i1 = j + k * r + 1
            i2 = min(j + (k + 1) * r, n)
            i3 = min(j + (k + 2) * r, n)
            m = i2 - i1 + 1
            a0, a1 = i1 - 1, i2  # 0-based slice of the block
            hasB = (i1 + r - 1) <= n
            f = m - 1 if hasB else m
            B0 = B[a0:a1, a0:a1].copy()
            if check:
                assert np.all(B0[m - 1, :m - 1] == 0.0) or not hasB, "last row of B1 not zero"
            if fresh or k not in F:
                R1, W = rq_full(B0[:f, :f])
            else:
                R1, W = F[k]
                assert R1.shape[0] == f, (j, k, R1.shape, f)
                if check:
                    nb = np.linalg.norm(B0[:f, :f])
                    if nb > 0:
                        worst = max(worst, np.linalg.norm(B0[:f, :f] - R1 @ W) / nb)
            R0 = np.zeros((m, m))
            Q0 = np.eye(m)
            R0[:f, :f] = R1
            Q0[:f, :f] = W
            if hasB:
                R0[:, m - 1] = B0[:, m - 1]
            # left reflector (Alg. 2 lines 17-19)
            v, tau, beta = house(A[a0:a1, jb - 1])
            A[a0:a1, jb - 1:] -= tau * np.outer(v, v @ A[a0:a1, jb - 1:])
            A[a0 + 1:a1, jb - 1] = 0.0
            A[a0, jb - 1] = beta
            B[a0:a1, a0:] -= tau * np.outer(v, v @ B[a0:a1, a0:])
            Q[:, a0:a1] -= tau * np.outer(Q[:, a0:a1] @ v, v)
            # opposite reflector from the updated factorisation
            Rt, Qt = rq_update(R0, Q0, v, tau)
            z, sig, _ = house(Qt[0, :])
            A[:i3, a0:a1] -= sig * np.outer(A[:i3, a0:a1] @ z, z)
            B[:i2, a0:a1] -= sig * np.outer(B[:i2, a0:a1] @ z, z)
            Z[:, a0:a1] -= sig * np.outer(Z[:, a0:a1] @ z, z)
            B[a0 + 1:a1, a0] = 0.0
            # hand-over: rows/columns 2..m of R~ and of Q~ Z
            QZ = Qt - sig * np.outer(Qt @ z, z)
            Fn[k] = (np.triu(Rt[1:, 1:]), QZ[1:, 1:])
        F = Fn
    return A, B, Q, Z, worst
