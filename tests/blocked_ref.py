"""Blocked stage two on the CPU (numpy) -- TEST-ONLY second reference ordering.

Implements the paper's blocked algorithm (Alg. 3 "Generate", PAPER.md:1843-1877,
and Alg. 4 "Apply") with the index corrections of
SURVEY.md App. A.2-A.3 (readings c8), in the SAME decomposition
the CUDA path uses:

* generate: per group of q sweeps, the catch-up of earlier sweeps' left
  reflectors on column jb (and B column i1+r-1) is applied as one mat-vec with
  the partial dense product U_k = Q_k^{j1} ... Q_k^{j-1} (instead of reflector
  by reflector), U_k and V_k are accumulated densely as reflectors are made;
* apply: staircase remainder reflector by reflector, then dense w x w blocks
  U_k, V_k in descending k.

It shares no code with oracle/ (own Householder and RQ, RQ by the
accumulated-P variant).  Uses: (1) design check of the blocked schedule the
kernels implement; (2) the "noise floor" of SURVEY §8(c) pin 7 -- the gap
between two correct CPU orderings on the real seeds.
"""
from __future__ import annotations

import numpy as np


def _house(x):
    """xLARFG convention (reading c1): returns v (v[0]=1), tau, beta."""
    x = np.asarray(x)
    m = x.shape[0]
    alpha = x[0]
    xn2 = float(np.sum(np.abs(x[1:]) ** 2)) if m > 1 else 0.0
    v = np.zeros(m, x.dtype)
    v[0] = 1
    if xn2 == 0.0 and np.imag(alpha) == 0:
        return v, 0.0 * alpha, np.real(alpha)
    nrm = np.sqrt(abs(alpha) ** 2 + xn2)
    beta = -nrm if np.real(alpha) >= 0 else nrm
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def _opposite(C):
    """Direction of the opposite reflector: conj(first row of Q~) where C = R~ Q~,
    by Householder RQ (rows bottom-up) with the product P = H_m ... H_2
    accumulated alongside (P e1 = Q~^* e1)."""
    C = np.array(C, copy=True)
    m = C.shape[0]
    P = np.eye(m, dtype=C.dtype)
    for i in range(m - 1, 0, -1):
        x = np.concatenate(([np.conj(C[i, i])], np.conj(C[i, :i])))
        vv, tau, beta = _house(x)
        h = np.concatenate((vv[1:], [1.0]))  # over columns 0..i
        S = np.vstack((C[:i, :i + 1], P[:, :i + 1]))
        S -= tau * np.outer(S @ h, h.conj())
        C[:i, :i + 1] = S[:i]
        P[:, :i + 1] = S[i:]
        C[i, :i] = 0
        C[i, i] = beta
    return P[:, 0]  # = Q~^* e1 = conj(Q~(1,:))^T


def blocked_stage2(H, T, r, q, Q=None, Z=None):
    dt = np.result_type(H, T, np.float64)
    A = np.array(H, dtype=dt, copy=True)
    B = np.array(T, dtype=dt, copy=True)
    n = A.shape[0]
    Q = np.eye(n, dtype=dt) if Q is None else np.array(Q, dtype=dt, copy=True)
    Z = np.eye(n, dtype=dt) if Z is None else np.array(Z, dtype=dt, copy=True)
    if n <= 2 or r <= 1:
        return A, B, Q, Z
    j1 = 1
    while j1 <= n - 2:
        qp = min(q, n - 1 - j1)
        K = 1 + (n - j1 - 2) // r
        base = [j1 + k * r + 1 for k in range(K)]               # first row/col of window k
        wk = [min(qp + r - 1, n - base[k] + 1) for k in range(K)]
        U = [np.eye(wk[k], dtype=dt) for k in range(K)]
        V = [np.eye(wk[k], dtype=dt) for k in range(K)]
        zref = {}
        # ---------------- generate (Alg. 3, corrected i4) ----------------
        for j in range(j1, j1 + qp):
            t = j - j1
            for k in range(min(K, 2 + (n - j - 1) // r)):
                jb = j + max(0, (k - 1) * r + 1)
                i1 = j + k * r + 1
                i2 = min(j + (k + 1) * r, n)
                i3 = min(j + (k + 2) * r, n)
                i4 = j1 + 1 + max(0, (k + j - j1 - qp + 1) * r)
                b0 = base[k]
                if t > 0:  # catch-up of Q_k^{j1..j-1} (Alg. 3 lines 9-16) as one mat-vec
                    L = min(j - 1 + (k + 1) * r, n) - b0 + 1
                    if L >= 1 and jb <= n:
                        Ut = U[k][:L, :L].conj().T
                        A[b0 - 1:b0 - 1 + L, jb - 1] = Ut @ A[b0 - 1:b0 - 1 + L, jb - 1]
                        if i1 + r - 1 <= n:
                            c = i1 + r - 1
                            B[b0 - 1:b0 - 1 + L, c - 1] = Ut @ B[b0 - 1:b0 - 1 + L, c - 1]
                m = i2 - i1 + 1
                if m < 2:
                    continue
                v, tau, beta = _house(A[i1 - 1:i2, jb - 1])
                A[i1 - 1:i2, jb - 1] = 0
                A[i1 - 1, jb - 1] = beta
                blk = B[i1 - 1:i2, i1 - 1:i2]
                blk -= np.conj(tau) * np.outer(v, v.conj() @ blk)
                Uk = U[k][:, t:t + m]
                Uk -= tau * np.outer(Uk @ v, v.conj())
                y = _opposite(B[i1 - 1:i2, i1 - 1:i2])
                wv, sig, _ = _house(y)
                for M, r0, r1 in ((A, i4, i3), (B, i4, i2)):
                    S = M[r0 - 1:r1, i1 - 1:i2]
                    S -= sig * np.outer(S @ wv, wv.conj())
                B[i1:i2, i1 - 1] = 0
                Vk = V[k][:, t:t + m]
                Vk -= sig * np.outer(Vk @ wv, wv.conj())
                zref[(t, k)] = (wv, sig, i1, i2)
        # ---------------- apply (Alg. 4, corrected) ----------------
        for k in range(K - 1, -1, -1):
            i5s = j1 + 1 + max(0, (k - qp + 1) * r)
            for t in range(1, qp):
                if (t, k) not in zref:
                    continue
                wv, sig, i1, i2 = zref[(t, k)]
                i4a = j1 + max(0, (k + t - qp + 1) * r)
                if i4a >= i5s:
                    for M in (A, B):
                        S = M[i5s - 1:i4a, i1 - 1:i2]
                        S -= sig * np.outer(S @ wv, wv.conj())
            c0, c1 = base[k], base[k] + wk[k] - 1
            i5b = j1 + max(0, (k - qp + 1) * r)
            A[:i5b, c0 - 1:c1] = A[:i5b, c0 - 1:c1] @ V[k]
            B[:i5b, c0 - 1:c1] = B[:i5b, c0 - 1:c1] @ V[k]
            Z[:, c0 - 1:c1] = Z[:, c0 - 1:c1] @ V[k]
        for k in range(K - 1, -1, -1):
            c0, c1 = base[k], base[k] + wk[k] - 1
            i5 = j1 + qp - 1 + max(0, (k - 1) * r + 1)
            i6 = j1 + qp + (k + 1) * r - 1
            Uh = U[k].conj().T
            A[c0 - 1:c1, i5:] = Uh @ A[c0 - 1:c1, i5:]
            B[c0 - 1:c1, i6:] = Uh @ B[c0 - 1:c1, i6:]
            Q[:, c0 - 1:c1] = Q[:, c0 - 1:c1] @ U[k]
        j1 += qp
    return A, B, Q, Z
