"""Independent Moler-Stewart Hessenberg-triangular reduction by Givens rotations.

TEST-ONLY second algorithm used to pin the oracle (SURVEY.md §8(c) pin 1;
PAPER.md:15 cites Moler & Stewart, "Traditionally, stage two ...
has been implemented using Givens rotations").  Shares no code with oracle/.

GVL-style: for j = 1..n-2, for i = n down to j+2: a row rotation on (i-1, i)
zeroes A(i, j); the fill it creates at B(i, i-1) is removed by a column
rotation on (i-1, i).  Output satisfies A_in = Q A Z^*, B_in = Q B Z^*,
with Q e1 = Z e1 = e1.  Works on any pencil with B upper triangular.
"""
from __future__ import annotations

import numpy as np


def _row_rot(a, b):
    """G = [[c, s], [-conj(s), c]], c real, with G [a; b] = [rho; 0]."""
    if b == 0:
        return 1.0, 0.0 * a
    if a == 0:
        return 0.0, 1.0 + 0.0 * a
    nu = np.sqrt(abs(a) ** 2 + abs(b) ** 2)
    c = abs(a) / nu
    s = (a / abs(a)) * np.conj(b) / nu
    return c, s


def _col_rot(x, y):
    """G = [[c, s], [-conj(s), c]] with [x, y] G = [0, *]."""
    if x == 0:
        return 1.0, 0.0 * x
    if y == 0:
        return 0.0, 1.0 + 0.0 * x
    nu = np.sqrt(abs(x) ** 2 + abs(y) ** 2)
    c = abs(y) / nu
    s = np.conj(x) * abs(y) / (np.conj(y) * nu)
    return c, s


def givens_ht(A, B):
    A = np.array(A, dtype=np.result_type(A, B, np.float64), copy=True)
    B = np.array(B, dtype=A.dtype, copy=True)
    n = A.shape[0]
    Q = np.eye(n, dtype=A.dtype)
    Z = np.eye(n, dtype=A.dtype)
    for j in range(n - 2):                      # 0-based column j (paper j+1)
        for i in range(n - 1, j + 1, -1):       # zero A(i, j), rows (i-1, i)
            if A[i, j] == 0:
                continue
            c, s = _row_rot(A[i - 1, j], A[i, j])
            G = np.array([[c, s], [-np.conj(s), c]], dtype=A.dtype)
            A[i - 1:i + 1, j:] = G @ A[i - 1:i + 1, j:]
            A[i, j] = 0.0
            B[i - 1:i + 1, i - 1:] = G @ B[i - 1:i + 1, i - 1:]
            Q[:, i - 1:i + 1] = Q[:, i - 1:i + 1] @ G.conj().T
            c, s = _col_rot(B[i, i - 1], B[i, i])
            G2 = np.array([[c, s], [-np.conj(s), c]], dtype=A.dtype)
            B[:i + 1, i - 1:i + 1] = B[:i + 1, i - 1:i + 1] @ G2
            B[i, i - 1] = 0.0
            A[:, i - 1:i + 1] = A[:, i - 1:i + 1] @ G2
            Z[:, i - 1:i + 1] = Z[:, i - 1:i + 1] @ G2
    return A, B, Q, Z
