"""Pins for the CPU oracle (oracle/, Alg. 2 of PAPER.md:1813-1841).

Each test pins the oracle to something other than itself: a closed form, a
library routine on a special case, an independent algorithm (Moler-Stewart
Givens, tests/givens_ref.py), invariants the mathematics fixes, or the
sparsity traces of the paper's Fig. 5.
"""
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
from givens_ref import givens_ht
from synth.check import U, invariants, normalize_phase, rel_diff, structure_violations
from synth.pencil import make_pencil

# ----------------------------------------------------------------------------- larfg


def test_larfg_closed_form_3_4():
    # reading c1 (xLARFG): beta = -sign(alpha)||x|| = -5, v = x/(alpha-beta) = [1, 4/8],
    # tau = (beta-alpha)/beta = 8/5   (SPEC.md:58 example; SURVEY §8(c) pin 3)
    v, tau, beta = oracle.larfg(np.array([3.0, 4.0]))
    assert beta == -5.0
    assert tau == 1.6
    assert np.array_equal(v, np.array([1.0, 0.5]))


def test_larfg_negative_alpha_sign():
    v, tau, beta = oracle.larfg(np.array([-3.0, 4.0]))
    assert beta == 5.0  # -sign(-3)*5
    H = np.eye(2) - tau * np.outer(v, v)
    assert np.allclose(H.T @ np.array([-3.0, 4.0]), [5.0, 0.0], atol=1e-15)


@pytest.mark.parametrize("x,beta", [(np.array([2.5]), 2.5), (np.zeros(3), 0.0), (np.array([-1.0, 0.0, 0.0]), -1.0)])
def test_larfg_trivial_tau_zero(x, beta):
    v, tau, b = oracle.larfg(x)
    assert tau == 0.0 and b == beta and v[0] == 1.0


@pytest.mark.parametrize("cplx", [False, True])
def test_larfg_annihilates_and_unitary(cplx):
    rng = np.random.default_rng(5)
    for m in (2, 3, 7, 16, 33):
        x = rng.standard_normal(m) + (1j * rng.standard_normal(m) if cplx else 0)
        v, tau, beta = oracle.larfg(x)
        H = np.eye(m) - tau * np.outer(v, v.conj())
        y = H.conj().T @ x
        assert abs(y[0] - beta) < 1e-14 * np.linalg.norm(x)
        assert np.linalg.norm(y[1:]) < 1e-14 * np.linalg.norm(x)
        assert np.linalg.norm(H.conj().T @ H - np.eye(m)) < 1e-14
        assert abs(abs(beta) - np.linalg.norm(x)) < 1e-14 * np.linalg.norm(x)


# ----------------------------------------------------------------------------- RQ / opposite reflector


@pytest.mark.parametrize("cplx", [False, True])
def test_rq_first_row_is_direction_of_inverse(cplx):
    # reading c3: conj(Q~(1,:))^T = Q~^* e1 = R~11 B^{-1} e1 -- checked against a library solve
    rng = np.random.default_rng(11)
    for m in (2, 3, 8, 16):
        C = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
        y, R = oracle.rq_first_row(C)
        assert abs(np.linalg.norm(y) - 1) < 1e-14
        assert np.allclose(np.tril(R, -1), 0, atol=0)  # exact zeros below diagonal
        x = np.linalg.solve(C, np.eye(m)[:, 0])
        x = x / np.linalg.norm(x)
        ph = np.vdot(x, y.conj())
        assert abs(abs(ph) - 1) < 1e-12
        assert np.linalg.norm(y.conj() - ph * x) < 1e-12


def test_rq_2x2_permutation():
    # SPEC.md:117 example: [[0,1],[1,0]] -> |R11| = |R22| = 1
    y, R = oracle.rq_first_row(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert abs(abs(R[0, 0]) - 1) < 1e-15 and abs(abs(R[1, 1]) - 1) < 1e-15 and R[1, 0] == 0
    assert abs(abs(y[1]) - 1) < 1e-15 and abs(y[0]) < 1e-15


@pytest.mark.parametrize("cplx", [False, True])
def test_rq_singular_block(cplx):
    # reading c4 / SURVEY [V5]: RQ stays well defined on singular blocks; conj(y) is
    # orthogonal to rows 2..m of C (the property B_blk Z e1 ∝ e1 needs)
    rng = np.random.default_rng(3)
    m = 6
    C = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
    C[:, 2] = C[:, 0] + C[:, 1]  # rank deficient
    y, R = oracle.rq_first_row(C)
    assert np.all(np.isfinite(y))
    assert np.linalg.norm(C[1:, :] @ y.conj()) < 1e-13 * np.linalg.norm(C)


# ----------------------------------------------------------------------------- trivial cases


@pytest.mark.parametrize("n,r", [(8, 1), (8, 0), (2, 5), (1, 3), (0, 2)])
def test_trivial_cases_exact_noop(n, r):
    # SURVEY §8(b) "n <= 2 or r <= 1 is an exact no-op"; r = 1 is already HT
    H, T = make_pencil(max(n, 1), max(r, 1), seed=1)
    H, T = H[:n, :n].copy(order="F"), T[:n, :n].copy(order="F")
    if r == 0:
        H = np.triu(H).copy(order="F")
    h, t, q, z, _ = oracle.stage2(H, T, r)
    assert np.array_equal(h, H) and np.array_equal(t, T)
    assert np.array_equal(q, np.eye(n)) and np.array_equal(z, np.eye(n))


def test_n3_r2_single_step():
    # n = 3, r = 2 is exactly one step (j,k) = (1,0)
    H, T = make_pencil(3, 2, seed=2)
    h, t, q, z, _ = oracle.stage2(H, T, 2)
    inv = invariants(H, T, h, t, q, z)
    assert inv["zeros_bad"] == 0 and h[2, 0] == 0 and t[2, 1] == 0
    assert inv["eA"] < inv["bound"] and inv["eB"] < inv["bound"]
    g = givens_ht(H, T)
    a, b = normalize_phase(h, t, q, z), normalize_phase(*g)
    for x, y in zip(a, b):
        assert rel_diff(x, y) < 1e-14


# ----------------------------------------------------------------------------- independent algorithm


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("n,r", [(6, 2), (20, 3), (48, 5), (64, 8), (90, 13)])
def test_matches_moler_stewart_givens(cplx, n, r):
    # SURVEY §8(c) pin 1: unique up to diagonal phase (reading c9) -> compare after c10
    H, T = make_pencil(n, r, cplx, seed=100 + n)
    h, t, q, z, _ = oracle.stage2(H, T, r)
    g = givens_ht(H, T)
    a, b = normalize_phase(h, t, q, z), normalize_phase(*g)
    tol = 200 * n * U
    for x, y in zip(a, b):
        assert rel_diff(x, y) < tol


@pytest.mark.parametrize("cplx", [False, True])
def test_b_identity_is_lapack_gehrd(cplx):
    # SURVEY §8(c) pin 2: with B = I the reduction IS the Hessenberg reduction of A
    # (LAPACK xGEHRD via scipy.linalg.hessenberg), T stays diagonal unitary.
    n, r = 60, 7
    H, _ = make_pencil(n, r, cplx, seed=9)
    T = np.eye(n, dtype=H.dtype)
    h, t, q, z, _ = oracle.stage2(H, T, r)
    assert np.linalg.norm(t - np.diag(np.diag(t))) < 50 * n * U
    assert np.allclose(np.abs(np.diag(t)), 1, atol=50 * n * U)
    Hs, Qs = scipy.linalg.hessenberg(H, calc_q=True)
    a = normalize_phase(h, t, q, z)
    b = normalize_phase(Hs, np.eye(n), Qs, Qs)
    assert rel_diff(a[0], b[0]) < 1e-12
    assert rel_diff(a[2], b[2]) < 1e-12


# ----------------------------------------------------------------------------- invariants


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("n,r,tdiag", [(256, 8, "abs"), (200, 16, "abs"), (160, 3, "graded"), (97, 32, "abs")])
def test_invariants_backward_error_orthogonality_zeros(cplx, n, r, tdiag):
    # north_star: ||A-QHZ*||/||A|| <= 10nu, same for B; ||Q*Q-I|| <= 10nu; exact zeros
    H, T = make_pencil(n, r, cplx, tdiag, seed=42 + n)
    h, t, q, z, _ = oracle.stage2(H, T, r)
    inv = invariants(H, T, h, t, q, z)
    assert inv["zeros_bad"] == 0
    for k in ("eA", "eB", "oQ", "oZ"):
        assert inv[k] <= inv["bound"], (k, inv)
    # Q e1 = Z e1 = e1 exactly (every reflector acts on indices >= 2)
    assert np.array_equal(q[:, 0], np.eye(n)[:, 0]) and np.array_equal(z[0, :], np.eye(n)[0, :])


def test_singular_T_still_backward_stable():
    # reading c4 / [V5]: exact zero diagonal entries in T (saddle-point style) stay stable
    n, r = 80, 6
    H, T = make_pencil(n, r, seed=5)
    T[np.arange(0, n, 4), np.arange(0, n, 4)] = 0.0
    h, t, q, z, _ = oracle.stage2(H, T, r)
    inv = invariants(H, T, h, t, q, z)
    assert inv["zeros_bad"] == 0 and np.all(np.isfinite(h))
    for k in ("eA", "eB", "oQ", "oZ"):
        assert inv[k] <= inv["bound"], (k, inv)


def test_accumulate_false_bitwise_same_HT():
    # SPEC.md:416 idea / SURVEY §8(b): Q = Z = NULL skips accumulation, H, T bitwise equal
    H, T = make_pencil(120, 9, seed=3)
    h1, t1, _, _, _ = oracle.stage2(H, T, 9)
    h2, t2, q2, z2, _ = oracle.stage2(H, T, 9, accumulate=False)
    assert q2 is None and np.array_equal(h1, h2) and np.array_equal(t1, t2)


def test_nonidentity_QZ_inputs_right_multiplied():
    # reading c13: Q <- Q_in Q2, Z <- Z_in Z2
    n, r = 50, 4
    H, T = make_pencil(n, r, seed=8)
    rng = np.random.default_rng(0)
    Qin, _ = np.linalg.qr(rng.standard_normal((n, n)))
    Zin, _ = np.linalg.qr(rng.standard_normal((n, n)))
    _, _, q0, z0, _ = oracle.stage2(H, T, r)
    _, _, q1, z1, _ = oracle.stage2(H, T, r, Q=Qin, Z=Zin)
    assert rel_diff(q1, Qin @ q0) < 1e-13 and rel_diff(z1, Zin @ z0) < 1e-13


def test_thread_count_bitwise_independent():
    # OpenMP splits only independent columns/rows -> bitwise identical
    H, T = make_pencil(300, 120, seed=4)
    old = oracle.set_threads(0)
    try:
        oracle.set_threads(1)
        a = oracle.stage2(H, T, 120)
        oracle.set_threads(8)
        b = oracle.stage2(H, T, 120)
    finally:
        oracle.set_threads(old)
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)


def test_flop_count_close_to_counted_8n3():
    # reading c7: Alg. 2's printed ranges perform ~8n^3 (+RQ), not the stated 10n^3
    n, r = 512, 16
    H, T = make_pencil(n, r, seed=1)
    fl = oracle.stage2(H, T, r)[4]
    assert 8.0 < fl / n**3 < 8.7  # 8.03n^3 + (2/3)r^2n^2 RQ + O(rn^2) at n=512


# ----------------------------------------------------------------------------- Fig. 5 structure traces


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _masks_after(ops):
    """Expected nonzero patterns for n = 10, r = 3 after the first `ops` reflector
    applications, hand-decoded from Fig. 5 (grid cell = one entry)
    and stored with their sub-figure citations in tests/golden/fig5_n10_r3_ops*.txt."""
    with open(os.path.join(GOLDEN, f"fig5_n10_r3_ops{ops}.txt")) as f:
        lines = [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]
    a = lines.index("A")
    b = lines.index("B")
    A = np.array([[c == "1" for c in row] for row in lines[a + 1:b]])
    B = np.array([[c == "1" for c in row] for row in lines[b + 1:]])
    return A, B


@pytest.mark.parametrize("ops", [0, 1, 2, 3, 4])
def test_fig5_structure_traces(ops):
    n, r = 10, 3
    H, T = make_pencil(n, r, seed=21)
    h, t, _, _, _ = oracle.stage2(H, T, r, max_ops=ops)
    mA, mB = _masks_after(ops)
    assert np.array_equal(h != 0, mA), (ops, (h != 0).astype(int), mA.astype(int))
    assert np.array_equal(t != 0, mB), (ops, (t != 0).astype(int), mB.astype(int))


# ----------------------------------------------------------------------------- worked example


def _read_sections(path):
    out, cur = {}, None
    with open(path) as f:
        for ln in f:
            ln = ln.strip()
            if not ln or ln.startswith("#"):
                continue
            if ln.isalpha():
                cur = ln
                out[cur] = []
            else:
                out[cur].append([float(x) for x in ln.split()])
    return {k: np.array(v) for k, v in out.items()}


def test_worked_example_n4_r2():
    # SURVEY.md App. A.5 (session-derived with the c1-c4 conventions and
    # cross-checked there against Moler-Stewart; the paper prints no values).
    g = _read_sections(os.path.join(GOLDEN, "worked_example_n4_r2.txt"))
    h, t, q, z, _ = oracle.stage2(g["A"], g["B"], 2)
    assert np.max(np.abs(h - g["H"])) < 1e-13 and np.max(np.abs(t - g["T"])) < 1e-13
    assert np.max(np.abs(q[1:, 1:] - g["Q"])) < 1e-13 and np.max(np.abs(z[1:, 1:] - g["Z"])) < 1e-13
    assert structure_violations(h, t) == 0
    # independent algorithm on the same input agrees after phase normalisation (reading c10)
    hg, tg, qg, zg = givens_ht(g["A"], g["B"])
    a = normalize_phase(h, t, q, z)
    b = normalize_phase(hg, tg, qg, zg)
    assert max(rel_diff(x, y) for x, y in zip(a, b)) < 1e-14


# ----------------------------------------------------------------------------- blocked == unblocked
@pytest.mark.parametrize("n,r,q,cplx", [(60, 4, 6, False), (97, 6, 5, False), (80, 5, 8, False), (64, 8, 1, False),
                                         (72, 3, 12, True), (90, 4, 9, True)])
def test_blocked_schedule_matches_oracle(n, r, q, cplx):
    # SURVEY §8(c) pin 6: the corrected blocked Alg. 3/4 (App. A.2-A.3; tests/blocked_ref.py, a second
    # CPU ordering sharing no code with oracle/) reorders Alg. 2's reflector applications only as
    # PAPER.md:720-732 allows, so it must give the oracle's result up to rounding -- this pins the
    # index corrections (reading c8) the GPU kernels implement, independently of the GPU
    from blocked_ref import blocked_stage2
    H, T = make_pencil(n, r, cplx, seed=500 + n)
    ho, to, qo, zo, _ = oracle.stage2(H, T, r)
    hb, tb, qb, zb = blocked_stage2(H, T, r, q)
    a = normalize_phase(hb, tb, qb, zb)
    b = normalize_phase(ho, to, qo, zo)
    assert max(rel_diff(x, y) for x, y in zip(a, b)) < 1e-12
    inv = invariants(H, T, hb, tb, qb, zb)
    assert inv["zeros_bad"] == 0 and max(inv["eA"], inv["eB"], inv["oQ"], inv["oZ"]) <= inv["bound"]
