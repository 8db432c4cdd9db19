"""CPU check of the RQ-update scheme the CUDA chase uses for real 32 < r <= 128:
tests/rqu_ref.py runs Alg. 2 with the opposite reflector taken from an RQ
factorisation handed from sweep to sweep and re-triangularised by Givens rotations (instead of a
fresh Householder RQ, reading c4).  It must reproduce the oracle (c9: the reduction is unique up to
diagonal phases for a nonsingular T), keep B1 = R1 W to rounding over many chained sweeps, and
keep the invariants for a singular T (where several results are correct)."""
import numpy as np
import pytest

import oracle
from synth.check import invariants, normalize_phase, rel_diff
from synth.pencil import make_pencil
from rqu_ref import house, rot, rq_full, rq_update, stage2_rqu


def test_rq_update_is_an_rq_of_the_rank_one_modified_block():
    rng = np.random.default_rng(3)
    m = 9
    R0 = np.triu(rng.standard_normal((m, m))) + 2 * np.eye(m)
    Q0, _ = np.linalg.qr(rng.standard_normal((m, m)))
    v, tau, _ = house(rng.standard_normal(m))
    Rt, Qt = rq_update(R0, Q0, v, tau)
    M = (np.eye(m) - tau * np.outer(v, v)) @ R0 @ Q0  # Q^T B0
    assert np.allclose(np.tril(Rt, -1), 0.0, atol=1e-15)
    assert rel_diff(Rt @ Qt, M) < 1e-14
    assert np.linalg.norm(Qt @ Qt.T - np.eye(m)) < 1e-14
    # the same first row (direction) as a fresh Householder RQ of M, up to sign
    Rf, Qf = rq_full(M)
    assert min(np.linalg.norm(Qf[0] - Qt[0]), np.linalg.norm(Qf[0] + Qt[0])) < 1e-13


def test_givens_rotation_zeroes_the_first_entry():
    c, s, rho = rot(3.0, 4.0)
    assert abs(3.0 * c - 4.0 * s) < 1e-15 and abs(3.0 * s + 4.0 * c - 5.0) < 1e-15 and rho == 5.0


@pytest.mark.parametrize("n,r,q", [(40, 4, None), (61, 8, 4), (64, 16, 8), (50, 5, 7)])
def test_rqu_scheme_matches_oracle(n, r, q):
    H, T = make_pencil(n, r, False, seed=11)
    ho, to, qo, zo, _ = oracle.stage2(H, T, r)
    h, t, qq, zz, worst = stage2_rqu(H, T, r, q, check=True)
    assert worst < 1e-14  # B1 = R1 W, chained over every sweep (no drift)
    a = normalize_phase(h, t, qq, zz)
    b = normalize_phase(ho, to, qo, zo)
    assert max(rel_diff(x, y) for x, y in zip(a, b)) < 1e-11
    inv = invariants(H, T, h, t, qq, zz)
    assert inv["zeros_bad"] == 0 and max(inv[k] for k in ("eA", "eB", "oQ", "oZ")) <= inv["bound"]


def test_rqu_scheme_singular_T_invariants():
    H, T = make_pencil(48, 6, False, tdiag="singular25", seed=5)
    h, t, qq, zz, worst = stage2_rqu(H, T, 6, 4, check=True)
    assert worst < 1e-14
    inv = invariants(H, T, h, t, qq, zz)
    assert inv["zeros_bad"] == 0 and max(inv[k] for k in ("eA", "eB", "oQ", "oZ")) <= inv["bound"]
