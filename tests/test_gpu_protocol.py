"""The wavefront protocol and the saddle-point-like workload on the GPU.

* Lag checker (compute-sanitizer is closed on this GPU pool): with HT_LAG_CHECK=1 every
  sweep step and far-strip helper item of the chase is stamped with the global timer and the
  library checks on the host that no step started before the steps it must follow had ended --
  sweep j's step k after sweep j-1's step k+2 (lag 3, SURVEY App. A.4 [V7][V11]), helper items
  after their sweep's step and the previous sweep's helper item.  Zero violations, results exact.
* Singular T with a quarter of its diagonal exactly zero (n/4 infinite eigenvalues, the paper's
  saddle-point setting PAPER.md:1697-1712): several reductions are correct there
  (reading c9), so invariants only.
"""
import os

import numpy as np
import pytest

from synth.pencil import make_pencil
from test_gpu_parity import check_parity, run_gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,r,q,cplx", [(300, 16, 32, False), (260, 64, 9, False), (200, 8, 12, True),
                                         (330, 32, 16, False), (300, 128, 9, False)])
def test_lag_checker_no_violations(n, r, q, cplx):
    import paper_2301_07964_b200 as ht
    os.environ["HT_LAG_CHECK"] = "1"
    try:
        H, T = make_pencil(n, r, cplx, seed=77)
        check_parity(H, T, r, q=q)
        checked, bad = ht.last_lag_check()
    finally:
        os.environ.pop("HT_LAG_CHECK", None)
    assert checked > 100, checked
    assert bad == 0, (bad, checked)


@pytest.mark.parametrize("n,r", [(512, 16), (400, 64), (300, 128)])
def test_singular25_invariants(n, r):
    H, T = make_pencil(n, r, tdiag="singular25", seed=1004)
    assert np.count_nonzero(np.diag(T) == 0) == n // 4
    check_parity(H, T, r, fwd=False)
