"""GPU parity of K1's RQ-update paths (rqu.cuh; real 32 < r <= 128).

* modes: HT_RQU=0 (Householder RQ per step), 1 (the sweep runs the RQ update, r <= 64),
  2 (default: the sweep solves for the direction, a helper runs the RQ update), and mode 2 with a
  share of the hand-overs run by the sweep itself (HT_RQU_SELF=num/den, m <= 64);
* the fallbacks of a singular R22 (exact zeros on T's diagonal reach the blocks): the sweep's own
  Givens chain at m <= 64, the helper's early answer (Freq / Fdirok) at m = 128 -- checked on
  invariants (several results are correct for a singular T, reading c9);
* the helper layouts (uniform / greedy by far-strip load) and the hand-over across groups
  (q small against n: many groups).
Each against the oracle (Alg. 2) like the default path."""
import os

import numpy as np
import pytest

from synth.pencil import make_pencil
from test_gpu_parity import check_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture
def env(request):
    saved = {k: os.environ.get(k) for k in request.param}
    os.environ.update(request.param)
    yield request.param
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


MODES = [{"HT_RQU": "0"}, {"HT_RQU": "1"}, {"HT_RQU": "2"}, {"HT_HELPER_BAL": "0"},
         {"HT_HELPER_BAL": "1", "HT_HELPER_F": "2"}, {"HT_NO_HELPERS": "1"}, {"HT_NO_GRAPH": "1"},
         {"HT_RQU_SELF": "1/2"}, {"HT_RQU_SELF": "2/3"}, {"HT_RQU_SELF": "1/1"}]


@pytest.mark.parametrize("env", MODES, indirect=True, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
@pytest.mark.parametrize("n,r,q", [(260, 40, 9), (400, 64, 32), (333, 64, 5), (520, 100, 24), (600, 128, 32),
                                    (300, 128, 7)])
def test_rqu_mode_parity(env, n, r, q):
    H, T = make_pencil(n, r, False, seed=131)
    check_parity(H, T, r, q=q)


@pytest.mark.parametrize("env", [{}, {"HT_RQU": "1"}, {"HT_RQU_SELF": "1/2"}], indirect=True, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()) or "default")
@pytest.mark.parametrize("n,r,q,every", [(400, 64, 32, 4), (300, 48, 16, 2), (500, 128, 32, 4), (380, 128, 9, 3)])
def test_rqu_singular_T_fallbacks(env, n, r, q, every):
    # exact zeros on T's diagonal: R22 of the hand-over is singular in many steps, so the solve
    # fails and the fallbacks run (sweep Givens at m <= 64, helper's early direction at m = 128)
    H, T = make_pencil(n, r, False, seed=37)
    d = np.arange(0, n, every)
    T[d, d] = 0.0
    check_parity(H, T, r, q=q, fwd=False)


def test_rqu_singular25_generator_invariants():
    H, T = make_pencil(640, 128, False, tdiag="singular25", seed=1004)
    check_parity(H, T, 128, fwd=False)
    H, T = make_pencil(512, 64, False, tdiag="singular25", seed=1004)
    check_parity(H, T, 64, fwd=False)
