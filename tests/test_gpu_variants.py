"""GPU parity of the alternative schedules the library can be switched to (DESIGN.md §9,
environment knobs): no far-strip helper CTAs (the chase then owns its whole band), 1 and 3
helpers, no window merging (K2m off), direct launches instead of the cached graph, and Q/Z
chains started right after K2, and the K1 profiler's instrumented path.  Each must give the
oracle's result like the default path."""
import os

import pytest

from synth.pencil import make_pencil
from test_gpu_parity import check_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

VARIANTS = [
    {"HT_NO_HELPERS": "1"},
    {"HT_HELPERS": "1"},
    {"HT_HELPERS": "3"},
    {"HT_MERGE": "0"},
    {"HT_NO_GRAPH": "1"},
    {"HT_QZ_LATE": "0"},
    {"HT_QZ_GROUPS": "0"},
    {"HT_FAR_SIDE": "1"},  # one GPU: far H/T tiles' right updates on the side stream
    {"HT_WY": "0"},  # dense window blocks everywhere (default: compact WY blocks for real r >= 64, q in (16, 32])
    {"HT_WY": "1", "HT_MERGE": "0"},  # compact WY blocks wherever feasible (real, q in (16, 32], 4 warp columns)  # Q/Z chains one tile per CTA (default: two tile groups per CTA where they fit)
    {"HT_HELPER_LAG": "0"},  # helpers also take the rows just above b0(k) (default only for r >= 32)
    {"HT_HELPER_LAG": "1"},
    {"HT_K1PROF": "1", "HT_K1PROF_T": "1"},  # the instrumented path (profile counters, direct launches)
]


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


@pytest.mark.parametrize("env", VARIANTS, indirect=True, ids=lambda d: ",".join(f"{k}={v}" for k, v in d.items()))
@pytest.mark.parametrize("n,r,q,cplx", [(300, 16, 32, False), (257, 64, 9, False), (200, 8, 12, True),
                                         (330, 32, 16, False), (300, 128, 9, False), (350, 64, 32, False),
                                         (420, 96, 24, False), (400, 128, 32, False), (300, 40, 17, False)])
def test_variant_parity(env, n, r, q, cplx):
    H, T = make_pencil(n, r, cplx, seed=97)
    check_parity(H, T, r, q=q)
