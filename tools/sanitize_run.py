"""Small reductions for compute-sanitizer (racecheck / synccheck / memcheck): direct launches
(HT_NO_GRAPH), shapes covering every chase instantiation (r = 8, 16, 32 real; 16 complex; 64; 128),
checked against the north_star invariants so a run that "passes" the tool also computed the
right thing.
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

os.environ.setdefault("HT_NO_GRAPH", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_07964_b200 as ht  # noqa: E402
from synth.check import invariants  # noqa: E402
from synth.pencil import make_pencil  # noqa: E402

CASES = [(256, 8, False), (200, 16, False), (160, 32, False), (128, 16, True), (260, 64, False), (300, 128, False)]
bad = 0
for n, r, cplx in CASES:
    H, T = make_pencil(n, r, cplx, seed=4242 + n)
    d = lambda A: torch.from_numpy(np.asfortranarray(A)).cuda()
    Hd, Td, Qd, Zd = d(H), d(T), d(np.eye(n, dtype=H.dtype)), d(np.eye(n, dtype=H.dtype))
    ht.ht_stage2(Hd, Td, r, Qd, Zd)
    torch.cuda.synchronize()
    inv = invariants(H, T, *(X.cpu().numpy() for X in (Hd, Td, Qd, Zd)))
    ok = inv["zeros_bad"] == 0 and max(inv["eA"], inv["eB"], inv["oQ"], inv["oZ"]) <= inv["bound"]
    bad += not ok
    print(f"n={n} r={r} complex={cplx}: eA={inv['eA']:.1e} oQ={inv['oQ']:.1e} oZ={inv['oZ']:.1e} {'ok' if ok else 'FAIL'}", flush=True)
sys.exit(1 if bad else 0)
