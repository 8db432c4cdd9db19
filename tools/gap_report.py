# dev helper: GPU-vs-oracle forward gaps (after reading-c10 phase normalisation) and invariants
# on the BASELINE generators at reduced n (the test_baseline_config_shapes_reduced_n cases)
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2301_07964_b200 as ht
from synth.check import invariants, normalize_phase, rel_diff
from synth.pencil import CONFIGS, config_pencil

for cfg, n in [(1, 256), (2, 1024), (3, 384), (4, 768), (5, 640)]:
    H, T = config_pencil(cfg, n)
    r = CONFIGS[cfg]["r"]
    d = lambda A: torch.from_numpy(np.asfortranarray(A)).cuda()
    Hd, Td, Qd, Zd = d(H), d(T), d(np.eye(n, dtype=H.dtype)), d(np.eye(n, dtype=H.dtype))
    ht.ht_stage2(Hd, Td, r, Qd, Zd)
    torch.cuda.synchronize()
    h, t, q, z = (X.cpu().numpy() for X in (Hd, Td, Qd, Zd))
    inv = invariants(H, T, h, t, q, z)
    ho, to, qo, zo, _ = oracle.stage2(H, T, r)
    invo = invariants(H, T, ho, to, qo, zo)
    gaps = [rel_diff(x, y) for x, y in zip(normalize_phase(h, t, q, z), normalize_phase(ho, to, qo, zo))]
    print(f"config {cfg} n={n} r={r}: gap H,T,Q,Z = " + ", ".join(f"{g:.1e}" for g in gaps) +
          f" | GPU eA={inv['eA']:.1e} eB={inv['eB']:.1e} oQ={inv['oQ']:.1e} oZ={inv['oZ']:.1e}"
          f" | oracle eA={invo['eA']:.1e} oQ={invo['oQ']:.1e} | bound {inv['bound']:.1e}", flush=True)
