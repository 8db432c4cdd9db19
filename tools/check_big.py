# dev: run one config through the C ABI (wall-timed, several calls) and check invariants on the host
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_07964_b200 as ht
from synth.pencil import config_pencil, CONFIGS
from synth.check import invariants
cfg = int(sys.argv[1]); q = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n_override = int(sys.argv[3]) if len(sys.argv) > 3 else None
c = CONFIGS[cfg]
H, T = config_pencil(cfg, n_override)
n = H.shape[0]
dt = torch.complex128 if c["complex"] else torch.float64
H0 = torch.from_numpy(H).cuda(); T0 = torch.from_numpy(T).cuda()
I0 = torch.eye(n, dtype=dt, device="cuda").t()
for it in range(3):
    Hd, Td, Qd, Zd = H0.clone(), T0.clone(), I0.clone(), I0.clone()
    torch.cuda.synchronize(); t0 = time.time()
    ht.ht_stage2(Hd, Td, c["r"], Qd, Zd, q=q, profile=(it == 2))
    torch.cuda.synchronize(); print("call", it, "wall %.1f ms" % (1e3 * (time.time() - t0)), ht.last_timing()[0] if it == 2 else "", flush=True)
h, t, qq, zz = (X.cpu().numpy() for X in (Hd, Td, Qd, Zd))
print("finite:", np.isfinite(h).all(), np.isfinite(t).all())
inv = invariants(H, T, h, t, qq, zz)
print(inv, "pass" if max(inv[k] for k in ("eA", "eB", "oQ", "oZ")) <= inv["bound"] and inv["zeros_bad"] == 0 else "FAIL")
