"""Dev: K1 profile of a config with / without the Q/Z side stream (contention check)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_07964_b200 as ht
from synth.pencil import CONFIGS, config_pencil
cfg, n, withqz = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
c = CONFIGS[cfg]
Hn, Tn = config_pencil(cfg, n)
A = torch.from_numpy(Hn).cuda(); B = torch.from_numpy(Tn).cuda()
I0 = torch.eye(n, dtype=A.dtype, device="cuda").t()
for it in range(2):
    H, T = A.clone(), B.clone()
    Q, Z = (I0.clone(), I0.clone()) if withqz else (None, None)
    torch.cuda.synchronize(); t0 = time.time()
    ht.ht_stage2(H, T, c["r"], Q, Z, profile=True)
    torch.cuda.synchronize()
    print("withqz", withqz, "wall", time.time() - t0, ht.last_timing()[0], flush=True)
