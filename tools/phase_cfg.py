# dev helper: per-phase device timing (profile=True: chase incl. K2/K2m, H/T chains, Q/Z) of a
# BASELINE config with Q and Z accumulated
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import paper_2301_07964_b200 as ht
from synth.pencil import CONFIGS, config_pencil
cfg = int(sys.argv[1])
r = CONFIGS[cfg]["r"]
Hn, Tn = config_pencil(cfg)
n = Hn.shape[0]
A = torch.from_numpy(np.asfortranarray(Hn)).cuda(); B = torch.from_numpy(np.asfortranarray(Tn)).cuda()
for it in range(2):
    H, T = A.clone(), B.clone()
    Q = torch.eye(n, dtype=A.dtype, device="cuda").t(); Z = torch.eye(n, dtype=A.dtype, device="cuda").t()
    torch.cuda.synchronize()
    ht.ht_stage2(H, T, r, Q, Z, profile=True)
    torch.cuda.synchronize()
    print("config", cfg, "iter", it, ht.last_timing(), flush=True)
