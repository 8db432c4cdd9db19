# dev helper: one config-2-like run with chase phase profiling (HT_K1PROF=1)
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import paper_2301_07964_b200 as ht
from synth.pencil import make_pencil
n, r, q = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 0
cplx = len(sys.argv) > 4 and sys.argv[4] == "c"
H, T = make_pencil(n, r, cplx, seed=1)
Hd = torch.from_numpy(H).cuda(); Td = torch.from_numpy(T).cuda()
for it in range(2):
    h, t = Hd.clone(), Td.clone()
    torch.cuda.synchronize(); t0 = time.time()
    ht.ht_stage2(h.t().contiguous().t() if False else h, t, r, q=q, profile=True)
    torch.cuda.synchronize(); print("wall", time.time() - t0, ht.last_timing())
