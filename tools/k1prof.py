# dev helper: chase phase profile (run with HT_K1PROF=1) and per-class device times of a pencil
#   python tools/k1prof.py n r [q] [c] [--lib path/to/libht_stage2.so]
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import torch  # noqa: E402

import paper_2301_07964_b200 as ht  # noqa: E402
from synth.pencil import make_pencil  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--lib")]
for a in sys.argv[1:]:
    if a.startswith("--lib="):
        ht._SO = a.split("=", 1)[1]  # A/B against another build of the same library
n, r = int(args[0]), int(args[1])
q = int(args[2]) if len(args) > 2 else 0
cplx = len(args) > 3 and args[3] == "c"
H, T = make_pencil(n, r, cplx, seed=1)
Hd = torch.from_numpy(H).cuda()
Td = torch.from_numpy(T).cuda()
for it in range(2):
    h, t = Hd.clone(), Td.clone()
    torch.cuda.synchronize()
    t0 = time.time()
    ht.ht_stage2(h, t, r, q=q, profile=True)
    torch.cuda.synchronize()
    print("wall", time.time() - t0, ht.last_timing(), flush=True)
