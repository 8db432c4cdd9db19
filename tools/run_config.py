"""One-off measurement of a BASELINE config at full size through the C ABI (dev tool, not the
bench contract): K calls (the first untimed), per-kernel-class device times of a profiled call,
device-timed default-path calls, and the north_star invariants on the GPU.

    python tools/run_config.py CFG [--calls K] [--q Q] [--profile-only]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_07964_b200 as ht  # noqa: E402
from synth.pencil import CONFIGS, config_pencil  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--calls", type=int, default=2)
    ap.add_argument("--q", type=int, default=0)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--lib", default="", help="A/B: another build of libht_stage2.so")
    args = ap.parse_args()
    if args.lib:
        ht._SO = args.lib
    c = CONFIGS[args.cfg]
    Hn, Tn = config_pencil(args.cfg, args.n or None)
    n, r = Hn.shape[0], c["r"]
    dt = torch.complex128 if c["complex"] else torch.float64
    A = torch.from_numpy(Hn).cuda()
    B = torch.from_numpy(Tn).cuda()
    del Hn, Tn
    I0 = torch.eye(n, dtype=dt, device="cuda").t()
    H, T, Q, Z = A.clone(), B.clone(), I0.clone(), I0.clone()
    q = args.q or ht.default_q(n, r, c["complex"])
    out = {"cfg": args.cfg, "n": n, "r": r, "q": q}

    def reset():
        H.copy_(A)
        T.copy_(B)
        Q.copy_(I0)
        Z.copy_(I0)

    reset()
    t0 = time.time()
    ht.ht_stage2(H, T, r, Q, Z, q=q, profile=True)
    torch.cuda.synchronize()
    out["profiled_call_wall_s"] = time.time() - t0
    out["breakdown_ms"], out["launches"] = ht.last_timing()
    times = []
    for _ in range(args.calls):
        reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ht.ht_stage2(H, T, r, Q, Z, q=q)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    out["call_ms"] = times
    best = min(times[1:] if len(times) > 1 else times)
    out["gflops_std"] = ht.flops_std(n, c["complex"]) / (best * 1e-3) / 1e9
    if not args.no_check:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from bench import _invariants_dev  # noqa: E402
        out["invariants"] = _invariants_dev(A, B, H, T, Q, Z)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
