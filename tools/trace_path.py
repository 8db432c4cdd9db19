"""Critical path of one chase launch from its global-timer stamps (dev tool).

    HT_LAG_CHECK=1 HT_TRACE_DUMP=/tmp/tr.bin [HT_TRACE_J1=j1] python tools/run_config.py 4 --n 8192 --calls 1 --no-check
    python tools/trace_path.py /tmp/tr.bin

Walks back from the last event along the binding dependency of the wavefront protocol (the
orderings `check_lag` in ht_stage2.cu checks: a sweep step waits for its own previous step, the
previous sweep's step k+2 and that sweep's helpers' item k+1; a helper item waits for its sweep's
step, its own previous item and the previous sweep's helpers) and splits the path into sweep-step
work, helper-item work and hand-off gaps (start minus the binding predecessor's end).
"""
import sys

import numpy as np


def load(path):
    raw = open(path, "rb").read()
    n, r, qp, j1, K, helpers = np.frombuffer(raw[:24], dtype=np.int32)
    hoff = np.frombuffer(raw[24:24 + 4 * (qp + 1)], dtype=np.int32)
    tr = np.frombuffer(raw[24 + 4 * (qp + 1):], dtype=np.uint64).astype(np.int64)
    return int(n), int(r), int(qp), int(j1), int(K), hoff, tr


def main(path):
    n, r, qp, j1, K, hoff, tr = load(path)

    def sb(t, k): return tr[(t * K + k) * 2]
    def se(t, k): return tr[(t * K + k) * 2 + 1]
    def hb(t, h, k): return tr[(qp * K + (hoff[t] + h) * K + k) * 2]
    def he(t, h, k): return tr[(qp * K + (hoff[t] + h) * K + k) * 2 + 1]
    def H(t): return int(hoff[t + 1] - hoff[t])
    def kc(t): return min(K, 2 + (n - (j1 + t) - 1) // r)

    def preds(node):
        if node[0] == "s":
            _, t, k = node
            out = []
            if k > 0:
                out.append(("s", t, k - 1))
            if t > 0:
                kprev = min(K, 2 + (n - (j1 + t)) // r)
                need, hneed = min(k + 3, kprev), min(k + 2, kprev)
                out.append(("s", t - 1, need - 1))
                out += [("h", t - 1, h, hneed - 1) for h in range(H(t - 1))]
            return out
        _, t, h, k = node
        out = [("s", t, k)]
        if k > 0:
            out.append(("h", t, h, k - 1))
        if t > 0:
            kprev = min(K, 2 + (n - (j1 + t)) // r)
            out += [("h", t - 1, hh, min(k + 2, kprev) - 1) for hh in range(H(t - 1))]
        return out

    def beg(x): return sb(x[1], x[2]) if x[0] == "s" else hb(x[1], x[2], x[3])
    def end(x): return se(x[1], x[2]) if x[0] == "s" else he(x[1], x[2], x[3])

    # last event of the launch
    nodes = [("s", t, kc(t) - 1) for t in range(qp)]
    nodes += [("h", t, h, kc(t) - 1) for t in range(qp) for h in range(H(t))]
    nodes = [x for x in nodes if end(x) > 0]
    t0 = min(beg(x) for x in nodes if beg(x) > 0)
    cur = max(nodes, key=end)
    total = end(cur) - t0
    work_s = work_h = gap = 0
    ns = nh = 0
    hops = {"own": 0, "prev_step": 0, "prev_helper": 0, "helper_own": 0, "helper_sweep": 0}
    while True:
        w = end(cur) - beg(cur)
        if cur[0] == "s":
            work_s += w
            ns += 1
        else:
            work_h += w
            nh += 1
        ps = [p for p in preds(cur) if p[-1] >= 0 and end(p) > 0]
        if not ps:
            gap += beg(cur) - t0
            break
        p = max(ps, key=end)
        gap += max(0, beg(cur) - end(p))
        if cur[0] == "s":
            hops["own" if p[0] == "s" and p[1] == cur[1] else ("prev_step" if p[0] == "s" else "prev_helper")] += 1
        else:
            hops["helper_sweep" if p[0] == "s" else ("helper_own" if p[1] == cur[1] else "prev_helper")] += 1
        cur = p
    steps = sum(kc(t) for t in range(qp))
    print(f"group j1={j1} n={n} r={r} qp={qp} K={K}: launch span {total / 1e3:.1f} us (global timer ns), "
          f"critical-path model K+3(qp-1) = {kc(0) + 3 * (qp - 1)} steps")
    print(f"  on the path: {ns} sweep steps ({work_s / max(ns, 1):.0f} ns each), {nh} helper items "
          f"({work_h / max(nh, 1):.0f} ns each), hand-off gaps {gap / 1e3:.1f} us total")
    print(f"  binding predecessors: {hops}")
    dur = np.array([se(t, k) - sb(t, k) for t in range(qp) for k in range(kc(t)) if se(t, k) > 0])
    print(f"  all sweep steps: {steps}, mean {dur.mean():.0f} ns, median {np.median(dur):.0f} ns")
    hd = np.array([he(t, h, k) - hb(t, h, k) for t in range(qp) for h in range(H(t)) for k in range(kc(t))
                   if he(t, h, k) > 0])
    if hd.size:
        print(f"  all helper items: {hd.size}, mean {hd.mean():.0f} ns, median {np.median(hd):.0f} ns")


if __name__ == "__main__":
    main(sys.argv[1])
