#!/usr/bin/env python
"""Benchmark: stage-two HT reduction throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step = one full ``ht_stage2`` call (all §8(a) rows: chase, accumulation, staircase,
off-window and Q/Z updates) on the config's synthetic r-HT pencil, inputs restored from a
pristine device copy inside the step (inputs 4 x n^2 x 8 B > 126 MB L2, so no L2 reuse across
steps).  value = 10n^3 / t_step (the paper's standard count) in GFLOP/s.
N > 1 (torchrun, one rank per GPU) solves ONE problem on N GPUs (strong scaling):
the root chases and updates H, T; every rank updates its row slab of Q and Z from reflector
records broadcast by NCCL per group; the slabs are gathered to the root inside the timed call.

--impl reference times the CPU oracle (Alg. 2, plain C, all host cores) on a bounded sample of
the same workload (the leading n_s x n_s sub-pencil of the config's pencil, same r and
generator) -- the only place besides cpu_baseline where bench.py executes oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth.pencil import CONFIGS, make_pencil  # noqa: E402

METRIC = "stage-2 GFLOP/s and fraction of FP64 tensor roofline vs n, r at 1/2/4/8 B200"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _chase_latency(n, r, q, chase_ms, clk):
    """K1 is a dependency chain: per group of qp sweeps the last sweep finishes after
    K + 3(qp-1) sweep steps (lag 3).  Steps on the critical path of the call
    and the measured cycles per such step (chase time incl. K2/K2m x SM clock / steps)."""
    steps = 0
    for j1 in range(1, n - 1, q):
        qp = min(q, n - 1 - j1)
        steps += 1 + (n - j1 - 2) // r + 3 * (qp - 1)
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    return {"critical_path_steps": steps, "cycles_per_step": chase_ms * 1e-3 * mhz * 1e6 / max(steps, 1),
            "sm_mhz": mhz}


def _dgemm_tflops(dev, n=8192, reps=3):
    """cuBLAS DGEMM (torch.matmul, fp64, n^3) throughput on this GPU: the library reference for
    the FP64 tensor ceiling next to the in-house DMMA probe; not on the path."""
    import torch
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    return 2.0 * n ** 3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12


def _ncu_traffic(kernel, n, r, q):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed
    `ncu --set full` capture summary (profiles/ncu_traffic.json), when it was taken on this
    workload; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d[kernel]
        if (e["n"], e["r"], e["q"]) == (n, r, q):
            return e["bytes_per_launch"]
    except Exception:
        pass
    return None


def _invariants_dev(A, B, H, T, Q, Z):
    """north_star's bounds on the GPU in fp64 (torch matmuls; a check, not the product path):
    ||A - QHZ*||_F/||A||_F, same for B, ||Q*Q - I||_F, ||Z*Z - I||_F, each also / (10 n u), and
    the count of entries that must be exactly zero but are not."""
    import torch
    n = A.shape[0]
    Zh = Z.conj().t()
    eA = float(torch.linalg.norm(A - Q @ (H @ Zh)) / torch.linalg.norm(A))
    eB = float(torch.linalg.norm(B - Q @ (T @ Zh)) / torch.linalg.norm(B))
    I = torch.eye(n, dtype=A.dtype, device=A.device)
    oQ = float(torch.linalg.norm(Q.conj().t() @ Q - I))
    oZ = float(torch.linalg.norm(Zh @ Z - I))
    del I, Zh
    zeros = int(torch.count_nonzero(torch.tril(H, -2))) + int(torch.count_nonzero(torch.tril(T, -1)))
    bound = 10.0 * n * 2.0 ** -53
    torch.cuda.empty_cache()
    return {"eA": eA, "eB": eB, "oQ": oQ, "oZ": oZ, "bound": bound,
            "over_bound": {k: v / bound for k, v in (("eA", eA), ("eB", eB), ("oQ", oQ), ("oZ", oZ))},
            "zeros_bad": zeros, "pass": max(eA, eB, oQ, oZ) <= bound and zeros == 0}


class ClockSampler:
    """SM clocks and throttling over the timed region (B200_PROFILING.md), through NVML
    in-process and WITHOUT queries inside the region (NVML / nvidia-smi queries during it were
    measured to stall the host side of the timed loop now and then, up to +0.9 s):
    - the power and thermal violation-time counters (cumulative, ns) just before and just after
      the region: any increase means the region was throttled (reported as sw_power_cap /
      sw_thermal_slowdown);
    - the SM clock and the current event-reason bits sampled just before and at the end of the
      region (the GPU is still at its load clock then).
    nvidia-smi is the fallback when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, interval: float = 0.0):
        self.index = index
        self.interval = interval
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reason bits)
        self.stop_ev = threading.Event()

    def _violations(self):
        nv = self.nvml
        out = {}
        for nm, pol in (("power", nv.NVML_PERF_POLICY_POWER), ("thermal", nv.NVML_PERF_POLICY_THERMAL)):
            try:
                out[nm] = int(nv.nvmlDeviceGetViolationStatus(self.h, pol).violationTime)
            except Exception:
                pass
        return out

    def _sample(self):
        nv = self.nvml
        try:
            self.samples.append((float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)), self.mx,
                                 int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
        except Exception:
            pass

    def start(self):
        if os.environ.get("HT_NO_SMI"):
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            try:
                self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            except Exception:
                self.mx = 0.0
            self.v0 = self._violations()
            self._sample()
            if self.interval > 0:  # sampled DURING the region too (long steps hide host stalls)
                self.th = threading.Thread(target=self._loop, daemon=True)
                self.th.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "250"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _loop(self):
        while not self.stop_ev.wait(self.interval):
            self._sample()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            nv = self.nvml
            self.stop_ev.set()
            if getattr(self, "th", None) is not None:
                self.th.join(timeout=5)
            self._sample()
            v1 = self._violations()
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            reasons = {nm for _, _, rs in self.samples for nm, b in bits.items() if rs & b}
            if v1.get("power", 0) > self.v0.get("power", 0):
                reasons.add("sw_power_cap")
            if v1.get("thermal", 0) > self.v0.get("thermal", 0):
                reasons.add("sw_thermal_slowdown")
            sm = [x[0] for x in self.samples]
            try:
                nv.nvmlShutdown()
            except Exception:
                pass
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.mx or None,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml (+ violation counters)"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


def cpu_sample(cfg, n_s):
    """Oracle (plain C Alg. 2, all host cores) on the leading n_s x n_s sub-pencil of config cfg.
    Returns (GFLOP/s at 10 n_s^3, threads used, seconds, CPU seconds / wall seconds)."""
    import oracle
    c = CONFIGS[cfg]
    H, T = make_pencil(c["n"] if c["n"] <= 4096 else n_s, c["r"], c["complex"], c["tdiag"], c["seed"])
    H = np.asfortranarray(H[:n_s, :n_s])
    T = np.asfortranarray(T[:n_s, :n_s])
    cores = oracle.set_threads(len(os.sched_getaffinity(0)))
    c0 = time.process_time()
    t0 = time.perf_counter()
    oracle.stage2(H, T, c["r"])
    dt = time.perf_counter() - t0
    par = (time.process_time() - c0) / max(dt, 1e-9)  # effective parallelism actually used
    fl = (40.0 if c["complex"] else 10.0) * n_s ** 3
    return fl / dt / 1e9, cores, dt, par


def _full_oracle_record(cfg):
    """The oracle's own full-size run on this config, if tools/oracle_cache.py cached it
    (builder container; not the GPU box): seconds, threads, invariants, noise floor."""
    try:
        d = np.load(os.path.join(ROOT, "oracle_cache", f"cfg{cfg}.npz"))
        m = json.loads(str(d["meta"]))
        fl = (40.0 if m["complex"] else 10.0) * m["n"] ** 3
        return {"seconds": m["oracle_s"], "threads": m["oracle_threads"], "gflops": fl / m["oracle_s"] / 1e9,
                "host": "builder container (tools/oracle_cache.py), not the GPU box", "noise_floor": m.get("floor")}
    except Exception:
        return None


def _sample_n(c):
    """Leading sub-pencil size of the CPU samples (about 10-30 s of oracle work on 8-16 cores)."""
    return min(c["n"], 1536 if c["complex"] else 2048)


def run_reference(args, rank):
    if rank != 0:
        return
    c = CONFIGS[args.config]
    n_s = args.sample_n or _sample_n(c)
    for _ in range(args.warmup):
        cpu_sample(args.config, min(n_s, 512))
    vals, times, pars = [], [], []
    cores = 1
    for _ in range(args.steps):
        v, cores, dt, par = cpu_sample(args.config, n_s)
        vals.append(v)
        times.append(dt)
        pars.append(par)
    v = statistics.mean(vals)
    sample = (f"oracle (Alg. 2, plain C, OpenMP) full reduction of the leading {n_s}x{n_s} sub-pencil "
              f"of config{args.config} (r={c['r']}, same generator/seed); rate = 10n_s^3/t")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64" if not c["complex"] else "c128",
        "data": "synthetic", "config": _config_dict(args, c, q=None),
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "effective_parallelism": statistics.mean(pars),
                         "full_config_oracle": _full_oracle_record(args.config)},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def _config_dict(args, c, q):
    td = getattr(args, "tdiag", "") or c["tdiag"]
    tdt = {"graded": "graded 10^U(-3,0)", "abs": "1+|N(0,1)|",
           "singular25": "1+|N(0,1)| with 25% exact zeros (singular T, saddle-point-like)"}[td]
    d = {"workload": f"config{args.config}{'-' + td if td != c['tdiag'] else ''}: n={c['n']} r={c['r']} "
                     f"{'complex' if c['complex'] else 'real'} fp64, T diag {tdt}, Q,Z accumulated",
         "n": c["n"], "r": c["r"], "complex": c["complex"], "seed": c["seed"],
         "l2": "inputs (4 n^2 fp64) larger than the 126 MB L2; restored from a device copy each step",
         "parallelism": (f"root chase + H/T, Q/Z row slabs x{args.gpus} (NCCL)" if args.gpus > 1 else "1 GPU")}
    if q is not None:
        d["q"] = q
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--q", type=int, default=0)
    ap.add_argument("--sample-n", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--tdiag", default="", choices=["", "abs", "graded", "singular25"],
                    help="override the config's T diagonal (singular25: SURVEY 8(f) row 2, saddle-point-like)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world and args.impl == "ours":
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2301_07964_b200 as ht

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = ht.comm_from_torch()
    c = CONFIGS[args.config]
    n, r, cplx = c["n"], c["r"], c["complex"]
    q = args.q or ht.default_q(n, r, cplx)
    tdt = torch.complex128 if cplx else torch.float64

    tdiag = args.tdiag or c["tdiag"]
    H_np, T_np = make_pencil(n, r, cplx, tdiag, c["seed"])

    def col_major_dev(A):
        return torch.from_numpy(A).to(dev)  # Fortran-ordered numpy -> stride (1, n)

    H0, T0 = col_major_dev(H_np), col_major_dev(T_np)
    I0 = torch.eye(n, dtype=tdt, device=dev).t()
    H, T = H0.clone(memory_format=torch.preserve_format), T0.clone(memory_format=torch.preserve_format)
    Qd, Zd = I0.clone(memory_format=torch.preserve_format), I0.clone(memory_format=torch.preserve_format)
    assert H.stride(0) == 1 and Qd.stride(0) == 1
    stream = torch.cuda.current_stream(dev)

    def step(profile=False):
        H.copy_(H0)
        T.copy_(T0)
        Qd.copy_(I0)
        Zd.copy_(I0)
        ht.ht_stage2(H, T, r, Qd, Zd, stream=stream, q=q, profile=profile, comm=comm)

    # warm-up: at least W steps and at least 3 s of work -- the first seconds of a fresh process
    # on a fresh box were measured up to 25 % slower (clock / power ramp)
    n_warm, t_warm = 0, time.time()
    while n_warm < max(3, args.warmup) or time.time() - t_warm < 3.0:
        step()
        torch.cuda.synchronize()
        n_warm += 1
    # one profiled call (per-kernel-class device times via events) outside the timed region
    step(profile=True)
    torch.cuda.synchronize()
    brk_ms, launches_per_call = ht.last_timing()

    def barrier():
        if world > 1:
            dist.barrier()

    # steps of a second or more: NVML samples every 0.5 s inside the region (a host stall there
    # is hidden by the queued work); shorter steps: only at both ends (see ClockSampler)
    clocks = ClockSampler(local, interval=0.5 if brk_ms["total"] > 1000.0 else 0.0)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    launches = launches_per_call * args.steps
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    fstd = ht.flops_std(n, cplx)
    value = fstd / (ms_step * 1e-3) / 1e9  # one problem on all ranks (strong scaling)
    brk = brk_ms

    # ---- roofline of the dominant kernel class (live CUDA-event durations) ----
    peaks = _peaks()
    dmma = ht.probe_dmma_tflops(20000)
    dgemm = _dgemm_tflops(dev)
    fcnt_upd = (8.03 if not cplx else 8.03 * 4) * n ** 3  # counted update flops (H,T 4.03 + Q,Z 4.00) n^3
    # The dominant kernel class is the one with the largest share of the step's critical path:
    # the chase (K1) and the H/T chains run back to back on the caller's stream; the Q/Z chains
    # overlap them on a side stream.
    rq = (2.0 / 3.0) * r * r * n * n * (4 if cplx else 1)
    band = 2.0 * r * (q + 2) * n * n * (4 if cplx else 1)
    dfma = ht.probe_dfma_tflops(20000)
    ach_k1 = (rq + band) / (brk["chase"] * 1e-3) / 1e12
    roof_k1 = {"kernel": "chase_kernel (K1)", "bound": "alu", "achieved": ach_k1, "peak": dfma, "unit": "TFLOP/s",
               "frac": ach_k1 / dfma, "traffic": _ncu_traffic("chase_kernel", n, r, q),
               "peak_source": "measured DFMA probe (ht_probe_dfma_tflops) on this GPU; MEASURED_PEAKS.json has no FP64 figure",
               "algorithmic": "RQ (2/3)r^2n^2 + generate band 2r(q+2)n^2 flops per call (a latency-bound chain)",
               "share_of_step": brk["chase"] / ms_step,
               "latency_model": _chase_latency(n, r, q, brk["chase"], clk)}
    ht_cnt = (4.03 if not cplx else 4.03 * 4) * n ** 3  # counted H,T update flops (left + right) [V2]
    ach_ht = ht_cnt / (brk["ht_updates"] * 1e-3) / 1e12
    roof_ht = {"kernel": "chain_kernel, H/T right + left (K3/K4)", "bound": "tensor", "achieved": ach_ht, "peak": dmma,
               "unit": "TFLOP/s", "frac": ach_ht / dmma, "traffic": _ncu_traffic("chain_kernel", n, r, q),
               "peak_source": "measured DMMA (mma.sync f64) probe on this GPU; MEASURED_PEAKS.json has no FP64 figure",
               "algorithmic": "counted H,T update flops 4.03n^3 per call (x4 complex); dense U/V execute (q+r-1)^2/(2qr) x",
               "share_of_step": brk["ht_updates"] / ms_step}
    qz_cnt = (4.0 if not cplx else 16.0) * n ** 3
    roof_qz = {"kernel": "chain_kernel, Q/Z (side stream, overlapped)", "bound": "tensor",
               "achieved": qz_cnt / (brk["qz_updates"] * 1e-3) / 1e12 if brk["qz_updates"] > 0 else None,
               "peak": dmma, "unit": "TFLOP/s"}
    if roof_qz["achieved"] is not None:
        roof_qz["frac"] = roof_qz["achieved"] / dmma
    roof = roof_k1 if brk["chase"] >= brk["ht_updates"] else roof_ht

    out = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": n_warm, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if not cplx else "c128", "data": "synthetic",
        "config": _config_dict(args, c, q),
        "roofline": roof,
        "roofline_other": [x for x in (roof_k1, roof_ht, roof_qz) if x is not roof],
        "fraction_fp64_roofline": value / (world * dmma * 1e3),
        "gflops_counted": fcnt_upd / (ms_step * 1e-3) / 1e9,
        "breakdown_ms": brk, "dmma_peak_tflops": dmma, "cublas_dgemm_tflops": dgemm,
        "clocks": clk, "gpu_launches": launches,
        "measured_peaks": {k: peaks.get(k) for k in ("hbm_gbs", "bf16_tflops")},
    }

    # ---- result check of the last timed step (north_star invariants; test-side fp64 torch matmuls) ----
    if not args.no_check:
        out["invariants"] = _invariants_dev(H0, T0, H, T, Qd, Zd)

    # ---- end to end: host pinned buffers -> device, C-ABI call, results -> host ----
    if not args.no_e2e:
        hp = [torch.from_numpy(A.T.copy()).pin_memory() for A in (H_np, T_np)]  # row-major of A^T
        ip = torch.eye(n, dtype=tdt).pin_memory()
        outs = [torch.empty((n, n), dtype=tdt).pin_memory() for _ in range(4)]

        def e2e_step():
            H.t().copy_(hp[0], non_blocking=True)
            T.t().copy_(hp[1], non_blocking=True)
            Qd.t().copy_(ip, non_blocking=True)
            Zd.t().copy_(ip, non_blocking=True)
            ht.ht_stage2(H, T, r, Qd, Zd, stream=stream, q=q, comm=comm)
            for o, X in zip(outs, (H, T, Qd, Zd)):
                o.copy_(X.t(), non_blocking=True)

        for _ in range(2):  # untimed: first transfers from / to the freshly pinned buffers
            e2e_step()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        esz = 16 if cplx else 8
        out["e2e"] = {"value": fstd / (e_ms / args.steps * 1e-3) / 1e9, "unit": "GFLOP/s",
                      "h2d_bytes_per_step": 4 * n * n * esz, "d2h_bytes_per_step": 4 * n * n * esz}

    if rank == 0 and not args.no_cpu:
        n_s = args.sample_n or _sample_n(c)
        v, cores, dt, par = cpu_sample(args.config, n_s)
        out["cpu_baseline"] = {
            "value": v, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "effective_parallelism": par,
            "sample": f"oracle (Alg. 2, plain C, OpenMP) full reduction of the leading {n_s}x{n_s} sub-pencil of "
                      f"config{args.config} (r={r}); {dt:.1f} s; rate = 10n_s^3/t",
            "full_config_oracle": _full_oracle_record(args.config)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        ht.comm_destroy(comm)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
