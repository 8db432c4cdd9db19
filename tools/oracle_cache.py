"""Cached oracle results at the BASELINE configs' own sizes (test infrastructure).

    python tools/oracle_cache.py CFG [--threads T] [--ncols 24] [--out oracle_cache]

Runs ONLY `oracle/` (Alg. 2) and `synth/` on config CFG at its full n and
writes `oracle_cache/cfg{CFG}.npz` (git-ignored; it travels to the GPU box with the snapshot):

* `cols`, `rows`: seeded sample of column / row indices (0-based; first and last included);
* for X in H, T, Q, Z (reading-c10 phase-normalised, synth/check.py): `X_cols` (n x len(cols)),
  `X_rows` (len(rows) x n) -- the GPU parity test normalises its own result the same way and
  compares these entries (tests/test_gpu_fullsize.py);
* the oracle's own invariants (eA, eB, oQ, oZ, bound, zero-structure violations) and its time;
* the noise floor of SURVEY §8(c) pin 7 (forward sensitivity, [V3]): the oracle rerun on the
  input with every nonzero entry perturbed by a relative u-sized amount (seeded), normalised and
  sampled the same way -- `floor_X` = relative difference of the samples of the two oracle runs.
  Two correct (backward-stable) reductions of the same pencil differ by about this much.

Nothing here reads or calls the CUDA path.  Takes minutes (config 2) to hours (config 4) on
the host cores; the configs' seeds are fixed in synth/pencil.py.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth.check import U, normalise_samples, phase_factors, sample_rel_diff, structure_violations  # noqa: E402
from synth.pencil import CONFIGS, config_pencil  # noqa: E402


def sample_indices(n: int, k: int, seed: int):
    rng = np.random.default_rng(seed)
    idx = set(rng.choice(n, size=min(k, n), replace=False).tolist()) | {0, n - 1}
    return np.array(sorted(idx), dtype=np.int64)


def normalised_samples(H, T, Q, Z, cols, rows):
    dq, dz = phase_factors(H, T)
    raw = {nm: (X[:, cols], X[rows, :]) for nm, X in (("H", H), ("T", T), ("Q", Q), ("Z", Z))}
    return normalise_samples(raw, dq, dz, cols, rows)


def invariants_blas(A, B, H, T, Q, Z):
    n = A.shape[0]
    Zh = Z.conj().T
    eA = np.linalg.norm(A - Q @ (H @ Zh)) / np.linalg.norm(A)
    eB = np.linalg.norm(B - Q @ (T @ Zh)) / np.linalg.norm(B)
    I = np.eye(n, dtype=A.dtype)
    oQ = np.linalg.norm(Q.conj().T @ Q - I)
    oZ = np.linalg.norm(Zh @ Z - I)
    return dict(eA=float(eA), eB=float(eB), oQ=float(oQ), oZ=float(oZ), bound=10.0 * n * U,
                zeros_bad=structure_violations(H, T))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", type=int)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ncols", type=int, default=24)
    ap.add_argument("--n", type=int, default=0, help="reduced n (testing this script)")
    ap.add_argument("--out", default=os.path.join(ROOT, "oracle_cache"))
    ap.add_argument("--no-floor", action="store_true")
    args = ap.parse_args()
    c = CONFIGS[args.cfg]
    H, T = config_pencil(args.cfg, args.n or None)
    n, r = H.shape[0], c["r"]
    threads = oracle.set_threads(args.threads)
    cols = sample_indices(n, args.ncols, 7000 + args.cfg)
    rows = sample_indices(n, args.ncols, 8000 + args.cfg)
    t0 = time.perf_counter()
    ho, to, qo, zo, fl = oracle.stage2(H, T, r)
    t_or = time.perf_counter() - t0
    print(f"cfg {args.cfg} n={n} r={r}: oracle {t_or:.1f} s on {threads} threads", flush=True)
    res = normalised_samples(ho, to, qo, zo, cols, rows)
    inv = invariants_blas(H, T, ho, to, qo, zo)
    print("oracle invariants", inv, flush=True)
    del ho, to, qo, zo
    meta = dict(cfg=args.cfg, n=n, r=r, seed=c["seed"], complex=c["complex"], tdiag=c["tdiag"],
                oracle_s=t_or, oracle_threads=threads, oracle_flops_counted=fl, invariants=inv,
                ncols=len(cols), nrows=len(rows))
    if not args.no_floor:
        # u-sized relative perturbation of every structural nonzero (seeded), same structure
        rng = np.random.default_rng(9000 + args.cfg)
        Hp = H * (1.0 + U * rng.uniform(-1.0, 1.0, H.shape))
        Tp = T * (1.0 + U * rng.uniform(-1.0, 1.0, T.shape))
        t0 = time.perf_counter()
        hp, tp, qp, zp, _ = oracle.stage2(np.asfortranarray(Hp), np.asfortranarray(Tp), r)
        meta["floor_oracle_s"] = time.perf_counter() - t0
        del Hp, Tp
        fp = normalised_samples(hp, tp, qp, zp, cols, rows)
        del hp, tp, qp, zp
        meta["floor"] = {nm: sample_rel_diff(fp, res, nm) for nm in "HTQZ"}
        print("noise floor (oracle vs oracle on u-perturbed input, sampled rel. diff)", meta["floor"], flush=True)
    os.makedirs(args.out, exist_ok=True)
    fn = os.path.join(args.out, f"cfg{args.cfg}" + (f"_n{n}" if args.n else "") + ".npz")
    np.savez(fn, cols=cols, rows=rows, meta=json.dumps(meta), **res)
    print("wrote", fn, json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
