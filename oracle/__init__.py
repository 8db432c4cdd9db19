"""CPU oracle for stage two of the two-stage HT reduction -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2301_07964_b200``) never imports it and shares no code with it.

It wraps ``liboracle_stage2.so`` (plain C, ``stage2_oracle.c``): the paper's
unblocked Alg. 2, one reflector at a time, fp64 real and
complex.  ``build()`` compiles it with gcc (building the checker is not using it).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_stage2.so")
_SRC = [os.path.join(_HERE, "stage2_oracle.c"), os.path.join(_HERE, "stage2_oracle_impl.h")]
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library in-tree (gcc, OpenMP)."""
    stale = not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in _SRC)
    if force or stale:
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _SO,
               os.path.join(_HERE, "stage2_oracle.c"), "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        p, i64, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        for sfx in ("d", "z"):
            f = getattr(lib, f"oracle_stage2_{sfx}")
            f.argtypes = [i64, i64, p, i64, p, i64, p, i64, p, i64, i64, dp]
            f.restype = ctypes.c_int
            g = getattr(lib, f"oracle_larfg_{sfx}")
            g.argtypes = [i64, p, p, p, dp]
            g.restype = None
            h = getattr(lib, f"oracle_rq_first_row_{sfx}")
            h.argtypes = [i64, p, p, p]
            h.restype = None
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_set_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def set_threads(n: int = 0) -> int:
    """Set the OpenMP thread count (0 = leave as is); returns the count in use."""
    return _load().oracle_set_threads(int(n))


def _sfx(a):
    return "z" if np.iscomplexobj(a) else "d"


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def larfg(x):
    """Householder generation (reading c1): returns (v, tau, beta) with H^* x = beta e1."""
    x = np.ascontiguousarray(x)
    dt = np.complex128 if np.iscomplexobj(x) else np.float64
    x = x.astype(dt)
    v = np.zeros_like(x)
    tau = np.zeros(1, dt)
    beta = ctypes.c_double(0.0)
    getattr(_load(), f"oracle_larfg_{_sfx(x)}")(len(x), _ptr(x), _ptr(v), _ptr(tau), ctypes.byref(beta))
    return v, tau[0], beta.value


def rq_first_row(C):
    """Householder RQ (reading c4) of a square block: returns (first row of Q~, R~)."""
    C = np.asfortranarray(C, dtype=np.complex128 if np.iscomplexobj(C) else np.float64).copy(order="F")
    m = C.shape[0]
    y = np.zeros(m, C.dtype)
    R = np.zeros((m, m), C.dtype, order="F")
    getattr(_load(), f"oracle_rq_first_row_{_sfx(C)}")(m, _ptr(C), _ptr(y), _ptr(R))
    return y, R


def stage2(H, T, r, Q=None, Z=None, accumulate=True, max_ops=-1):
    """Run the oracle (Alg. 2) on copies; returns (H, T, Q, Z, flops).

    Inputs are n x n arrays (any order); outputs are Fortran-ordered copies.
    Q, Z default to the identity when ``accumulate`` (reading c13: right-multiplied
    onto the inputs); with ``accumulate=False`` they are not formed (returned None).
    """
    cplx = np.iscomplexobj(H) or np.iscomplexobj(T) or (Q is not None and np.iscomplexobj(Q)) \
        or (Z is not None and np.iscomplexobj(Z))
    dt = np.complex128 if cplx else np.float64
    n = H.shape[0]
    A = np.array(H, dtype=dt, order="F", copy=True)
    B = np.array(T, dtype=dt, order="F", copy=True)
    if accumulate:
        Qo = np.array(Q if Q is not None else np.eye(n), dtype=dt, order="F", copy=True)
        Zo = np.array(Z if Z is not None else np.eye(n), dtype=dt, order="F", copy=True)
    else:
        Qo = Zo = None
    fl = ctypes.c_double(0.0)
    ld = max(1, n)
    rc = getattr(_load(), f"oracle_stage2_{'z' if cplx else 'd'}")(
        n, int(r), _ptr(A), ld, _ptr(B), ld, _ptr(Qo), ld, _ptr(Zo), ld, int(max_ops), ctypes.byref(fl))
    if rc != 0:
        raise ValueError(f"oracle_stage2 returned {rc}")
    return A, B, Qo, Zo, fl.value
