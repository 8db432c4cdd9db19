"""B200-native stage two of the two-stage Hessenberg-triangular reduction (arxiv 2301.07964).

Thin ctypes binding over the C ABI in ``include/ht_stage2.h`` (``libht_stage2.so``,
hand-written sm_100a CUDA).  Argument marshalling only: every step of the reduction
runs in the library's kernels.  There is NO CPU fallback: if the library is missing
or no CUDA device is present, calls raise.

PyTorch is used for device memory and streams only.  Matrices are column-major:
an n x n tensor ``X`` with ``X.stride(0) == 1`` and ``X.stride(1) = ld >= n``
(e.g. ``torch.empty(n, n, dtype=torch.float64, device='cuda').t()`` or a tensor
created from a Fortran-ordered numpy array).
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["ht_stage2", "ht_stage2_host", "HTError", "flops_std", "default_q", "strerror",
           "last_timing", "probe_dmma_tflops", "probe_dfma_tflops", "library_path", "Opts",
           "release_cache"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libht_stage2.so")
_lib = None


class HTError(RuntimeError):
    def __init__(self, code: int):
        self.code = code
        super().__init__(f"ht_stage2 returned {code}: {strerror(code) if _lib else ''}")


class Opts(ctypes.Structure):
    _fields_ = [("q", ctypes.c_int64), ("reserved0", ctypes.c_int32), ("root", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("reserved", ctypes.c_int32 * 5)]


def library_path() -> str:
    return _SO


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} is missing: run `python -m paper_2301_07964_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(_SO)
    p, i64 = ctypes.c_void_p, ctypes.c_int64
    for sfx in ("d", "z"):
        f = getattr(lib, f"ht_stage2_{sfx}_ex")
        f.argtypes = [i64, i64, p, i64, p, i64, p, i64, p, i64, p, p, ctypes.POINTER(Opts)]
        f.restype = ctypes.c_int
        g = getattr(lib, f"ht_stage2_{sfx}")
        g.argtypes = [i64, i64, p, i64, p, i64, p, i64, p, i64, p, p]
        g.restype = ctypes.c_int
    lib.ht_strerror.argtypes = [ctypes.c_int]
    lib.ht_strerror.restype = ctypes.c_char_p
    lib.ht_flops_std.argtypes = [i64, ctypes.c_int]
    lib.ht_flops_std.restype = ctypes.c_double
    lib.ht_default_q.argtypes = [i64, i64, ctypes.c_int]
    lib.ht_default_q.restype = i64
    lib.ht_last_timing.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
    lib.ht_last_timing.restype = ctypes.c_int
    for nm in ("ht_probe_dmma_tflops", "ht_probe_dfma_tflops"):
        getattr(lib, nm).argtypes = [ctypes.c_int]
        getattr(lib, nm).restype = ctypes.c_double
    lib.ht_nccl_unique_id.argtypes = [p]
    lib.ht_nccl_unique_id.restype = ctypes.c_int
    lib.ht_comm_create.argtypes = [p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(p)]
    lib.ht_comm_create.restype = ctypes.c_int
    lib.ht_comm_destroy.argtypes = [p]
    lib.ht_comm_destroy.restype = ctypes.c_int
    lib.ht_slab_range.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.ht_slab_range.restype = ctypes.c_int
    lib.ht_last_lag_check.argtypes = [ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.ht_last_lag_check.restype = ctypes.c_int
    lib.ht_far_tile_plan.argtypes = [i64, i64, ctypes.c_int, i64, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(i64),
                                     ctypes.POINTER(i64)]
    lib.ht_far_tile_plan.restype = ctypes.c_int
    lib.ht_chain_smem_strides.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    lib.ht_chain_smem_strides.restype = ctypes.c_int
    lib.ht_release_cache.argtypes = []
    lib.ht_release_cache.restype = ctypes.c_int
    _lib = lib
    return lib


EXPORTED_SYMBOLS = ("ht_stage2_d", "ht_stage2_z", "ht_stage2_d_ex", "ht_stage2_z_ex",
                    "ht_nccl_unique_id", "ht_comm_create", "ht_comm_destroy", "ht_slab_range", "ht_strerror",
                    "ht_flops_std", "ht_default_q", "ht_last_timing", "ht_probe_dmma_tflops",
                    "ht_probe_dfma_tflops", "ht_release_cache", "ht_last_lag_check", "ht_far_tile_plan",
                    "ht_chain_smem_strides")


def slab_range(n: int, nranks: int, rank: int):
    """(row0, nrows) of the Q/Z row slab rank `rank` of `nranks` updates (multi-GPU, C ABI)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    rc = _load().ht_slab_range(int(n), int(nranks), int(rank), ctypes.byref(a), ctypes.byref(b))
    if rc != 0:
        raise HTError(rc)
    return a.value, b.value


def chain_smem_strides(is_complex: bool, wp: int):
    """(ldx, ldb): shared-memory strides of the chain kernels in elements (C ABI ht_chain_smem_strides)."""
    a, b = ctypes.c_int(), ctypes.c_int()
    rc = _load().ht_chain_smem_strides(int(bool(is_complex)), int(wp), ctypes.byref(a), ctypes.byref(b))
    if rc != 0:
        raise HTError(rc)
    return a.value, b.value


def far_tile_plan(n: int, q: int, nranks: int, tile: int):
    """(owner, group, col0) of H/T row tile `tile` in the multi-GPU plan (C ABI ht_far_tile_plan);
    (-1, -1, -1) for tiles that never turn far."""
    o, g, c = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
    rc = _load().ht_far_tile_plan(int(n), int(q), int(nranks), int(tile), ctypes.byref(o), ctypes.byref(g), ctypes.byref(c))
    if rc != 0:
        raise HTError(rc)
    return o.value, g.value, c.value


def nccl_comm(rank: int, nranks: int, unique_id: bytes):
    """Create an NCCL communicator (ht_comm_create) from a 128-byte unique id; returns an opaque int."""
    out = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    rc = _load().ht_comm_create(buf, int(rank), int(nranks), ctypes.byref(out))
    if rc != 0:
        raise HTError(rc)
    return out.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = _load().ht_nccl_unique_id(buf)
    if rc != 0:
        raise HTError(rc)
    return buf.raw


def comm_from_torch(group=None):
    """NCCL communicator over a torch.distributed process group (rank 0's unique id is broadcast
    with broadcast_object_list: torch's own NCCL communicator is not exposed by a stable API)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return nccl_comm(rank, world, obj[0])


def release_cache() -> None:
    """Free this thread's cached CUDA graphs, their workspace and the input-check state (C ABI
    ``ht_release_cache``)."""
    rc = _load().ht_release_cache()
    if rc != 0:
        raise HTError(rc)


def comm_destroy(comm) -> None:
    if comm:
        _load().ht_comm_destroy(ctypes.c_void_p(comm))


def strerror(code: int) -> str:
    return _load().ht_strerror(int(code)).decode()


def flops_std(n: int, is_complex: bool = False) -> float:
    """The paper's standard stage-two count: 10 n^3 (real), 40 n^3 (complex)."""
    return _load().ht_flops_std(int(n), int(bool(is_complex)))


def default_q(n: int, r: int, is_complex: bool = False) -> int:
    return int(_load().ht_default_q(int(n), int(r), int(bool(is_complex))))


def last_timing():
    """(ms dict, launches) of the last call on this thread (timings need profile=True)."""
    ms = (ctypes.c_double * 4)()
    nl = ctypes.c_int64()
    _load().ht_last_timing(ms, ctypes.byref(nl))
    return dict(chase=ms[0], ht_updates=ms[1], qz_updates=ms[2], total=ms[3]), nl.value


def last_lag_check():
    """(orderings checked, violations) of the last call with HT_LAG_CHECK=1 (C ABI ht_last_lag_check)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _load().ht_last_lag_check(ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def probe_dmma_tflops(iters: int = 20000) -> float:
    return _load().ht_probe_dmma_tflops(int(iters))


def probe_dfma_tflops(iters: int = 20000) -> float:
    return _load().ht_probe_dfma_tflops(int(iters))


def _check_mat(X, n, name, dtype):
    import torch
    if X is None:
        return None, 1
    if not isinstance(X, torch.Tensor) or not X.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if X.dtype != dtype:
        raise TypeError(f"{name} dtype {X.dtype} != {dtype}")
    if tuple(X.shape) != (n, n) or (n > 0 and X.stride(0) != 1):
        raise ValueError(f"{name} must be n x n column-major (stride(0) == 1)")
    return ctypes.c_void_p(X.data_ptr()), max(1, X.stride(1) if n > 1 else n)


def ht_stage2(H, T, r: int, Q=None, Z=None, stream=None, q: int = 0,
              validate: bool = True, profile: bool = False, comm=None, root: int = 0,
              emulate_slabs: int = 0):
    """In-place stage two on device tensors (C ABI ``ht_stage2_{d,z}_ex``).

    H, T: n x n column-major CUDA tensors (float64 or complex128) holding an r-HT pencil.
    Q, Z: optional n x n tensors, right-multiplied by the accumulated transforms.
    Raises HTError on a nonzero return code.  Stream-ordered on ``stream``
    (default: torch's current stream).
    """
    import torch
    lib = _load()
    n = H.shape[0]
    cplx = H.dtype == torch.complex128
    dt = torch.complex128 if cplx else torch.float64
    ph, ldh = _check_mat(H, n, "H", dt)
    pt, ldt = _check_mat(T, n, "T", dt)
    pq, ldq = _check_mat(Q, n, "Q", dt)
    pz, ldz = _check_mat(Z, n, "Z", dt)
    for X, nm in ((T, "T"), (Q, "Q"), (Z, "Z")):
        if X is not None and X.device != H.device:
            raise ValueError(f"{nm} is on {X.device}, H on {H.device}")
    s = stream if stream is not None else torch.cuda.current_stream(H.device)
    opts = Opts(q=int(q), root=int(root),
                flags=(0 if validate else 1) | (2 if profile else 0) | (4 if emulate_slabs > 1 else 0))
    opts.reserved[0] = int(emulate_slabs)
    fn = lib.ht_stage2_z_ex if cplx else lib.ht_stage2_d_ex
    with torch.cuda.device(H.device):  # the C ABI works on the calling thread's current device
        rc = fn(n, int(r), ph, ldh, pt, ldt, pq, ldq, pz, ldz, ctypes.c_void_p(s.cuda_stream),
                ctypes.c_void_p(comm) if comm else None, ctypes.byref(opts))
    if rc != 0:
        raise HTError(rc)
    return H, T, Q, Z


def ht_stage2_host(H, T, r: int, accumulate: bool = True, q: int = 0, device=None, stream=None):
    """End-to-end convenience path: host (numpy, any order) in, host (numpy, Fortran) out.

    Copies the pencil to the device (via pinned staging), runs ``ht_stage2`` with
    Q = Z = I formed on the device, and copies H, T, Q, Z back.
    """
    import numpy as np
    import torch
    dev = torch.device(device or "cuda")
    cplx = np.iscomplexobj(H) or np.iscomplexobj(T)
    dt = torch.complex128 if cplx else torch.float64
    n = H.shape[0]

    def to_dev(A):
        h = torch.from_numpy(np.asfortranarray(A, dtype=np.complex128 if cplx else np.float64))
        return h.t().contiguous().pin_memory().to(dev, non_blocking=True).t()

    with torch.cuda.device(dev):
        Hd, Td = to_dev(H), to_dev(T)
        Qd = Zd = None
        if accumulate:
            Qd = torch.eye(n, dtype=dt, device=dev).t()
            Zd = torch.eye(n, dtype=dt, device=dev).t()
        cur = torch.cuda.current_stream(dev)
        s = stream if stream is not None else cur
        if s != cur:
            s.wait_stream(cur)  # the uploads and eye() ran on the current stream
        ht_stage2(Hd, Td, r, Qd, Zd, stream=s, q=q)
        s.synchronize()  # the call may return while the reduction still runs on s

    def to_host(X):
        return None if X is None else X.t().cpu().numpy().T

    return to_host(Hd), to_host(Td), to_host(Qd), to_host(Zd)
