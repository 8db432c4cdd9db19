"""C-ABI boundary tests that need no GPU (-m "not gpu"): the library loads, exports every
function include/ht_stage2.h declares, and its host-only entry points and synchronous argument
checks behave as the header states.  Plus the multi-GPU row-slab decomposition,
checked single-process and across a world_size-2 gloo process group on CPU."""
import ctypes
import os
import re
import socket

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ht_stage2.h")


@pytest.fixture(scope="module")
def ht():
    import paper_2301_07964_b200 as ht
    from paper_2301_07964_b200 import build
    build.build()  # nvcc cross-compiles for sm_100a without a GPU
    ht._load()
    return ht


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ht_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("ht_stage2_d", "ht_stage2_z", "ht_stage2_d_ex", "ht_stage2_z_ex", "ht_nccl_unique_id",
                     "ht_comm_create", "ht_strerror", "ht_flops_std"):
        assert required in names


def test_library_exports_every_declared_symbol(ht):
    lib = ctypes.CDLL(ht.library_path())
    missing = [nm for nm in declared_functions() if not hasattr(lib, nm)]
    assert not missing, missing
    assert set(declared_functions()) == set(ht.EXPORTED_SYMBOLS)


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("wp", [32, 64, 96, 128, 160])
def test_chain_fragment_loads_are_bank_conflict_free(ht, cplx, wp):
    """DESIGN.md section 10 "Chain shared-memory strides": an m8n8k4 DMMA fragment load has lane & 3
    along the stride and lane >> 2 along the contiguous direction.  Shared memory has 32 four-byte
    banks; a warp's 8-byte loads are served per half-warp and its 16-byte loads per quarter-warp,
    so within each such phase every lane must fall on its own bank group.  Enumerated here for the
    strides the library reports (the old strides, stride = 8 mod 16 doubles, fail this check)."""
    ldx, ldb = ht.chain_smem_strides(cplx, wp)
    assert ldx >= 32 and ldb >= wp  # a column of X holds 32 tile rows; a block row holds wp columns
    words = 4 if cplx else 2        # 4-byte words per element
    phase = 8 if cplx else 16       # lanes served together
    for ld in (ldx, ldb):
        for first in range(0, 32, phase):
            banks = set()
            for lane in range(first, first + phase):
                elem = (lane & 3) * ld + (lane >> 2)
                banks.add(((elem * words) % 32) // words)
            assert len(banks) == phase, (ld, first, sorted(banks))
    # the check itself rejects the strides of rounds 1-2 (X: 32 + 8, blocks: wp + 8)
    bad = {(((lane & 3) * 40 + (lane >> 2)) * 2 % 32) // 2 for lane in range(16)}
    assert len(bad) < 16
    with pytest.raises(ht.HTError):
        ht.chain_smem_strides(cplx, 7)


def test_host_only_entry_points(ht):
    assert ht.flops_std(1000) == 10.0 * 1000 ** 3  # PAPER.md:712 "10n^3"
    assert ht.flops_std(1000, True) == 40.0 * 1000 ** 3
    assert ht.strerror(0) == "success"
    assert "structure" in ht.strerror(1)
    assert ht.strerror(-3).startswith("invalid argument")
    q = ht.default_q(4096, 16)
    assert 1 <= q <= 4094
    ms, nl = ht.last_timing()
    assert set(ms) == {"chase", "ht_updates", "qz_updates", "total"} and nl >= 0


def test_argument_errors_are_synchronous(ht):
    lib = ht._load()
    d = ctypes.c_void_p(0x1000)  # never dereferenced: argument checks come first
    nul = ctypes.c_void_p(0)
    f = lib.ht_stage2_d
    assert f(-1, 3, d, 10, d, 10, nul, 10, nul, 10, nul, nul) == -1
    assert f(10, -1, d, 10, d, 10, nul, 10, nul, 10, nul, nul) == -2
    assert f(10, 3, nul, 10, d, 10, nul, 10, nul, 10, nul, nul) == -3
    assert f(10, 3, d, 5, d, 10, nul, 10, nul, 10, nul, nul) == -4
    assert f(10, 3, d, 10, nul, 10, nul, 10, nul, 10, nul, nul) == -5
    assert f(10, 3, d, 10, d, 9, nul, 10, nul, 10, nul, nul) == -6
    assert f(10, 3, d, 10, d, 10, d, 3, nul, 10, nul, nul) == -8
    assert f(10, 3, d, 10, d, 10, nul, 10, d, 3, nul, nul) == -10
    assert f(0, 3, nul, 1, nul, 1, nul, 1, nul, 1, nul, nul) == 0  # empty problem: nothing to do


@pytest.mark.parametrize("n,G", [(1, 1), (31, 2), (100, 3), (4096, 8), (16384, 8), (32768, 5), (33, 8)])
def test_slab_range_partitions_rows(ht, n, G):
    rows = [ht.slab_range(n, G, i) for i in range(G)]
    pos = 0
    for a, ln in rows:
        assert a == pos and ln >= 0
        if a < n and ln > 0:
            assert a % 32 == 0  # whole chain tiles
        pos = a + ln
    assert pos == n
    lens = [ln for _, ln in rows]
    assert max(lens) - min(lens) <= 32 * 1 + (n % 32 != 0) * 32


def test_slab_range_rejects_bad_arguments(ht):
    with pytest.raises(ht.HTError):
        ht.slab_range(10, 0, 0)
    with pytest.raises(ht.HTError):
        ht.slab_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, n, out):
    import torch
    import torch.distributed as dist
    import paper_2301_07964_b200 as ht
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    a, ln = ht.slab_range(n, world, rank)
    t = torch.tensor([a, ln], dtype=torch.int64)
    allt = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allt, t)
    # the multi-GPU path's unique-id exchange (comm_from_torch) uses broadcast_object_list
    obj = [b"x" * 128 if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    out.put((rank, [tuple(x.tolist()) for x in allt], obj[0]))
    dist.destroy_process_group()


def test_slabs_across_gloo_ranks(ht):
    import torch.multiprocessing as mp
    world, n = 2, 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    views = {r: (slabs, obj) for r, slabs, obj in res}
    assert views[0][0] == views[1][0]  # every rank sees the same decomposition
    slabs = views[0][0]
    assert slabs[0][0] == 0 and slabs[0][0] + slabs[0][1] == slabs[1][0] and slabs[1][0] + slabs[1][1] == n
    assert views[1][1] == b"x" * 128


# ---------------------------------------------------------------------------- far H/T tile plan (§8(e))
def _far_plan_worker(rank, world, port, n, q, out):
    import torch
    import torch.distributed as dist
    import paper_2301_07964_b200 as ht
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    tiles = (n + 31) // 32
    plan = [ht.far_tile_plan(n, q, world, t) for t in range(tiles)]
    root = 0
    # this rank's message schedule, in issue order: hand-offs group by group, then the final gather
    sends, recvs = [], []
    for g in range((n - 2 + q - 1) // q):
        for t, (o, gt, c0) in enumerate(plan):
            if gt == g and o != root:
                msg = ("handoff", g, t, c0)
                if rank == root:
                    sends.append((o,) + msg)
                if rank == o:
                    recvs.append((root,) + msg)
    for t, (o, gt, c0) in enumerate(plan):
        if o not in (-1, root):
            msg = ("gather", gt, t, c0)
            if rank == o:
                sends.append((root,) + msg)
            if rank == root:
                recvs.append((o,) + msg)
    allp = [None] * world
    dist.all_gather_object(allp, {"plan": plan, "sends": sends, "recvs": recvs})
    out.put((rank, allp))
    dist.destroy_process_group()


@pytest.mark.parametrize("n,q,world", [(1000, 32, 2), (777, 13, 3)])
def test_far_tile_plan_across_gloo_ranks(n, q, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_far_plan_worker, args=(r, world, port, n, q, qu)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(qu.get(timeout=180) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    views = res[0]
    assert all(res[r] == views for r in range(world))  # every rank saw the same exchange
    plans = [v["plan"] for v in views]
    assert all(pl == plans[0] for pl in plans)  # one deterministic plan on every rank
    plan = plans[0]
    tiles = (n + 31) // 32
    ngroups = (n - 2 + q - 1) // q
    far = [t for t, (o, g, c) in enumerate(plan) if o >= 0]
    # a tile turns far at the first group whose j1 = 1 + g q is at or below its last row + 1, once
    for t, (o, g, c) in enumerate(plan):
        if o < 0:
            assert 1 + (ngroups - 1) * q < 32 * (t + 1)
            continue
        assert o == t % world and c == 1 + g * q and 32 * (t + 1) <= c and (g == 0 or 1 + (g - 1) * q < 32 * (t + 1))
    assert far == list(range(len(far)))  # far tiles are a prefix, turning far in order
    owned = [sum(1 for t in far if plan[t][0] == r) for r in range(world)]
    assert max(owned) - min(owned) <= 1  # balanced
    # every send has exactly one matching receive, in the same order between each pair of ranks
    for a in range(world):
        for b in range(world):
            s_ab = [m[1:] for m in views[a]["sends"] if m[0] == b]
            r_ba = [m[1:] for m in views[b]["recvs"] if m[0] == a]
            assert s_ab == r_ba, (a, b)
    # each far tile not owned by the root is handed off once and gathered back once
    hand = sorted(m[3] for m in views[0]["sends"] if m[1] == "handoff")
    gath = sorted(m[3] for m in views[0]["recvs"] if m[1] == "gather")
    assert hand == gath == [t for t in far if plan[t][0] != 0]
    assert tiles > len(far) > 0
