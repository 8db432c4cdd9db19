// chain.cuh -- K3/K4: the apply phase of one group (Alg. 4
// "Application phase of stage two", corrected per DESIGN.md §3 / c8) as fused
// descending-k GEMM chains on the FP64 tensor cores (mma.sync f64 -> DMMA.8x8x4).
//
// One CTA owns a tile of BM "tile rows" of one matrix and streams the group's windows
// k = kstart ... kend (descending):
//   non-transposed (right updates  M(rows, C_k) <- M(rows, C_k) X_k):  tile rows = matrix
//       rows, chain index = matrix columns; X_k = V_k (H, T, Z) or U_k (Q);
//   transposed (left updates  M(R_k, cols) <- U_k^* M(R_k, cols)): tile rows = matrix
//       columns, chain index = matrix rows; computed as M^T <- M^T conj(U_k).
// The tile's window columns live in a circular on-chip buffer of w+r columns: window k
// occupies [p_k, p_k+w_k), window k-1 starts r columns earlier, so the q-1 overlap columns
// stay in place between windows (each entry of M is read and written once per group), the
// r fresh columns of the next window are prefetched (cp.async) while the current window
// computes, and the w x w blocks stream through a 3-stage ring filled by bulk async copies
// (cp.async.bulk + mbarrier, SASS UBLKCP).
// Rows of H/T right updates split per window into the block region (rows <= i5), the
// staircase (rows i5s..i4(k,j), reflector by reflector, Alg. 4 lines 4-9) and untouched
// rows; left updates touch columns > i5 (H) / > i6 (T) only.
#pragma once
#include <type_traits>

#include "scalar.cuh"

#ifndef IDX
#define IDX(p, ld, i, j) (p)[((int64_t)(i) - 1) + ((int64_t)(j) - 1) * (int64_t)(ld)]
#endif

// Shared-memory strides of X (tile rows per column) and of the block rows.  An m8n8k4 fragment load
// has lane & 3 along k (the stride) and lane >> 2 along the tile row / block column (contiguous); a
// 64-bit load is served per half-warp (4 k x 4 rows), a 128-bit load per quarter-warp (4 k x 2
// rows), so the stride must be 4 or 12 mod 16 doubles (real) and 2 or 6 mod 8 elements (complex):
// stride 8 mod 16 put k and k + 2 on the same banks (two-way conflicts on every fragment load,
// four-way for complex).  HT_CHAIN_PAD=8 restores the old strides (A/B builds).
#ifndef HT_CHAIN_PAD
#define HT_CHAIN_PAD 0
#endif
template <typename S>
__host__ __device__ constexpr int chain_pad() { return HT_CHAIN_PAD ? HT_CHAIN_PAD : (sizeof(S) == 8 ? 4 : 2); }

template <typename S>
__host__ __device__ constexpr int chain_ldb(int WP) { return WP + chain_pad<S>(); }

enum ChainMode { CM_PLAIN = 0, CM_AB_RIGHT = 1, CM_A_LEFT = 2, CM_B_LEFT = 3 };

template <typename S>
struct ChainJob {
    S* M;
    int64_t ld;
    const S* Blk;  // K blocks, each WP rows x LDB (row-major, padded rows/cols zero)
    const S* MBlk; // merged blocks (P > 1): ceil(K/P) blocks of P consecutive windows, same layout
    int mode;
    int trans;
    int ntiles;
    int tile0;  // first tile of this job (row slab of a multi-GPU rank; 0 = whole matrix)
    int tstride;  // tiles tile0, tile0 + tstride, ... (far H/T tiles of a rank: the rank count; 0 = 1)
};

template <typename S>
struct ChainParams {
    int n, r, qp, j1, K;
    ChainJob<S> job[2];
    int njobs;
    const S* Zr;  // staircase reflectors: (qp*K) records of (r+1)
    int P;        // window merge factor (1 = off): steps cover P windows where the tile is fully inside
    int spread;   // > 0 (H/T, two jobs of equal tile count): block order longest chain first (see below)
    long long* prof;  // optional (HT_K1PROF): cycles by phase of one tile's steps (8 slots)
    int prof_tile;    // the profiled tile of job 0 (HT_CHAIN_PROF_TILE)
    int stair_first;  // right chains: staircase-band tiles dispatched first (HT_STAIR_FIRST=0: off)
    const unsigned long long* gate;  // input-check verdict (input_rejected)
    // WY blocks ("compact WY"): each window's block
    // is I - Y T Y^* (forward xLARFT over the window's q reflectors) stored as Y (WP x (QP + 8),
    // row-major) followed by T Y^* (QP x (WP + 8)); a step is X <- X - (X Y)(T Y^*): 2 w q MACs per
    // tile row instead of w^2 (real fp64, single windows; wy = 0: dense blocks)
    int wy;
    int QP;  // q rounded up to 16
    // CM_PLAIN tiles (Q, Z: every entry read and written once per group, next touched a group later)
    // load and store with an L2 evict-first policy, so that the side-stream Q/Z traffic does not push
    // the chase's band and the window blocks out of L2 (HT_QZ_STREAM=0: default policy)
    int stream_plain = 0;
    int tmap = 0;  // transposed tiles (left updates): 4 x 8 lane map of the tile loads / stores (HT_CHAIN_TMAP)
};

template <typename S>
__host__ __device__ constexpr int chain_wy_ldy(int QP) { return QP + chain_pad<S>(); }
template <typename S>
__host__ __device__ constexpr size_t chain_wy_stride(int WP, int QP) {  // scalars per window in WY layout
    return (size_t)WP * chain_wy_ldy<S>(QP) + (size_t)QP * chain_ldb<S>(WP);
}

// H/T chains are latency-bound by their longest tiles (right updates: the top row tiles walk
// every window; left updates: the rightmost column tiles).  With spread = G (the SM count) the
// first G blocks -- one per SM in the first dispatch round -- take the G longest tiles (H and T
// interleaved) and block G + x takes the x-th SHORTEST, so an SM's second tile finishes early and
// leaves the long chain alone on the SM.  Returns (job, tile) of block b.
inline __host__ __device__ int chain_spread(int nsm) { return nsm > 0 ? nsm : 148; }
// Right chains: the row tiles of the staircase band [sb0, sb1) (single-window steps with the
// staircase, measured the slowest) come first, then the others top-down (band0 = band1: plain
// top-down order).
__device__ __forceinline__ void chain_order(int b, int total, int spread, bool longest_low, int nt, int& job,
                                            int& tile, int band0 = 0, int band1 = 0) {
    const int rank = (spread > 0 && b >= spread) ? total - 1 - (b - spread) : b;
    job = rank & 1;
    int tr = rank >> 1;
    const int nb = band1 - band0;
    if (longest_low && nb > 0) tr = (tr < nb) ? band0 + tr : ((tr - nb < band0) ? tr - nb : tr);
    tile = longest_low ? tr : nt - 1 - tr;
}

constexpr int CH_BM = 32;      // tile rows per CTA (one warp row of 4 m8 tiles)
constexpr int CH_KC = 16;      // k rows per ring chunk
constexpr int CH_STAGES = 3;   // ring depth
template <typename S>
__host__ __device__ constexpr int chain_ldx() { return CH_BM + chain_pad<S>(); }  // smem column stride of X
#ifndef HT_STAIR_BZ
#define HT_STAIR_BZ 4
#endif
constexpr int CH_SBZ = HT_STAIR_BZ;  // staircase reflectors per compact-WY block

// warps along the window's columns: each warp owns WP/WN columns (a multiple of 8)
__host__ __device__ constexpr int chain_wn(int WP) { return (WP % 64 == 0) ? 8 : 4; }
// warps along the tile rows: 8 warps per CTA (the chains are latency-bound; a warp's DMMA
// sequence per step is what a step costs)
#ifndef HT_CHAIN_WM
#define HT_CHAIN_WM 2
#endif
__host__ __device__ constexpr int chain_wm(int WP) { return chain_wn(WP) == 8 ? 1 : HT_CHAIN_WM; }
__host__ __device__ constexpr int chain_nt(int WP) { return 32 * chain_wn(WP) * chain_wm(WP); }

// dynamic smem: [64 B mbarriers][circular X: (w+r) x chain_ldx][block ring][staircase refl.]
template <typename S, int WP>
__host__ __device__ constexpr size_t chain_smem_bytes(int r, int q, int P = 1, int QP = 0) {
    return 64 + (size_t)(P > 1 ? q + 2 * P * r - 1 : q + r - 1 + r) * chain_ldx<S>() * sizeof(S) +
           (size_t)CH_STAGES * CH_KC * chain_ldb<S>(WP) * sizeof(S) + (size_t)(q + 1) * (r + 1) * sizeof(S) +
           (size_t)2 * ((q + CH_SBZ - 1) / CH_SBZ) * CH_SBZ * CH_SBZ * sizeof(S) +  // staircase block factors
           (size_t)QP * chain_ldx<S>() * sizeof(S);  // WY: the tile's X Y (QP columns)
}

// ---- PTX helpers ---------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(s)), "l"(g));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g));
}
template <typename S>
__device__ __forceinline__ void cp_async_elem(S* s, const S* g) {
    if constexpr (sizeof(S) == 8) cp_async8(s, g);
    else cp_async16(s, g);
}
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
template <typename S>
__device__ __forceinline__ void cp_async_elem_hint(S* s, const S* g, unsigned long long pol) {
    if constexpr (sizeof(S) == 8)
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(smem_u32(s)), "l"(g), "l"(pol));
    else
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(s)), "l"(g), "l"(pol));
}
template <typename S>
__device__ __forceinline__ void st_hint(S* g, const S& v, unsigned long long pol) {
    if constexpr (sizeof(S) == 8) {
        asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(g), "d"(v), "l"(pol) : "memory");
    } else {
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(g), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(s)),
        "l"(g), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

template <typename S>
struct Acc;
template <>
struct Acc<double> {
    double v[2];
};
template <>
struct Acc<zc> {
    double re[2], im[2];
};

// One k-step of 4 on an 8x8 tile: acc += a (8x4) * b (4x8); complex = 4 real DMMAs.
__device__ __forceinline__ void mma_step(Acc<double>& c, double a, double b) { dmma(c.v[0], c.v[1], a, b); }
__device__ __forceinline__ void mma_step(Acc<zc>& c, zc a, zc b) {
    dmma(c.re[0], c.re[1], a.x, b.x);
    dmma(c.re[0], c.re[1], -a.y, b.y);
    dmma(c.im[0], c.im[1], a.x, b.y);
    dmma(c.im[0], c.im[1], a.y, b.x);
}
__device__ __forceinline__ double acc_get(const Acc<double>& c, int h) { return c.v[h]; }
__device__ __forceinline__ zc acc_get(const Acc<zc>& c, int h) { return zc(c.re[h], c.im[h]); }
__device__ __forceinline__ void acc_zero(Acc<double>& c) { c.v[0] = c.v[1] = 0.0; }
__device__ __forceinline__ void acc_zero(Acc<zc>& c) { c.re[0] = c.re[1] = c.im[0] = c.im[1] = 0.0; }

template <typename S>
__device__ __forceinline__ S maybe_conj(S x, bool c) {
    if constexpr (sizeof(S) == 8) return x;
    else return c ? conjv(x) : x;
}

// ---------------------------------------------------------------------------------------
// One tile's descending-k chain.  Returns true if it initialised (and so must invalidate) the
// ring's mbarriers.
template <typename S, int WP>
__device__ __forceinline__ bool chain_tile(const ChainParams<S>& P, int bid, unsigned char* smraw, int grp, int gbar) {
    constexpr int LDB = chain_ldb<S>(WP);
    constexpr int CH_LDX = chain_ldx<S>();
    constexpr int CH_NT = chain_nt(WP);
    constexpr int NW = CH_NT / 32;
    constexpr int WN = chain_wn(WP);
    constexpr int WM = chain_wm(WP);
    constexpr int MT = CH_BM / 8 / WM;  // 8-row tiles per warp
    constexpr int NTL = WP / (8 * WN);  // 8-col tiles per warp
    static_assert(WP % (8 * WN) == 0, "window padding");
    const int n = P.n, r = P.r, qp = P.qp, j1 = P.j1, K = P.K;
    const int w = qp + r - 1;
    const int PM = P.P;
    const int CIRC = PM > 1 ? qp + 2 * PM * r - 1 : w + r;  // circular buffer columns

    // ---- which job / tile ----
    int jb_ = 0;
    if (P.spread > 0 && P.njobs == 2 && P.job[0].ntiles == P.job[1].ntiles) {
        const int m0 = P.job[0].mode;
        int band0 = 0, band1 = 0;
        if (m0 == CM_AB_RIGHT && P.stair_first) {  // tiles holding rows j1+1 .. j1+(qp-1) r
            // (tile indices relative to the jobs' first tile; both jobs start at the same tile)
            band0 = max(0, min(P.job[0].ntiles, P.j1 / CH_BM - P.job[0].tile0));
            band1 = max(0, min(P.job[0].ntiles, (P.j1 + (P.qp - 1) * P.r) / CH_BM + 1 - P.job[0].tile0));
        }
        chain_order(bid, 2 * P.job[0].ntiles, P.spread, m0 == CM_AB_RIGHT, P.job[0].ntiles, jb_, bid, band0, band1);
    } else if (P.njobs > 1 && bid >= P.job[0].ntiles) {
        bid -= P.job[0].ntiles;
        jb_ = 1;
    }
    const ChainJob<S> J = (jb_ == 0) ? P.job[0] : P.job[1];  // (no dynamic param indexing: no local memory)
    const int mode = J.mode;
    const bool trans = J.trans != 0;
    const int R0 = (J.tile0 + bid * (J.tstride > 0 ? J.tstride : 1)) * CH_BM + 1;  // first tile row (1-based)
    if (R0 > n) return false;
    const int nr = min(CH_BM, n - R0 + 1);
    const int R1 = R0 + nr - 1;

    uint64_t* bars = reinterpret_cast<uint64_t*>(smraw);
    S* X = reinterpret_cast<S*>(smraw + 64);
    S* ring = X + (size_t)CIRC * CH_LDX;
    S* zsm = ring + (size_t)CH_STAGES * CH_KC * LDB;
    // WY: the tile's A = X Y (QP columns x CH_LDX), after the staircase records and factors
    const bool WYm = P.wy != 0;
    const int QPw = P.QP, LDY = chain_wy_ldy<S>(P.QP);
    S* Abuf = zsm + (size_t)(qp + 1) * (r + 1) + (size_t)2 * ((qp + CH_SBZ - 1) / CH_SBZ) * CH_SBZ * CH_SBZ;

    // ---- window range of this tile ----
    auto rowmax = [&](int k) {  // last row touched by window k in the apply phase (H, T right)
        return (qp >= 2) ? j1 + max(0, k * r) : j1 + max(0, (k - qp + 1) * r);
    };
    auto cstart = [&](int k) {  // left updates touch columns > cstart(k) (corrected i5 / i6)
        return mode == CM_A_LEFT ? j1 + qp - 1 + max(0, (k - 1) * r + 1) : j1 + qp + (k + 1) * r - 1;
    };
    int kstart = K - 1, kend = 0;
    if (mode == CM_AB_RIGHT) {
        if (rowmax(K - 1) < R0) return false;
        while (kend < K - 1 && rowmax(kend) < R0) ++kend;
    } else if (mode == CM_A_LEFT || mode == CM_B_LEFT) {
        while (kstart >= 0 && cstart(kstart) >= R1) --kstart;
        if (kstart < 0) return false;
    }
    const int tid = threadIdx.x - grp * CH_NT, lane = tid & 31, warp = tid >> 5;  // (within the group)
    const int wn = warp % WN, wm = warp / WN;
    // gbar: barrier of this tile group (chain_kernel2: group g uses bar g + 1; chain_kernel: the CTA
    // barrier 0)
    auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(gbar), "r"(CH_NT) : "memory"); };
    // ---- step sequence: from window khi downward, a step covers windows [klo, khi]: a whole
    // merge group [mg P, mg P + P - 1] when khi is its top and the tile is fully inside every
    // window of it (no staircase / column limit), else the single window khi ----
    auto step_lo = [&](int khi) -> int {
        if (PM <= 1) return khi;
        const int glo = (khi / PM) * PM;
        if (khi != min(K - 1, glo + PM - 1) || glo < kend) return khi;
        bool full = true;
        if (mode == CM_AB_RIGHT) full = R1 <= j1 + max(0, (glo - qp + 1) * r);
        else if (mode == CM_A_LEFT || mode == CM_B_LEFT) full = R0 > cstart(khi);
        return full ? glo : khi;
    };
    auto step_blk = [&](int khi, int klo) -> const S* {
        if (WYm) return J.Blk + (size_t)khi * chain_wy_stride<S>(WP, QPw);
        return klo < khi ? J.MBlk + ((size_t)(klo / PM) * WP) * LDB : J.Blk + ((size_t)khi * WP) * LDB;
    };
    auto step_w = [&](int khi, int klo) { return min(qp + (khi - klo + 1) * r - 1, n - (j1 + klo * r + 1) + 1); };

    // zero the circular buffer (padded K rows of the blocks are zero; keep X finite)
    for (int e = tid; e < CIRC * CH_LDX; e += CH_NT) X[e] = S(0.0);
    if (tid == 0) {
        for (int s = 0; s < CH_STAGES; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    gsync();

    // global element access (1-based tile row g, chain index c)
    auto gptr = [&](int g, int c) -> S* {
        return trans ? &IDX(J.M, J.ld, c, g) : &IDX(J.M, J.ld, g, c);
    };
    // load chain indices [c0, c0+cnt) into circular positions starting at p (cp.async)
    // (lanes run along the contiguous direction of the global matrix; no integer division)
    const bool hint = mode == CM_PLAIN && P.stream_plain != 0;
    const unsigned long long pol = hint ? l2_evict_first_policy() : 0ull;
    auto load_cols = [&](int c0, int cnt, int p) {
        if (!trans) {
            for (int l = warp; l < cnt; l += NW) {
                int pos = p + l;
                if (pos >= CIRC) pos -= CIRC;
                if (hint)
                    for (int i = lane; i < nr; i += 32) cp_async_elem_hint(&X[pos * CH_LDX + i], gptr(R0 + i, c0 + l), pol);
                else
                    for (int i = lane; i < nr; i += 32) cp_async_elem(&X[pos * CH_LDX + i], gptr(R0 + i, c0 + l));
            }
        } else {
            if (P.tmap) {
                // 4 consecutive chain indices (32 B of one matrix column) x 8 tile rows per warp
                // instruction: conflict-free in shared memory with the strides above (a warp along
                // the chain index alone writes with stride CH_LDX: four-way conflicts)
                const int ngl = (cnt + 3) >> 2;
                for (int u = warp; u < 4 * ngl; u += NW) {
                    const int i = (u & 3) * 8 + (lane >> 2), l = (u >> 2) * 4 + (lane & 3);
                    if (i < nr && l < cnt) {
                        int pos = p + l;
                        if (pos >= CIRC) pos -= CIRC;
                        cp_async_elem(&X[pos * CH_LDX + i], gptr(R0 + i, c0 + l));
                    }
                }
            } else
            for (int i = warp; i < nr; i += NW)
                for (int l = lane; l < cnt; l += 32) {
                    int pos = p + l;
                    if (pos >= CIRC) pos -= CIRC;
                    cp_async_elem(&X[pos * CH_LDX + i], gptr(R0 + i, c0 + l));
                }
        }
    };
    auto store_cols = [&](int c0, int cnt, int p) {
        if (!trans) {
            for (int l = warp; l < cnt; l += NW) {
                int pos = p + l;
                if (pos >= CIRC) pos -= CIRC;
                if (hint)
                    for (int i = lane; i < nr; i += 32) st_hint(gptr(R0 + i, c0 + l), X[pos * CH_LDX + i], pol);
                else
                    for (int i = lane; i < nr; i += 32) *gptr(R0 + i, c0 + l) = X[pos * CH_LDX + i];
            }
        } else {
            if (P.tmap) {
                const int ngl = (cnt + 3) >> 2;
                for (int u = warp; u < 4 * ngl; u += NW) {
                    const int i = (u & 3) * 8 + (lane >> 2), l = (u >> 2) * 4 + (lane & 3);
                    if (i < nr && l < cnt) {
                        int pos = p + l;
                        if (pos >= CIRC) pos -= CIRC;
                        *gptr(R0 + i, c0 + l) = X[pos * CH_LDX + i];
                    }
                }
            } else
            for (int i = warp; i < nr; i += NW)
                for (int l = lane; l < cnt; l += 32) {
                    int pos = p + l;
                    if (pos >= CIRC) pos -= CIRC;
                    *gptr(R0 + i, c0 + l) = X[pos * CH_LDX + i];
                }
        }
    };

    // ---- block ring producer (thread 0): chunk sequence over (step, chunk) ----
    int pk = kstart, pc = 0;  // top window of the step being issued, next chunk of it
    int pklo = step_lo(kstart);
    unsigned pseq = 0;
    // chunks per step: dense -- ceil(w / 16) chunks of the block's rows; WY -- ceil(w / 16) chunks of
    // Y's rows (16 x LDY), then QP / 16 chunks of T Y^* (16 x LDB)
    auto step_chunks = [&](int khi, int klo) {
        const int nk = (step_w(khi, klo) + CH_KC - 1) / CH_KC;
        return WYm ? nk + QPw / CH_KC : nk;
    };
    auto issue_next = [&]() {
        if (tid != 0 || pk < kend) return;
        const int s = pseq % CH_STAGES;
        const S* src;
        unsigned bytes;
        if (WYm) {
            const int nk = (step_w(pk, pklo) + CH_KC - 1) / CH_KC;
            if (pc < nk) {
                src = step_blk(pk, pklo) + (size_t)pc * CH_KC * LDY;
                bytes = CH_KC * LDY * sizeof(S);
            } else {
                src = step_blk(pk, pklo) + (size_t)WP * LDY + (size_t)(pc - nk) * CH_KC * LDB;
                bytes = CH_KC * LDB * sizeof(S);
            }
        } else {
            src = step_blk(pk, pklo) + (size_t)pc * CH_KC * LDB;
            bytes = CH_KC * LDB * sizeof(S);
        }
        mbar_expect_tx(&bars[s], bytes);
        bulk_g2s(ring + (size_t)s * CH_KC * LDB, src, bytes, &bars[s]);
        ++pseq;
        if (++pc == step_chunks(pk, pklo)) {
            pc = 0;
            pk = pklo - 1;
            if (pk >= kend) pklo = step_lo(pk);
        }
    };
    for (int s = 0; s < CH_STAGES - 1; ++s) issue_next();

    // first step: all of its columns
    int p = 0;  // circular position of the current step's first column
    {
        const int klo0 = step_lo(kstart);
        const int c0 = j1 + klo0 * r + 1;
        load_cols(c0, step_w(kstart, klo0), 0);
        cp_async_commit();
    }
    unsigned cseq = 0;  // consumer chunk sequence
    // profile (tile 0 of job 0, thread 0): 0 wait+prefetch, 1 MMA, 2 epilogue, 3 staircase,
    // 4 store, 5 steps, 6 merged steps, 7 staircase steps
    const bool prf = P.prof && jb_ == 0 && bid == P.prof_tile && tid == 0;
    long long pc_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc_ = clock64();
    auto tick = [&](int slot) {
        if (prf) {
            const long long now = clock64();
            pc_[slot] += now - tc_;
            tc_ = now;
        }
    };
    for (int k = kstart, klo = step_lo(kstart); k >= kend;) {
        const bool merged = klo < k;
        const int c0 = j1 + klo * r + 1;
        const int wk = step_w(k, klo);
        const bool has_next = klo - 1 >= kend;
        const int nklo = has_next ? step_lo(klo - 1) : 0;
        const int shift = has_next ? (klo - nklo) * r : 0;  // fresh columns of the next step
        const int cn = has_next ? min(qp - 1, wk) : 0;      // carried into the next step
        cp_async_wait_all();
        gsync();
        // prefetch: fresh columns of the next step and (H/T right) this window's staircase reflectors
        if (has_next) {
            int pn = p - shift;
            if (pn < 0) pn += CIRC;
            load_cols(c0 - shift, shift, pn);
        }
        const int i5s = j1 + 1 + max(0, (k - qp + 1) * r);
        const bool stair = !merged && mode == CM_AB_RIGHT && qp >= 2 && max(i5s, R0) <= min(rowmax(k), R1);
        if (stair) {
            const S* src = P.Zr + (size_t)k * (r + 1);
            for (int t = 1 + warp; t < qp; t += NW)
                for (int c = lane; c <= r; c += 32)
                    cp_async_elem(&zsm[(size_t)t * (r + 1) + c], src + (size_t)t * K * (r + 1) + c);
        }
        cp_async_commit();
        tick(0);

        // ---- Y = X(:, window) * B_k on the tensor cores ----
        Acc<S> acc[MT][NTL];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NTL; ++nt) acc_zero(acc[mt][nt]);
        const int nch = (wk + CH_KC - 1) / CH_KC;
        const int rowb = wm * (CH_BM / WM) + (lane >> 2);
        const int colb = wn * (WP / WN) + (lane >> 2);
        if (WYm) {
            // ---- WY step: A = X(:, window) Y (QP = 32 columns, one 8-column slice per warp column),
            // staged in smem, then acc = A (T Y^*) and X -= acc in the epilogue ----
            constexpr int KS = CH_KC / 4;
            Acc<S> a1[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) acc_zero(a1[mt]);
            const int colq = wn * 8 + (lane >> 2);
            for (int ch = 0; ch < nch; ++ch) {
                const int s = cseq % CH_STAGES;
                mbar_wait(&bars[s], (cseq / CH_STAGES) & 1);
                gsync();
                issue_next();
                const S* Bs = ring + (size_t)s * CH_KC * LDB;
                S a[KS][MT], b[KS];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int kl = ch * CH_KC + ks * 4 + (lane & 3);
                    int pos = p + kl;
                    if (pos >= CIRC) pos -= CIRC;
                    if (pos >= CIRC) pos -= CIRC;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) a[ks][mt] = X[pos * CH_LDX + rowb + mt * 8];
                    b[ks] = Bs[(ks * 4 + (lane & 3)) * LDY + colq];
                }
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) mma_step(a1[mt], a[ks][mt], b[ks]);
                ++cseq;
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h) Abuf[(wn * 8 + (lane & 3) * 2 + h) * CH_LDX + rowb + mt * 8] = acc_get(a1[mt], h);
            gsync();  // A complete
            for (int ch = 0; ch < QPw / CH_KC; ++ch) {
                const int s = cseq % CH_STAGES;
                mbar_wait(&bars[s], (cseq / CH_STAGES) & 1);
                gsync();
                issue_next();
                const S* Bs = ring + (size_t)s * CH_KC * LDB;
                if (wn * (WP / WN) < wk) {
                    S a[KS][MT], b[KS][NTL];
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {
                        const int kk = ch * CH_KC + ks * 4 + (lane & 3);
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) a[ks][mt] = Abuf[kk * CH_LDX + rowb + mt * 8];
#pragma unroll
                        for (int nt = 0; nt < NTL; ++nt) b[ks][nt] = Bs[(ks * 4 + (lane & 3)) * LDB + colb + nt * 8];
                    }
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                            for (int nt = 0; nt < NTL; ++nt) mma_step(acc[mt][nt], a[ks][mt], b[ks][nt]);
                }
                ++cseq;
            }
        } else
        for (int ch = 0; ch < nch; ++ch) {
            const int s = cseq % CH_STAGES;
            mbar_wait(&bars[s], (cseq / CH_STAGES) & 1);
            gsync();  // everyone is past chunk cseq-1: its stage may be refilled
            issue_next();
            const S* Bs = ring + (size_t)s * CH_KC * LDB;
            if (wn * (WP / WN) < wk) {  // warp-uniform: this warp's columns exist in the step
                // the chunk's fragments first (their shared-memory latencies overlap), then the MMAs
                constexpr int KS = CH_KC / 4;
                S a[KS][MT], b[KS][NTL];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int kl = ch * CH_KC + ks * 4 + (lane & 3);  // window-local column (K index)
                    int pos = p + kl;
                    if (pos >= CIRC) pos -= CIRC;
                    if (pos >= CIRC) pos -= CIRC;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) a[ks][mt] = X[pos * CH_LDX + rowb + mt * 8];
#pragma unroll
                    for (int nt = 0; nt < NTL; ++nt)
                        b[ks][nt] = maybe_conj(Bs[(ks * 4 + (lane & 3)) * LDB + colb + nt * 8], trans);
                }
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int nt = 0; nt < NTL; ++nt) mma_step(acc[mt][nt], a[ks][mt], b[ks][nt]);
            }
            ++cseq;
        }
        gsync();  // all reads of X done
        tick(1);
        // ---- epilogue: write Y back in place for the rows the mode updates ----
        const int ylo = (!merged && (mode == CM_A_LEFT || mode == CM_B_LEFT)) ? cstart(k) : 0;
        const int yhi = (!merged && mode == CM_AB_RIGHT) ? j1 + max(0, (k - qp + 1) * r) : 0x7fffffff;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int row = rowb + mt * 8;
            const int g = R0 + row;
            const bool upd = row < nr && g > ylo && g <= yhi;
#pragma unroll
            for (int nt = 0; nt < NTL; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = wn * (WP / WN) + nt * 8 + (lane & 3) * 2 + h;
                    if (upd && col < wk) {
                        int pos = p + col;
                        if (pos >= CIRC) pos -= CIRC;
                        if (WYm) X[pos * CH_LDX + row] -= acc_get(acc[mt][nt], h);  // X - (X Y)(T Y^*)
                        else X[pos * CH_LDX + row] = maybe_conj(acc_get(acc[mt][nt], h), false);
                    }
                }
        }
        tick(2);
        if (stair) {
            // Alg. 4 lines 4-9: rows i5s..i4(k,j) get Z_k^j, j ascending, in blocks of BZ reflectors
            // (compact WY per block: Z_t ... Z_{t+BZ-1} = I - Y T Y^*): the BZ dots of a row are
            // independent, so a block costs about one reflector's latency.  A row gets the
            // reflectors t with g <= i4a(t) (a suffix); zeroing the dots outside it and the upper
            // triangular T keep exactly that suffix.  Steps without a reflector have a zero record.
            cp_async_wait_all();
            gsync();
            tick(2);  // (profile: the wait for the staircase data counts as epilogue)
            constexpr int TPR = CH_NT / CH_BM, BZ = CH_SBZ;  // threads per row, reflectors per block
            const int row = tid / TPR, part = tid % TPR;
            const int g = R0 + row;
            const bool active = row < nr && g >= i5s && g <= rowmax(k);
            const int lo = max(i5s, R0);
            int t0 = 1;  // first reflector reaching this tile's staircase rows (uniform)
            if (j1 < lo) t0 = max(1, (lo - j1 + r - 1) / r - k + qp - 1);
            const int nbk = (qp - t0 + BZ - 1) / BZ;
            S* Gs = zsm + (size_t)(qp + 1) * (r + 1);
            S* Ts = Gs + (size_t)((qp + BZ - 1) / BZ) * BZ * BZ;
            auto msz = [&](int t) { return (t < qp) ? min(r, n - (j1 + t + k * r)) : 0; };
            auto zrec = [&](int t) { return zsm + (size_t)t * (r + 1); };
            // G(i,j) = z_i^* z_j over the columns both touch (i < j within a block)
            for (int e = tid; e < nbk * BZ * BZ; e += CH_NT) {
                const int bi = e / (BZ * BZ), i = (e / BZ) % BZ, jj = e % BZ;
                const int ti = t0 + bi * BZ + i, tj = t0 + bi * BZ + jj;
                S gg = S(0.0);
                if (i < jj && tj < qp) {
                    const int mi = msz(ti), mj = msz(tj);
                    const S* zi = zrec(ti);
                    const S* zj = zrec(tj);
                    for (int c = tj; c < min(ti + mi, tj + mj); ++c) gg += conj_mul(zi[c - ti], zj[c - tj]);
                }
                Gs[e] = gg;
            }
            gsync();
            // block factor (xLARFT forward): T(i,i) = sigma_i, T(i,j) = -sigma_j sum_l T(i,l) G(l,j)
            // rows of T are independent given G: T(i,j) = -sigma_j sum_{l=i}^{j-1} T(i,l) G(l,j),
            // so one thread per (block, row) runs along its row
            for (int e = tid; e < nbk * BZ; e += CH_NT) {
                const int bi = e / BZ, i = e % BZ;
                S* Tr = Ts + ((size_t)bi * BZ + i) * BZ;
                const S* Gb = Gs + (size_t)bi * BZ * BZ;
                S tr[BZ];
#pragma unroll
                for (int jj = 0; jj < BZ; ++jj) {
                    const int tj = t0 + bi * BZ + jj;
                    const S sj = (tj < qp && msz(tj) >= 2) ? zrec(tj)[r] : S(0.0);
                    S v = S(0.0);
                    if (jj == i) {
                        v = sj;
                    } else if (jj > i) {
                        S acc = S(0.0);
#pragma unroll
                        for (int l = 0; l < BZ; ++l)
                            if (l >= i && l < jj) acc += tr[l] * Gb[l * BZ + jj];
                        v = -(sj * acc);
                    }
                    tr[jj] = v;
                    Tr[jj] = v;
                }
            }
            gsync();
            tick(0);  // (profile: the block factors count as wait+prefetch)
            // block rounds, with compile-time trip counts (MR >= r): no loop branches in the chain
            auto rounds = [&](auto mrc) {
                constexpr int MR = decltype(mrc)::value;
                constexpr int ND = (MR + TPR - 1) / TPR, NU = (BZ - 1 + MR + TPR - 1) / TPR;
                for (int bi = 0; bi < nbk; ++bi) {
                    const int tb = t0 + bi * BZ;
                    S wv[BZ];
                    int mt[BZ];
#pragma unroll
                    for (int i = 0; i < BZ; ++i) {
                        const int t = tb + i;
                        const int m = msz(t);
                        mt[i] = m;
                        const bool on = active && m >= 2 && g <= j1 + max(0, (k + t - qp + 1) * r);
                        const S* zr = zrec(t);
                        S d = S(0.0);
#pragma unroll
                        for (int u = 0; u < ND; ++u) {
                            const int c = part + u * TPR;
                            if (on && c < m) {
                                int pos = p + t + c;
                                if (pos >= CIRC) pos -= CIRC;
                                d = fma_s(X[pos * CH_LDX + row], zr[c], d);
                            }
                        }
                        wv[i] = d;
                    }
#pragma unroll
                    for (int o = 1; o < TPR; o <<= 1)
#pragma unroll
                        for (int i = 0; i < BZ; ++i) wv[i] += shfl_xor(wv[i], o);
                    S w2[BZ];
#pragma unroll
                    for (int i = 0; i < BZ; ++i) {
                        S acc = S(0.0);
#pragma unroll
                        for (int jj = 0; jj <= i; ++jj) acc += wv[jj] * Ts[(bi * BZ + jj) * BZ + i];
                        w2[i] = acc;
                    }
                    if (active) {
#pragma unroll
                        for (int u = 0; u < NU; ++u) {  // window columns tb + cc
                            const int cc = part + u * TPR;
                            S acc = S(0.0);
#pragma unroll
                            for (int i = 0; i < BZ; ++i) {
                                const int ci = cc - i;
                                if (ci >= 0 && ci < mt[i]) acc += w2[i] * conjv(zrec(tb + i)[ci]);
                            }
                            if (cc < BZ - 1 + mt[0] && tb + cc < wk) {
                                int pos = p + tb + cc;
                                if (pos >= CIRC) pos -= CIRC;
                                X[pos * CH_LDX + row] -= acc;
                            }
                        }
                    }
                }
            };
            if (r <= 8) rounds(std::integral_constant<int, 8>{});
            else if (r <= 16) rounds(std::integral_constant<int, 16>{});
            else if (r <= 32) rounds(std::integral_constant<int, 32>{});
            else if (r <= 64) rounds(std::integral_constant<int, 64>{});
            else rounds(std::integral_constant<int, 128>{});
        }
        gsync();
        tick(3);
        // columns [cn, wk) are final for this group; [0, cn) stay as window k-1's carry
        {
            int po = p + cn;
            if (po >= CIRC) po -= CIRC;
            store_cols(c0 + cn, wk - cn, po);
        }
        tick(4);
        if (prf) {
            pc_[5] += 1;
            pc_[6] += merged;
            pc_[7] += stair;
        }
        p -= shift;
        if (p < 0) p += CIRC;
        k = klo - 1;
        klo = nklo;
    }
    cp_async_wait_all();
    if (prf)
        for (int i = 0; i < 8; ++i) atomicAdd((unsigned long long*)&P.prof[i], (unsigned long long)pc_[i]);
    return true;
}

// Persistent over tiles: CTA b processes tiles b, b + gridDim.x, ... (a grid smaller than the
// tile count leaves SMs free for the chase kernel running concurrently on another stream).
// resident CTAs per SM the register budget targets (real: 3 x 256 threads; complex: 2)
template <typename S, int WP>
__host__ __device__ constexpr int chain_minb() { return (sizeof(S) == 8 && WP <= 128) ? 768 / chain_nt(WP) : 512 / chain_nt(WP); }

template <typename S, int WP>
__global__ void __launch_bounds__(chain_nt(WP), chain_minb<S, WP>()) chain_kernel(ChainParams<S> P) {
    if (input_rejected(P.gate)) return;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int total = P.job[0].ntiles + (P.njobs > 1 ? P.job[1].ntiles : 0);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smraw);
    for (int b = blockIdx.x; b < total; b += gridDim.x) {
        const bool used = chain_tile<S, WP>(P, b, smraw, 0, 0);
        __syncthreads();
        if (used && threadIdx.x == 0)
            for (int s = 0; s < CH_STAGES; ++s)
                asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&bars[s])) : "memory");
        __syncthreads();
    }
}

// Two tile groups per CTA (2 x CH_NT threads, 2 x the shared memory of chain_kernel): group g walks
// tiles 2 b + g.  For the side-stream Q/Z chains, which must keep to one CTA per SM (the rest of the
// SMs belong to the next chase): the groups' steps interleave, so one group's epilogue, stores and
// barriers overlap the other group's DMMA stream (named barriers per group).
template <typename S, int WP>
__global__ void __launch_bounds__(2 * chain_nt(WP), 1) chain_kernel2(ChainParams<S> P, unsigned grp_bytes) {
    if (input_rejected(P.gate)) return;
    extern __shared__ __align__(16) unsigned char smraw[];
    constexpr int NT = chain_nt(WP);
    const int grp = threadIdx.x / NT;
    unsigned char* sm = smraw + (size_t)grp * grp_bytes;
    const int total = P.job[0].ntiles + (P.njobs > 1 ? P.job[1].ntiles : 0);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
    for (int b = 2 * blockIdx.x + grp; b < total; b += 2 * gridDim.x) {
        const bool used = chain_tile<S, WP>(P, b, sm, grp, 1 + grp);
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(NT) : "memory");
        if (used && threadIdx.x == grp * NT)
            for (int s = 0; s < CH_STAGES; ++s)
                asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&bars[s])) : "memory");
        asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(NT) : "memory");
    }
}
