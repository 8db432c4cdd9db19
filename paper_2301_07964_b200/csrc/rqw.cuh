// rqw.cuh -- the opposite reflector's RQ for long reflectors (MAXM = 64, 128): Householder RQ of
// the m x m block B(i1:i2,i1:i2), rows bottom-up in xGERQ2 order (readings c3/c4),
// returning only uu = Q~^* e1 = conj(Q~(1,:))^T (the direction of Z_k^j).
//
// Same mathematics as rq_direction (chase.cuh), organised for latency at large m:
//  * warp w owns the RPW = MAXM/NW consecutive rows [w RPW, (w+1) RPW) in registers: lane group
//    g = lane/4 (8 groups of 4 lanes) holds rows w RPW + g + 8s (s < RPL = RPW/8), lane q = lane%4
//    of the group the columns 4e + q (e < CPT = MAXM/4) -- a row's dot products are in-lane
//    partial sums finished by a 2-level shuffle within the group;
//  * stage i (pivot row i, i = m-1 .. 1) is computed by the warp owning row i: the pivot row goes
//    through shared memory (it is also the record the reverse pass needs), every row of the warp
//    forms its dot with it in the same pass (the pivot row's own dot is its norm), so the RPW
//    stages of a block run inside one warp with no CTA barrier on the chain;
//  * the warps owning rows above apply each published stage to their rows, trailing (pivot row,
//    scalars in shared memory, an mbarrier per stage); when a warp's own rows come up it has already
//    applied every stage below them.
// Stage i generates H_i = I - tau h h^* with h_c = conj(C[i][c]) / K2 (c < i), h_i = 1,
// tau = K1 |K2|^2 (K2 = alpha - beta, K1 = tau / |K2|^2; real K1 = 1/(s2 + |alpha| nrm)) from
// alpha = conj(C[i][i]) and the tail conj(C[i][0:i)) (oracle_rq_first_row's larfg), and applies it
// to rows 0..i-1 on columns 0..i-1 (column i is dead after stage i).
//
// uu = H_{m-1} ... H_1 (H_0) e1 is formed at the end by warp 0 from the stored pivot rows, one
// block (the RPW stages of a warp, ascending) at a time.  With b_p = h_p^* z the block's sequence
// of applications is z <- z - sum_p delta_p h_p, delta = M b, M = (I + L)^{-1} diag(tau),
// L_pj = tau_p h_p^* h_j (j < p).  The dead rows of a block (rows whose stage is done still hold
// their pivot rows) get their dot with each later pivot in the same reduction as the live rows,
// which gives L; the owning warp forms M once its block is done.
//
// Storage (shared): hb (row-major, ld HLD >= MAXM + 4): the pivot row i at hb[i HLD + c], c <= i;
// L_pj / M_pj (j < p, same block) at hb[j HLD + p] (strict upper part); hb[i HLD + MAXM + 0..3] =
// K1, K2, 1/conj(K2) (0 if K2 = 0), tau of stage i; bars: MAXM mbarriers (rqw_bars_init), par:
// the parity of this call (0, 1, 0, ... per CTA).  hb may alias the input block (read into
// registers first).
#pragma once
#include "scalar.cuh"

#ifdef RQW_TRACE
__device__ long long rqw_trace[4096];  // dev: clock at each stage start (pivot warp), per warp block start/end
#define RQW_T(idx) do { if ((threadIdx.x & 31) == 0) rqw_trace[idx] = clock64(); } while (0)
#define RQW_TS(i, k) do { if ((i) == 60 && (threadIdx.x & 31) == 0) rqw_trace[3200 + (k)] = clock64(); } while (0)
#else
#define RQW_T(idx) do { } while (0)
#define RQW_TS(i, k) do { } while (0)
#endif

__device__ __forceinline__ void rqw_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename S, int MAXM, int NW>
struct RQW {
    static constexpr int RPW = MAXM / NW;  // rows per warp
    static constexpr int RPL = RPW / 8;    // rows per lane (8 lane groups)
    static constexpr int CPT = MAXM / 4;   // columns per lane (4 lanes per row)
    static constexpr int CPL = MAXM / 32;  // reverse pass: columns per lane
    static constexpr int NTHR = NW * 32;
    static_assert(RPW % 8 == 0 && (RPL == 1 || RPL == 2) && MAXM % 32 == 0, "rqw layout");
};

// Sum of N values over the 32 lanes of a warp, every lane receiving all N totals:
// reduce-scatter (halve the value set at each of the first log2 N butterfly levels), the rest of
// the butterfly on one value, then N broadcasts.  N - 1 + (5 - log2 N) + N shuffles instead of 5N.
template <typename S, int N>
__device__ __forceinline__ void warp_allreduce_n(S (&v)[N]) {
    static_assert((N & (N - 1)) == 0 && N >= 1 && N <= 32, "N power of two <= 32");
    const int lane = threadIdx.x & 31;
    S a[N];
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = v[k];
    int lvl = 16;
#pragma unroll
    for (int h = N / 2; h >= 1; h /= 2) {  // level with offset lvl keeps h of the 2h values
        const bool up = (lane & lvl) != 0;
#pragma unroll
        for (int k = 0; k < h; ++k) {
            const S keep = up ? a[k + h] : a[k];
            const S send = up ? a[k] : a[k + h];
            a[k] = keep + shfl_xor(send, lvl);
        }
        lvl >>= 1;
    }
    S t = a[0];
#pragma unroll
    for (int o = lvl; o >= 1; o >>= 1) t += shfl_xor(t, o);
    // the total of value k sits in the lanes whose top log2 N bits (16, 8, ...) spell k
#pragma unroll
    for (int k = 0; k < N; ++k) {
        int src = 0, bit = 16;
#pragma unroll
        for (int h = N / 2; h >= 1; h /= 2) {
            if (k & h) src |= bit;
            bit >>= 1;
        }
        v[k] = shfl_idx(t, src);
    }
}

// Stage hand-off: one mbarrier per stage (count 32).  Every lane of the pivot warp arrives
// (release, CTA scope: its own shared-memory stores of the stage), trailing warps sleep in
// try_wait (acquire).  The barriers are initialised once per CTA (rqw_bars_init) and every one of
// them completes exactly one phase per RQ call -- warp 0 arrives on the unused ones (stages 0 and
// >= m) at the start -- so call c waits for parity c & 1.  (Polling a shared-memory flag instead
// put a MEMBAR on the pivot warp's chain; re-initialising the barriers per call was unreliable.)
__device__ __forceinline__ void rqw_bars_init(uint64_t* bars, int n) {  // one warp, then a CTA barrier
    const int lane = threadIdx.x & 31;
    for (int k = lane; k < n; k += 32) {
        const unsigned a = (unsigned)__cvta_generic_to_shared(bars + k);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(a) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void rqw_arrive(uint64_t* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void rqw_wait(uint64_t* bar, int parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RQW_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RQW_WAIT_%=;\n"
        "}\n" ::"r"(a), "r"(parity)
        : "memory");
}
__device__ __forceinline__ double rqw_rcp(double x) { return fast_rcp(x); }
__device__ __forceinline__ zc rqw_rcp(zc x) { return conjv(x) * fast_rcp(abs2(x)); }

// Householder scalars of a stage (reading c1 applied to conj(row i)): K1, K2 (both zero: H = I).
template <typename S>
__device__ __forceinline__ void rqw_scalars(S alpha, double nx, S& K1, S& K2) {
    K1 = S(0.0);
    K2 = S(0.0);
    if (nx == 0.0 && im(alpha) == 0.0) return;
    const double s2 = abs2(alpha) + nx;
    const double y = fast_rsqrt(s2);
    const double nrm = s2 * y;
    const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
    K2 = alpha - S(beta);
    if constexpr (sizeof(S) == 8) {
        K1 = S(fast_rcp(s2 + fabs(re(alpha)) * nrm));
    } else {
        const S tau = (S(beta) - alpha) * ((re(alpha) >= 0.0) ? -y : y);  // (beta - alpha) / beta
        K1 = tau * fast_rcp(abs2(K2));
    }
}

// CPT (a multiple of 8) doubles p[4 e + q] (stride 4) from shared memory, issued back to back in
// blocks of 8 (ptxas otherwise interleaves each load with its consumer and serialises them)
template <int CPT>
__device__ __forceinline__ void rqw_lds_stride4(double (&x)[CPT], const double* p) {
    static_assert(CPT % 8 == 0, "rqw_lds_stride4");
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
#pragma unroll
    for (int b = 0; b < CPT; b += 8)
        asm volatile(
            "ld.shared.f64 %0, [%8];\n ld.shared.f64 %1, [%8+32];\n ld.shared.f64 %2, [%8+64];\n"
            "ld.shared.f64 %3, [%8+96];\n ld.shared.f64 %4, [%8+128];\n ld.shared.f64 %5, [%8+160];\n"
            "ld.shared.f64 %6, [%8+192];\n ld.shared.f64 %7, [%8+224];\n"
            : "=d"(x[b]), "=d"(x[b + 1]), "=d"(x[b + 2]), "=d"(x[b + 3]), "=d"(x[b + 4]), "=d"(x[b + 5]),
              "=d"(x[b + 6]), "=d"(x[b + 7])
            : "r"(a + 256u * (unsigned)(b / 8))
            : "memory");
}
template <int CPT>
__device__ __forceinline__ void rqw_lds_stride4(zc (&x)[CPT], const zc* p) {  // (complex: plain loads)
#pragma unroll
    for (int e = 0; e < CPT; ++e) x[e] = p[4 * e];
}

// v[e] for a run-time, warp-uniform e < N (N a power of two) by a binary tree of selects on the
// bits of e (a run-time register index would put v in local memory)
template <typename S, int N>
__device__ __forceinline__ S rqw_sel(const S (&v)[N], int e) {
    static_assert((N & (N - 1)) == 0, "power of two");
    S t[N];
#pragma unroll
    for (int k = 0; k < N; ++k) t[k] = v[k];
#pragma unroll
    for (int h = N / 2, b = 1; h >= 1; h /= 2, b <<= 1)
#pragma unroll
        for (int k = 0; k < h; ++k) t[k] = (e & b) ? t[2 * k + 1] : t[2 * k];
    return t[0];
}

// val[sp][e] for a run-time slot sp < RPL <= 2 as an explicit select (a run-time register index
// would put the whole array in local memory)
template <typename S, int RPL, int CPT>
__device__ __forceinline__ S rqw_pick(const S (&val)[RPL][CPT], int sp, int e) {
    static_assert(RPL == 1 || RPL == 2, "rows per lane");
    if constexpr (RPL == 1) return val[0][e];
    else return sp ? val[1][e] : val[0][e];
}

// One stage i applied by a warp to its rows.  OWN: the warp owns row i (it publishes the pivot row
// and the scalars, and its dead rows -- index in (i, ihi] -- record L entries); otherwise the pivot
// row and scalars are read after the stage's barrier.  val[s][e] = row (row0 + g + 8 s), column
// 4 e + q.  Once K2 is known the pivot warp replaces alpha = C[i][i] in the published row by
// conj(K2): a trailing row's f = K1 (row . conj(piv) + K2 row[i]) is then ONE dot over c <= i
// (column i is dead after stage i, so the update may write anything there).
template <typename S, int MAXM, int NW, bool OWN>
__device__ __forceinline__ void rqw_apply(S (&val)[RQW<S, MAXM, NW>::RPL][RQW<S, MAXM, NW>::CPT], int i, int row0,
                                          int ihi, S* hb, int HLD, uint64_t* bars, int par) {
    using CF = RQW<S, MAXM, NW>;
    constexpr int RPL = CF::RPL, CPT = CF::CPT;
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    S* pv = hb + (size_t)i * HLD;
    S pe[CPT];
    if constexpr (!OWN) {
        rqw_wait(bars + i, par);
        const S K1 = pv[MAXM];
        if (is_zero(K1)) return;  // H_i = I (uniform)
        // (every load issued unconditionally into its own register, masked afterwards: a predicated
        // load into a shared temporary serialises the loads; columns beyond i hold stale data)
        rqw_lds_stride4<CPT>(pe, pv + q);
#pragma unroll
        for (int e = 0; e < CPT; ++e) pe[e] = (4 * e + q <= i) ? pe[e] : S(0.0);
        S d[RPL];
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            S a0 = S(0.0), a1 = S(0.0);
#pragma unroll
            for (int e = 0; e < CPT; ++e) {
                if (e & 1) a1 = fma_s(val[s][e], conjv(pe[e]), a1);
                else a0 = fma_s(val[s][e], conjv(pe[e]), a0);
            }
            d[s] = a0 + a1;
        }
#pragma unroll
        for (int s = 0; s < RPL; ++s) d[s] += shfl_xor(d[s], 1);
#pragma unroll
        for (int s = 0; s < RPL; ++s) d[s] += shfl_xor(d[s], 2);
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            const S f = K1 * d[s];
#pragma unroll
            for (int e = 0; e < CPT; ++e) val[s][e] -= f * pe[e];  // (column i: dead)
        }
        return;
    } else {
        const int pr = i - row0;  // pivot slot: group pr & 7, row slot pr >> 3
        const int sp = pr >> 3, ei = i >> 2;  // column i: register ei of lane q = i & 3 (uniform)
        // The pivot row's columns 4 e + q for every lane q: CPT <= 16 by shuffles from the pivot's
        // lanes (no shared-memory round trip on the chain); CPT = 32 (register-bound) through shared
        // memory, where the trailing warps read it anyway.
        constexpr bool SHPIV = CPT <= 16;
        S alpha;
        if constexpr (SHPIV) {
            const int src = ((pr & 7) << 2) | q;
#pragma unroll
            for (int e = 0; e < CPT; ++e) pe[e] = shfl_idx(rqw_pick<S, RPL>(val, sp, e), src);
            alpha = conjv(shfl_idx(rqw_sel<S, CPT>(pe, ei), i & 3));
        } else {
            if (g == (pr & 7)) {
#pragma unroll
                for (int e = 0; e < CPT; ++e)
                    if (4 * e + q < i) pv[4 * e + q] = rqw_pick<S, RPL>(val, sp, e);
            }
            __syncwarp();
            rqw_lds_stride4<CPT>(pe, pv + q);
            {
                S av = (RPL == 2 && sp == 0) ? rqw_sel<S, CPT>(val[0], ei) : rqw_sel<S, CPT>(val[RPL - 1], ei);
                alpha = conjv(shfl_idx(av, ((pr & 7) << 2) | (i & 3)));
            }
        }
#pragma unroll
        for (int e = 0; e < CPT; ++e) pe[e] = (4 * e + q < i) ? pe[e] : S(0.0);
        RQW_TS(i, 1);
        // my rows: partial dots with conj(pivot) over c < i (the pivot row's own = its tail
        // norm^2), and row[i] (from the lane q = i & 3, summed by the same group reduction)
        S d[RPL], ri[RPL];
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            S a0 = S(0.0), a1 = S(0.0);
#pragma unroll
            for (int e = 0; e < CPT; ++e) {
                if (e & 1) a1 = fma_s(val[s][e], conjv(pe[e]), a1);
                else a0 = fma_s(val[s][e], conjv(pe[e]), a0);
            }
            d[s] = a0 + a1;
            ri[s] = (q == (i & 3)) ? rqw_sel<S, CPT>(val[s], ei) : S(0.0);
        }
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            d[s] += shfl_xor(d[s], 1);
            ri[s] += shfl_xor(ri[s], 1);
        }
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            d[s] += shfl_xor(d[s], 2);
            ri[s] += shfl_xor(ri[s], 2);
        }
        RQW_TS(i, 2);
        S dp = d[0];
        if constexpr (RPL == 2) dp = sp ? d[1] : d[0];
        const double nx = re(shfl_idx(dp, (pr & 7) << 2));
        S K1, K2;
        rqw_scalars(alpha, nx, K1, K2);
        RQW_TS(i, 3);
        const S tau = K1 * S(abs2(K2));
        // publish: (SHPIV: the pivot row, columns < i,) column i = conj(K2) (see above), the scalars;
        // then every lane arrives on the stage's barrier
        if constexpr (SHPIV) {
            if (lane < 4) {
#pragma unroll
                for (int e = 0; e < CPT; ++e)
                    if (4 * e + q < i) pv[4 * e + q] = pe[e];
            }
        }
        if (lane == 0) {
            pv[i] = conjv(K2);
            pv[MAXM] = K1;
            pv[MAXM + 1] = K2;
            pv[MAXM + 3] = tau;
        }
        __syncwarp();
        rqw_arrive(bars + i);
        RQW_TS(i, 4);
        // live rows (index < i): row[c] -= K1 (d + K2 row[i]) piv[c], c < i  (the next stage's input)
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            const int r = row0 + g + 8 * s;
            const S f = (r < i) ? K1 * (d[s] + K2 * ri[s]) : S(0.0);
#pragma unroll
            for (int e = 0; e < CPT; ++e) val[s][e] -= f * pe[e];
        }
        // off the chain: 1/conj(K2_i) for the reverse pass, and the dead rows r in (i, ihi]:
        // L_ri = tau_r h_r^* h_i = tau_r (d / K2_i + piv_r[i]) / conj(K2_r)
        const S rk = is_zero(K2) ? S(0.0) : rqw_rcp(conjv(K2));
        if (lane == 0) pv[MAXM + 2] = rk;
        const S r2 = conjv(rk);  // 1 / K2_i
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
            const int r = row0 + g + 8 * s;
            if (r > i && r <= ihi && q == 0) {
                const S* pr_ = hb + (size_t)r * HLD;
                hb[(size_t)i * HLD + r] = pr_[MAXM + 3] * ((d[s] * r2 + ri[s]) * pr_[MAXM + 2]);
            }
        }
        RQW_TS(i, 5);
    }
}

// Called by threads [0, NW*32) of the CTA (all of them together; named barrier 1).  Cb: m x m
// block (col-major, ld LDC); hb/HLD: work storage (see above); uu: output (m entries, written by
// warp 0); the caller synchronises before reading uu.
#ifndef HT_RQW_INLINE
#define HT_RQW_ATTR __noinline__
#else
#define HT_RQW_ATTR __forceinline__
#endif
// (not inlined: inside the chase kernel the caller's live state pushed this function into spills;
// as a call, the caller's registers are saved once around it and the RQ gets the register file)
template <typename S, int MAXM, int NW>
__device__ HT_RQW_ATTR void rq_direction_w(int m, const S* Cb, int LDC, S* hb, int HLD,
                                               uint64_t* bars, int par, S* uu) {
    using CF = RQW<S, MAXM, NW>;
    constexpr int RPW = CF::RPW, RPL = CF::RPL, CPT = CF::CPT, CPL = CF::CPL;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int row0 = w * RPW;
    // ---- rows into registers ----
    S val[RPL][CPT];
#pragma unroll
    for (int s = 0; s < RPL; ++s)
#pragma unroll
        for (int e = 0; e < CPT; ++e) {
            const int l = row0 + g + 8 * s, c = 4 * e + q;
            val[s][e] = (l < m && c < m) ? Cb[l + (size_t)c * LDC] : S(0.0);
        }
    if (w == 0)  // the stages this call does not have complete their phase now (see rqw_arrive)
        for (int i = 0; i < MAXM; ++i)
            if (i == 0 || i >= m) rqw_arrive(bars + i);
    rqw_bar(1, CF::NTHR);  // every row is in registers before hb (which may alias Cb) is written
    const int ihi = min(row0 + RPW, m) - 1;  // own stages: ihi .. ilo (descending)
    const int ilo = max(row0, 1);
    // ---- trailing: the stages of the rows below (i > ihi), as they are published ----
    for (int i = m - 1; i > ihi; --i) rqw_apply<S, MAXM, NW, false>(val, i, row0, ihi, hb, HLD, bars, par);
    RQW_T(1024 + w);
    // ---- own stages ----
    for (int i = ihi; i >= ilo; --i) {
        RQW_T(i);
        rqw_apply<S, MAXM, NW, true>(val, i, row0, ihi, hb, HLD, bars, par);
    }
    RQW_T(2048 + w);
    // ---- M = (I + L)^{-1} diag(tau) of this warp's block, in place of L (lane k: column k) ----
    if (ilo <= ihi) {
        __syncwarp();
        const int k = lane;
        if (k < RPW && row0 + k >= ilo && row0 + k <= ihi) {
            S x[RPW];  // column k of X = (I + L)^{-1} (unit lower triangular)
#pragma unroll
            for (int a = 0; a < RPW; ++a) x[a] = S(a == k ? 1.0 : 0.0);
#pragma unroll
            for (int a = 1; a < RPW; ++a) {
                if (a > k && row0 + a <= ihi) {
                    S acc0 = S(0.0), acc1 = S(0.0);
#pragma unroll
                    for (int b = 0; b < a; ++b)
                        if (b >= k) {
                            const S l = hb[(size_t)(row0 + b) * HLD + row0 + a];  // L_ab
                            if (b & 1) acc1 = fma_s(l, x[b], acc1);
                            else acc0 = fma_s(l, x[b], acc0);
                        }
                    x[a] = -(acc0 + acc1);
                }
            }
            const S tk = hb[(size_t)(row0 + k) * HLD + MAXM + 3];
            __syncwarp(__activemask());  // every L entry is read before M overwrites it
#pragma unroll
            for (int a = 1; a < RPW; ++a)
                if (a > k && row0 + a <= ihi) hb[(size_t)(row0 + k) * HLD + row0 + a] = x[a] * tk;  // M_ak
        }
    }
    rqw_bar(1, CF::NTHR);  // every stage and M entry stored
    RQW_T(3072 + w);
    if (w != 0) return;
    // ---- reverse pass (warp 0): z = H_{m-1} ... H_1 (H_0) e1, block by block; lane l holds
    // z[l + 32 e] ----
    S z[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) z[e] = S((lane + 32 * e) == 0 ? 1.0 : 0.0);
    if constexpr (sizeof(S) != 8) {
        // complex stage 0: H_0 = I - tau0 e1 e1^*, alpha = conj(R~(0,0)) (row 0 after all stages:
        // lane 0 of warp 0, register (0, 0))
        const S a00 = shfl_idx(val[0][0], 0);
        const S alpha = conjv(a00);
        S tau0 = S(0.0);
        if (im(alpha) != 0.0) {
            const double nrm = sqrt(abs2(alpha));
            const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
            tau0 = (S(beta) - alpha) * (1.0 / beta);
        }
        if (lane == 0) z[0] -= tau0 * z[0];
    }
    for (int W = 0; W < NW; ++W) {
        const int lo = max(W * RPW, 1), hi = min((W + 1) * RPW, m) - 1;
        if (lo > hi) break;
        // a_p = sum_{c<i} piv_i[c] z_c  (i = W RPW + p); b_p = h_i^* z = a_p / conj(K2_i) + z_i
        S a[RPW], pvr[RPW][CPL];
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const int i = W * RPW + p;
            const bool on = i >= lo && i <= hi;
            const S* pi = hb + (size_t)min(i, MAXM - 1) * HLD;
            S a0 = S(0.0);
#pragma unroll
            for (int e = 0; e < CPL; ++e) pvr[p][e] = pi[lane + 32 * e];
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const int c = lane + 32 * e;
                pvr[p][e] = (on && c < i) ? pvr[p][e] : S(0.0);
                a0 = fma_s(pvr[p][e], z[e], a0);
            }
            a[p] = a0;
        }
        // everything this block needs from shared memory, issued before the reduction:
        // rk_p = 1/conj(K2_i), and lane p's row of M (M_pj, j < p, at hb[(lo_W + j) HLD + i_p];
        // M_pp = tau_p)
        S rkv[RPW], mrow[RPW];
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const int i = min(W * RPW + p, MAXM - 1);
            rkv[p] = hb[(size_t)i * HLD + MAXM + 2];
            const int ij = min(W * RPW + p, MAXM - 1), il = min(W * RPW + lane, MAXM - 1);
            mrow[p] = hb[(size_t)ij * HLD + (p == lane ? MAXM + 3 : il)];
        }
        warp_allreduce_n<S, RPW>(a);
        double mb[CPL];  // the block's rows share one register column (RPW divides 32)
#pragma unroll
        for (int e = 0; e < CPL; ++e) mb[e] = (e == ((W * RPW) >> 5)) ? 1.0 : 0.0;
        S zl = S(0.0);
#pragma unroll
        for (int e = 0; e < CPL; ++e) zl += z[e] * mb[e];
        // b_j = h_j^* z = a_j / conj(K2_j) + z_j; delta = M b (lane p < RPW forms delta_p)
        S d0 = S(0.0), d1 = S(0.0);
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
            const int ij = W * RPW + j;
            const S bj = a[j] * rkv[j] + shfl_idx(zl, ij & 31);
            const bool use = lane < RPW && j <= lane && ij >= lo && W * RPW + lane <= hi;
            const S mj = use ? mrow[j] : S(0.0);
            if (j & 1) d1 = fma_s(mj, bj, d1);
            else d0 = fma_s(mj, bj, d0);
        }
        const S dp = d0 + d1;
        // z <- z - sum_p delta_p h_p,  h_p[c] = conj(piv_i[c]) / K2_i (c < i), h_p[i] = 1
        S dd[RPW];
#pragma unroll
        for (int p = 0; p < RPW; ++p) dd[p] = shfl_idx(dp, p);
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const int i = W * RPW + p;
            const bool on = i >= lo && i <= hi;
            const S di = on ? dd[p] : S(0.0);
            const S sp = di * conjv(rkv[p]);  // delta_p / K2_i
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const int c = lane + 32 * e;
                z[e] -= (c == i) ? di : sp * conjv(pvr[p][e]);  // (pvr = 0 for c > i)
            }
        }
    }
#pragma unroll
    for (int e = 0; e < CPL; ++e) {
        const int c = lane + 32 * e;
        if (c < m) uu[c] = z[e];
    }
    RQW_T(3100);
}
