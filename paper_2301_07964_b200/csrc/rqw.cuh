// rqw.cuh -- the opposite reflector's RQ for long reflectors (MAXM = 64, 128): Householder RQ of
// the m x m block B(i1:i2,i1:i2), rows bottom-up in xGERQ2 order (readings c3/c4),
// returning only uu = Q~^* e1 = conj(Q~(1,:))^T (the direction of Z_k^j).
//
// Same mathematics as rq_direction (chase.cuh), organised for latency at large m:
//  * warp w owns the RPW = MAXM/NW consecutive rows [w RPW, (w+1) RPW) in registers, TRANSPOSED:
//    lane l holds columns l, l+32, ... (CPL = MAXM/32 of them) of every one of its rows;
//  * stage i (pivot row i, i = m-1 .. 1) is computed by the warp that owns row i: the dot products
//    of its rows with the pivot row and the pivot's tail norm are in-lane partial sums finished by
//    ONE warp reduction (reduce-scatter + broadcast of RPW values), so the RPW stages of a block
//    run inside one warp with no CTA barrier on the chain;
//  * the warps owning rows above apply each published stage to their rows, trailing (they read
//    the pivot row and the two scalars of the stage from shared memory after a flag);
//  * when a warp's own rows come up it has already applied every stage below them.
// Stage i generates H_i = I - tau h h^* with h_c = conj(C[i][c]) / K2 (c < i), h_i = 1,
// tau = K1 |K2|^2 (K2 = alpha - beta, K1 = tau / |K2|^2; real K1 = 1/(s2 + |alpha| nrm)), from
// alpha = conj(C[i][i]) and the tail conj(C[i][0:i)) (oracle_rq_first_row's larfg), and applies it
// to rows 0..i-1 on columns 0..i-1 (column i is dead after stage i).
//
// uu = H_{m-1} ... H_1 (H_0) e1 is formed at the end by warp 0 from the stored pivot rows, block
// by block (a block = the RPW stages of one warp): with a_i = h_i^* z and the block's Gram matrix
// G_ij = h_i^* h_j (j < i, built by the owning warp once its block is done, off the chain),
// d_i = a_i - sum_{j<i} tau_j G_ij d_j and z <- z - sum_j tau_j h_j d_j -- exactly the
// ascending sequence of reflector applications of the block.
//
// Storage (shared): hb (row-major, ld HLD >= MAXM): the pivot row i at hb[i HLD + c], c < i
// (strict lower part), G_ij (j < i, same block) at hb[j HLD + i] (strict upper part), K1 and K2
// of stage i at hb[i HLD + MAXM] and hb[i HLD + MAXM + 1] (HLD >= MAXM + 2); flag: volatile
// stage counter (> m - 1 on entry).  hb may alias the input block (read into registers first).
#pragma once
#include "scalar.cuh"

__device__ __forceinline__ void rqw_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename S, int MAXM, int NW>
struct RQW {
    static_assert(MAXM % 32 == 0 && MAXM % NW == 0, "rqw layout");
    static constexpr int CPL = MAXM / 32;  // columns per lane
    static constexpr int RPW = MAXM / NW;  // rows per warp
    static constexpr int NTHR = NW * 32;
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
    int cnt = N, lvl = 16;
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
        cnt = h;
    }
    (void)cnt;
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

// Called by threads [0, NW*32) of the CTA (all of them together; named barrier 1).  Cb: m x m
// block (col-major, ld LDC); hb/HLD: work storage (see above); uu: output (m entries, written by
// warp 0); the caller synchronises before reading uu.
template <typename S, int MAXM, int NW>
__device__ __forceinline__ void rq_direction_w(int m, const S* Cb, int LDC, S* hb, int HLD,
                                               volatile int* flag, S* uu) {
    using CF = RQW<S, MAXM, NW>;
    constexpr int CPL = CF::CPL, RPW = CF::RPW;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int row0 = w * RPW;
    // ---- rows into registers (transposed: lane l holds columns l + 32 e) ----
    S val[RPW][CPL];
#pragma unroll
    for (int p = 0; p < RPW; ++p)
#pragma unroll
        for (int e = 0; e < CPL; ++e) {
            const int l = row0 + p, c = lane + 32 * e;
            val[p][e] = (l < m && c < m) ? Cb[l + (size_t)c * LDC] : S(0.0);
        }
    rqw_bar(1, CF::NTHR);  // every row is in registers before hb (which may alias Cb) is written
    // stage range owned by this warp: i = ihi .. ilo (descending)
    const int ihi = min(row0 + RPW, m) - 1;
    const int ilo = max(row0, 1);
    // ---- trailing: apply the stages of the rows below (i > ihi), as they are published ----
    for (int i = m - 1; i > ihi; --i) {
        while (*flag > i) {
        }
        __threadfence_block();
        const S* pv = hb + (size_t)i * HLD;
        S pe[CPL];
#pragma unroll
        for (int e = 0; e < CPL; ++e) {
            const int c = lane + 32 * e;
            pe[e] = (c < i) ? pv[c] : S(0.0);
        }
        const S K1 = hb[(size_t)i * HLD + MAXM], K2 = hb[(size_t)i * HLD + MAXM + 1];
        if (is_zero(K1) && is_zero(K2)) continue;  // H_i = I (uniform)
        S g[RPW];
        const int ei = i >> 5, li = i & 31;
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            S a0 = S(0.0);
#pragma unroll
            for (int e = 0; e < CPL; ++e) a0 = fma_s(val[p][e], conjv(pe[e]), a0);
            // + K2 row[i] (the lane holding column i adds it: one reduction for both terms)
            S ri = S(0.0);
#pragma unroll
            for (int e = 0; e < CPL; ++e)
                if (e == ei) ri = val[p][e];
            if (lane == li) a0 += K2 * ri;
            g[p] = a0;
        }
        warp_allreduce_n<S, RPW>(g);
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const S f = K1 * g[p];
#pragma unroll
            for (int e = 0; e < CPL; ++e) val[p][e] -= f * pe[e];  // (pe = 0 for columns >= i)
        }
    }
    // ---- own stages: pivot rows ihi .. ilo, in-warp ----
    // Rows p > pr are dead (their stages are done) and still hold their pivot rows: the same
    // reduction gives the Gram numerators of this block for the reverse pass, off the chain.
    for (int i = ihi; i >= ilo; --i) {
        const int pr = i - row0;
        S pe[CPL];
#pragma unroll
        for (int p = 0; p < RPW; ++p)
            if (p == pr)
#pragma unroll
                for (int e = 0; e < CPL; ++e) pe[e] = val[p][e];
        const int ei = i >> 5, li = i & 31;
        S alpha = S(0.0);
#pragma unroll
        for (int e = 0; e < CPL; ++e)
            if (e == ei) alpha = pe[e];
        alpha = conjv(shfl_idx(alpha, li));
        // the pivot row for the rows above and the reverse pass (columns < i)
        S* pv = hb + (size_t)i * HLD;
#pragma unroll
        for (int e = 0; e < CPL; ++e) {
            const int c = lane + 32 * e;
            if (c < i) pv[c] = pe[e];
            else pe[e] = S(0.0);
        }
        // partial sums: slot pr = tail norm^2; slots p != pr = row_p . conj(pivot) over c < i
        // (p < pr: live rows to update; p > pr: dead pivot rows -> Gram numerators)
        S g[RPW];
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            S a0 = S(0.0);
            if (p == pr) {
                double nn = 0.0;
#pragma unroll
                for (int e = 0; e < CPL; ++e) nn += abs2(pe[e]);
                a0 = S(nn);
            } else {
#pragma unroll
                for (int e = 0; e < CPL; ++e) a0 = fma_s(val[p][e], conjv(pe[e]), a0);
            }
            g[p] = a0;
        }
        warp_allreduce_n<S, RPW>(g);
        S K1, K2;
        double nx = 0.0;
#pragma unroll
        for (int p = 0; p < RPW; ++p)
            if (p == pr) nx = re(g[p]);
        rqw_scalars(alpha, nx, K1, K2);
        if (lane == 0) {
            hb[(size_t)i * HLD + MAXM] = K1;
            hb[(size_t)i * HLD + MAXM + 1] = K2;
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0) *flag = i;
        // the lane holding column i owns row_p[i]: it forms f_p = K1 (g_p + K2 row_p[i]) for the live
        // rows and writes the Gram entries G_{i' i} = h_{i'}^* h_i of the dead rows i' = row0 + p
        // (= (g_p / K2 + piv_i'[i]) / conj(K2_i'), see the header)
        const S r2 = is_zero(K2) ? S(0.0) : recip(K2);
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            S ri = S(0.0);
#pragma unroll
            for (int e = 0; e < CPL; ++e)
                if (e == ei) ri = val[p][e];
            if (p < pr) {
                const S f = shfl_idx(K1 * (g[p] + K2 * ri), li);
#pragma unroll
                for (int e = 0; e < CPL; ++e) val[p][e] -= f * pe[e];
            } else if (p > pr && row0 + p <= ihi && lane == li) {
                const S k2p = hb[(size_t)(row0 + p) * HLD + MAXM + 1];
                S gv = S(0.0);
                if (!is_zero(K2) && !is_zero(k2p)) gv = (g[p] * r2 + ri) * recip(conjv(k2p));
                hb[(size_t)i * HLD + row0 + p] = gv;
            }
        }
    }
    rqw_bar(1, CF::NTHR);  // every stage and Gram entry stored
    if (w != 0) return;
    // ---- reverse pass (warp 0): z = H_{m-1} ... H_1 (H_0) e1, block by block ----
    S z[CPL];
#pragma unroll
    for (int e = 0; e < CPL; ++e) z[e] = S((lane + 32 * e) == 0 ? 1.0 : 0.0);
    if constexpr (sizeof(S) != 8) {
        // complex stage 0: H_0 = I - tau0 e1 e1^*, alpha = conj(R~(0,0)) (row 0 after all stages)
        S a00 = shfl_idx(val[0][0], 0);
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
        // a_i = h_i^* z = sum_{c<i} piv_i[c] z_c / conj(K2_i) + z_i  for the block's RPW stages
        S a[RPW];
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const int i = W * RPW + p;
            S a0 = S(0.0);
            if (i >= lo && i <= hi) {
                const S* pi = hb + (size_t)i * HLD;
#pragma unroll
                for (int e = 0; e < CPL; ++e) {
                    const int c = lane + 32 * e;
                    if (c < i) a0 = fma_s(pi[c], z[e], a0);
                }
            }
            a[p] = a0;
        }
        warp_allreduce_n<S, RPW>(a);
        S zi[RPW];  // z_i of every stage of the block (broadcast from the lane holding it)
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const int i = min(W * RPW + p, MAXM - 1);
            S v = S(0.0);
#pragma unroll
            for (int e = 0; e < CPL; ++e)
                if (e == (i >> 5)) v = z[e];
            zi[p] = shfl_idx(v, i & 31);
        }
        // d_i = a_i - sum_{j<i} tau_j G_ij d_j  (ascending i; tau_j = K1_j |K2_j|^2)
        S d[RPW], td[RPW];
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const int i = W * RPW + p;
            d[p] = S(0.0);
            td[p] = S(0.0);
            if (i < lo || i > hi) continue;
            const S K1 = hb[(size_t)i * HLD + MAXM], K2 = hb[(size_t)i * HLD + MAXM + 1];
            if (is_zero(K2)) continue;
            S di = a[p] * recip(conjv(K2)) + zi[p];
#pragma unroll
            for (int q2 = 0; q2 < p; ++q2) {
                const int j = W * RPW + q2;
                if (j >= lo) di -= td[q2] * hb[(size_t)j * HLD + i];
            }
            d[p] = di;
            td[p] = (K1 * S(abs2(K2))) * di;
        }
        // z <- z - sum_j tau_j d_j h_j,  h_j[c] = conj(piv_j[c]) / K2_j (c < j), h_j[j] = 1
#pragma unroll
        for (int p = 0; p < RPW; ++p) {
            const int i = W * RPW + p;
            if (i < lo || i > hi || is_zero(td[p])) continue;
            const S* pi = hb + (size_t)i * HLD;
            const S s = td[p] * recip(hb[(size_t)i * HLD + MAXM + 1]);
#pragma unroll
            for (int e = 0; e < CPL; ++e) {
                const int c = lane + 32 * e;
                if (c < i) z[e] -= s * conjv(pi[c]);
                else if (c == i) z[e] -= td[p];
            }
        }
    }
#pragma unroll
    for (int e = 0; e < CPL; ++e) {
        const int c = lane + 32 * e;
        if (c < m) uu[c] = z[e];
    }
}
