// chase.cuh -- K1: the generate phase of one group of q sweeps (PAPER.md:1843-1877,
// Alg. 3 "Generate phase of stage two", with the index corrections of DESIGN.md §3 / c8),
// run as a wavefront: CTA t owns sweep j = j1+t; step (j,k) starts once sweep j-1 has
// finished step k+2 (lag 3, SURVEY App. A.4 [V7][V11]), so up to q bulges are in flight.
//
// Per step (j,k), 1-based as in the paper:
//   jb = j + max(0,(k-1)r+1), i1 = j+kr+1, i2 = min(j+(k+1)r,n), i3 = min(j+(k+2)r,n),
//   i4 = j1 + 1 + max(0,(k+j-j1-q+1)r)                                 (corrected, c8)
//   (a) catch-up of Q_k^{j1..j-1} on A(.,jb) and B(.,i1+r-1)  (Alg. 3 lines 9-16), applied in
//       compact-WY form U_k^* x = x - Y T^* Y^* x (three parallel rounds instead of a chain of
//       t reflector applications); sweep j appends column t of window k's T factor (xLARFT)
//   (b) Q_k^j reduces A(i1:i2,jb); B(i1:i2,i1:i2) <- Q^* B           (lines 17-19)
//   (c) Householder RQ of B(i1:i2,i1:i2) (xGERQ2 order, reading c4); the first row of Q~
//       comes out of the [C; P] stacked rows (P accumulates H_{m-1}...H_1 so P e1 = Q~^* e1);
//       Z_k^j = larfg(conj(Q~(1,:))^T)                                 (lines 20-21, c3)
//   (d) A(i4:i3,i1:i2) <- A Z ; B(i4:i2,i1:i2) <- B Z                   (lines 22-23)
// The reflectors (v, tau) of Q_k^j and Z_k^j are stored as records; K2 (accum.cuh) folds them
// into the dense window blocks U_k, V_k for the apply phase.
#pragma once
#include "scalar.cuh"
#include "rqw.cuh"
#include "rqu.cuh"

#ifndef IDX
#define IDX(p, ld, i, j) (p)[((int64_t)(i) - 1) + ((int64_t)(j) - 1) * (int64_t)(ld)]
#endif

template <typename S>
struct ChaseArgs {
    int n, r, qp, j1, K;
    S* A;
    int64_t lda;
    S* B;
    int64_t ldb;
    S* Qr;      // (qp*K) records of (r+1): v of Q_k^j (v[0]=1, m entries), tau at [r]
    S* Zr;      // (qp*K) records of (r+1): v of Z_k^j, sigma at [r]
    S* Tr;      // (qp*K) records of TLD: column t of window k's WY factor T (rows 0..t)
    int TLD;
    S* Mg;        // K blocks of mst: M_t(k) = (Q_k^{j1+t-1})^* ... (Q_k^{j1})^*, the catch-up operator
    int mld;      // of sweep t on window k (row-major, ld mld), updated in place sweep by sweep
    int64_t mst;  // (dense path only: chase_dense_catchup)
    int* prog;  // prog[0..qp): steps completed by each sweep; prog[qp]: ticket;
                // prog[qp+1 .. 2qp+1): far-strip items completed by each helper
    int strip_cap;  // strip rows (A then B) staged in shared memory per step
    int helpers;    // H >= 1: far strips (rows above b0(k-1)) go to H helper CTAs per sweep, which
                    // own interleaved 64-row blocks of the matrix (hprog[t*H + h])
    long long* prof;  // optional: per-CTA cycle counts of the step phases (12 slots)
    int prof_t0;      // >= 0: only sweep prof_t0 of each group records
    int hlag;         // helpers take the band rows above b0(k - hlag): 1, or 0 (see far_strip_helper)
    const unsigned long long* gate;  // input-check verdict (input_rejected)
    // lag checker (HT_LAG_CHECK, debug): global-timer stamps of every sweep step and helper item,
    // [start, end] pairs -- sweeps at trace[(t K + k) 2 + 0/1], helpers after qp K pairs at
    // trace[(qp K + (t H + h) K + k) 2 + 0/1]; checked on the host (ht_stage2.cu, check_lag)
    unsigned long long* trace;
    // RQ update (rqu.cuh, real r in (32, 64]): the hand-over of sweep j to sweep j+1 per window k,
    // R~(2:m,2:m) then (Q~ Z)(2:m,2:m), each row-major with ld MAXM, at Fg + k fst
    double* Fg = nullptr;
    int64_t fst = 0;
    int rqu = 0;        // 0: Householder RQ per step; 1: RQ update in the sweep; 2: direction by a
                        // triangular solve, the RQ update (hand-over) by the sweep's helper h = k mod H
    double* Fb = nullptr;  // rqu 2: the caught-up column b of step (j,k) per k (MAXM each)
    int* Fdone = nullptr;  // rqu 2: per k, j+1 once the hand-over of sweep j's step k is in Fg
    // helper layout (nullptr: `helpers` per sweep): lay[t] = first helper index of sweep t (prefix
    // sums, t <= qp), lay[qp + 1 + ticket] = (t << 8) | role of a CTA ticket (role 0: the sweep)
    const int* lay = nullptr;
    int* Freq = nullptr;   // rqu 2, MAXM 128: per k, j+1 when sweep j's solve failed (direction requested)
    int* Fdirok = nullptr; // ... j+1 once the helper put Q~(1,:) in Fdir
    double* Fdir = nullptr;
    // rqu 2, MAXM 64: the sweep runs the RQ update itself (as after a failed solve) on the steps k
    // with (k num) mod den < num -- a share num/den of the hand-overs moves from the helpers (the
    // critical resource at config 4: a helper's strip item plus its hand-overs outlast a sweep
    // step) to the sweep (HT_RQU_SELF=num/den; 0/1: none)
    int rqu_self_num = 0, rqu_self_den = 1;
};

// shared-memory buffers of the RQ update (chase_kernel carves them; helpers use them too)
struct RQUBufs {
    double *Rs, *Qs, *wpart, *cs1, *cs2, *xs, *v, *z, *uu;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void k1_cp_async(void* s, const void* g, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(g));
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
template <typename S>
__device__ __forceinline__ void k1_ld(S* s, const S* g) { k1_cp_async(s, g, (int)sizeof(S)); }
__device__ __forceinline__ void k1_commit_wait() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ void k1_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void k1_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// Stage flag of the RQ's two warp groups.  The producer publishes after a named barrier that
// orders every producer thread's ring writes before the flag store; shared-memory stores of one
// SM are performed in issue order, so a volatile store suffices (no MEMBAR on the RQ chain).
__device__ __forceinline__ void st_release_cta(volatile int* p, int v) {
    const unsigned a = (unsigned)__cvta_generic_to_shared((const void*)p);
    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(volatile int* p) {
    const unsigned a = (unsigned)__cvta_generic_to_shared((const void*)p);
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Warp-collective Householder generation, reading c1 (xLARFG): x[0..m) -> v (v[0]=1),
// tau, beta real with H^* x = beta e1.  vout may alias x.  All lanes return tau/beta.
template <typename S>
__device__ __forceinline__ void warp_larfg(int m, const S* x, S* vout, S& tau, double& beta) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
    for (int i = 1 + lane; i < m; i += 32) s += abs2(x[i]);
    s = warp_sum(s);
    const S alpha = x[0];
    __syncwarp();
    if (s == 0.0 && im(alpha) == 0.0) {
        tau = S(0.0);
        beta = re(alpha);
        for (int i = 1 + lane; i < m; i += 32) vout[i] = S(0.0);
    } else {
        const double nrm = sqrt(abs2(alpha) + s);
        beta = (re(alpha) >= 0.0) ? -nrm : nrm;
        tau = divr(S(beta) - alpha, beta);
        const S scal = recip(alpha - S(beta));
        for (int i = 1 + lane; i < m; i += 32) vout[i] = x[i] * scal;
    }
    if (lane == 0) vout[0] = S(1.0);
    __syncwarp();
}

// Register form of the same reflector for m <= 32 (lane l holds x[l]; lanes >= m hold 0), with
// the MUFU-seeded rsqrt / reciprocal of the RQ instead of IEEE sqrt and division:
// beta = -sign(re alpha) ||x||, tau = 1 - alpha / beta (beta real), v = x / (alpha - beta).
// Returns v[lane] (v[0] = 1).
__device__ __forceinline__ double fast_recip_s(double d) { return fast_rcp(d); }
__device__ __forceinline__ zc fast_recip_s(zc d) { return conjv(d) * fast_rcp(abs2(d)); }
template <typename S>
__device__ __forceinline__ S larfg_reg(S xv, int m, S& tau, double& beta) {
    const int lane = threadIdx.x & 31;
    const S alpha = shfl_idx(xv, 0);
    double s = (lane >= 1 && lane < m) ? abs2(xv) : 0.0;
    s = warp_sum(s);
    if (s == 0.0 && im(alpha) == 0.0) {
        tau = S(0.0);
        beta = re(alpha);
        return S(lane == 0 ? 1.0 : 0.0);
    }
    const double a2 = abs2(alpha) + s;
    const double rs = fast_rsqrt(a2);
    const bool pos = re(alpha) >= 0.0;
    beta = pos ? -(a2 * rs) : a2 * rs;
    tau = S(1.0) - alpha * (pos ? -rs : rs);
    const S sc = fast_recip_s(alpha - S(beta));
    return lane == 0 ? S(1.0) : xv * sc;
}

// The same for m <= 32 EPL: lane l holds x[l + 32 e]; x and vout in shared memory (vout may alias x).
// (warp_larfg's IEEE sqrt / divisions measured ~4k cycles at m = 64 on the step's chain.)
template <typename S, int EPL>
__device__ __forceinline__ void larfg_regn(int m, const S* x, S* vout, S& tau, double& beta) {
    const int lane = threadIdx.x & 31;
    S xv[EPL];
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int i = lane + 32 * e;
        xv[e] = i < m ? x[i] : S(0.0);
        if (i >= 1) s += abs2(xv[e]);
    }
    s = warp_sum(s);
    const S alpha = shfl_idx(xv[0], 0);
    __syncwarp();
    if (s == 0.0 && im(alpha) == 0.0) {
        tau = S(0.0);
        beta = re(alpha);
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            const int i = lane + 32 * e;
            if (i < m) vout[i] = S(i == 0 ? 1.0 : 0.0);
        }
        __syncwarp();
        return;
    }
    const double a2 = abs2(alpha) + s;
    const double rs = fast_rsqrt(a2);
    const bool pos = re(alpha) >= 0.0;
    beta = pos ? -(a2 * rs) : a2 * rs;
    tau = S(1.0) - alpha * (pos ? -rs : rs);
    const S sc = fast_recip_s(alpha - S(beta));
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int i = lane + 32 * e;
        if (i < m) vout[i] = (i == 0) ? S(1.0) : xv[e] * sc;
    }
    __syncwarp();
}

// RQ thread layout.  Group A (threads [0, NA)) holds the m rows of C, group B (threads
// [NA, 2NA)) the m rows of P; LPR threads per row, each with E columns in REGISTERS, columns
// interleaved (thread part p holds columns LPR*e + p) so that the per-stage skip of the columns
// a stage does not touch (H_i acts on columns 0..i) is warp-uniform, in sub-blocks of SB.
// Group A carries the sequential chain (pivot rows, scalars); group B only consumes each stage's
// pivot row and scalars from a shared-memory ring and trails it (never blocks group A).
// For MAXM > 64 the [C; P] rows do not fit the register file: group B is dropped (NOB) and
// Q~^* e1 = H_{m-1}...H_0 e1 is formed afterwards by one warp from the stored reflectors.
template <typename S, int MAXM>
struct RQCfg {
#ifndef HT_RQ_LPR64
#define HT_RQ_LPR64 2
#endif
    static constexpr int LPR = (MAXM == 64) ? HT_RQ_LPR64 : ((MAXM >= 16) ? 2 : 1);
    static constexpr int E = MAXM / LPR;
    static constexpr int SB = 8;
    static constexpr int NSB = (E + SB - 1) / SB;
    static constexpr int ROWT = MAXM * LPR;
    static constexpr int NA = (ROWT < 32) ? 32 : ROWT;
#ifndef HT_RQ_NOB_ABOVE
#define HT_RQ_NOB_ABOVE 64
#endif
    static constexpr bool NOB = MAXM > HT_RQ_NOB_ABOVE;
    static constexpr int NTHR = NOB ? NA : 2 * NA;
    static constexpr int PLD = LPR * NSB * SB + 4;  // ring slot: pivot row (de-interleaved) + K1, K2
};

template <typename S, int LPR>
__device__ __forceinline__ S lpr_sum(S v) {
#pragma unroll
    for (int o = 1; o < LPR; o <<= 1) v += shfl_xor(v, o);
    return v;
}

#ifndef HT_RQ_ATTR
#define HT_RQ_ATTR __forceinline__
#endif
// Householder RQ (readings c3/c4), rows bottom-up (xGERQ2 order) on C = B(i1:i2,i1:i2) (m x m,
// col-major, ld LDC) with P = I alongside.  Stage i (i = m-1 .. 1, plus 0 for complex) generates
// H_i from row i of C (alpha = conj(C[i][i]), tail conj(C[i][0..i)): oracle_rq_first_row's larfg)
// and right-multiplies C rows 0..i-1 and all P rows by H_i on columns 0..i.  Then
// P = H_{m-1}...H_0 = Q~^*, and uu = P e1 = Q~^* e1 = conj(Q~(1,:))^T.
// Per row: g = sum_{c<i} row[c] conj(C[i][c]), ri = row[i];  row[c] -= f C[i][c] (c < i) with
// f = K1 (g + K2 ri), K1 = tau |1/(alpha-beta)|^2, K2 = alpha - beta (real: K1 = 1/(s + |alpha| nrm),
// s = |alpha|^2 + |tail|^2).  Column i is dead after stage i (later stages act on columns < i,
// the output is column 0), so it is not updated.  ring: m slots of PLD; flag: volatile counter.
template <typename S, int MAXM>
__device__ HT_RQ_ATTR void rq_direction(int m, const S* Cb, int LDC, S* ring, volatile int* flag, S* uu) {
    using CF = RQCfg<S, MAXM>;
    constexpr int LPR = CF::LPR, E = CF::E, SB = CF::SB, NSB = CF::NSB, NA = CF::NA, PLD = CF::PLD;
    constexpr int EP = NSB * SB;  // padded elements per thread
    const int tid = threadIdx.x;
    const bool grpB = tid >= NA;
    const int gt = grpB ? tid - NA : tid;
    const int l = gt / LPR, part = gt % LPR;
    const bool live = gt < CF::ROWT && l < m;
    S row[EP];
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        const int c = LPR * e + part;
        S v = S(0.0);
        if (live && e < E && c < m) v = grpB ? S(l == c ? 1.0 : 0.0) : Cb[l + c * LDC];
        row[e] = v;
    }
    auto syncA = [&]() {
        if (NA <= 32) __syncwarp();
        else named_bar(1, NA);
    };
    auto write_pivot = [&](int slot, int upto) {  // this thread's chunk of its row into ring slot
        S* dst = ring + (size_t)slot * PLD + part * EP;
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb)
            if (sb * SB * LPR < upto)
#pragma unroll
                for (int e = 0; e < SB; ++e) dst[sb * SB + e] = row[sb * SB + e];
    };
    // per-stage local work: g, nx (partial over my columns < i), ri
    constexpr bool NOB = CF::NOB;
    S bk[NOB ? 1 : EP];
    auto dots = [&](const S* pv, int i, S& g, double& nx, S& ri) {
        const int eth = (i - part + LPR - 1) / LPR;  // my elements e < eth have column < i
        const int sbi = eth / SB;
        double n0 = 0.0, n1 = 0.0;
        S g0 = S(0.0), g1 = S(0.0);
        ri = S(0.0);
        const int ei = (i % LPR == part) ? i / LPR : -1;
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb) {
            if (sb * SB * LPR <= i) {  // uniform: the block holds columns <= i for some part
#pragma unroll
                for (int e = 0; e < SB; ++e) {
                    const int ee = sb * SB + e;
                    const S b = (ee < eth) ? pv[part * EP + ee] : S(0.0);
                    if constexpr (!NOB) bk[ee] = b;
                    if (e & 1) {
                        n1 += abs2(b);
                        g1 = fma_s(row[ee], conjv(b), g1);
                    } else {
                        n0 += abs2(b);
                        g0 = fma_s(row[ee], conjv(b), g0);
                    }
                    if (ee == ei) ri = row[ee];
                }
            }
        }
        (void)sbi;
        g = g0 + g1;
        nx = n0 + n1;
    };
    auto update = [&](const S* pv, int i, S f) {  // bk (zero for columns >= i) from dots()
        const int eth = (i - part + LPR - 1) / LPR;
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb) {
            if (sb * SB * LPR <= i) {
#pragma unroll
                for (int e = 0; e < SB; ++e) {
                    const int ee = sb * SB + e;
                    if constexpr (NOB) {
                        if (ee < eth) row[ee] -= f * pv[part * EP + ee];
                    } else {
                        row[ee] -= f * bk[ee];
                    }
                }
            }
        }
    };
    const int ilast = (sizeof(S) == 8) ? 1 : 0;
    if (!grpB) {
        // ---------------- group A: C rows, the sequential chain ----------------
        syncA();  // every row is in registers before the ring (which may overlay Cb) is written
        if (live && l == m - 1) write_pivot(m - 1, m);
        syncA();
        for (int i = m - 1; i >= 1; --i) {
            const S* pv = ring + (size_t)i * PLD;
            const S alpha = conjv(pv[(i % LPR) * EP + i / LPR]);
            S g, ri;
            double nx;
            dots(pv, i, g, nx, ri);
            nx = lpr_sum<double, LPR>(nx);
            g = lpr_sum<S, LPR>(g);
            ri = lpr_sum<S, LPR>(ri);
            S K1 = S(0.0), K2 = S(0.0);
            if (!(nx == 0.0 && im(alpha) == 0.0)) {  // uniform
                const double s2 = abs2(alpha) + nx;
                const double y = fast_rsqrt(s2);
                const double nrm = s2 * y;
                const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
                K2 = alpha - S(beta);
                if constexpr (sizeof(S) == 8) {
                    K1 = S(fast_rcp(s2 + fabs(re(alpha)) * nrm));
                } else {
                    const S tau = (S(beta) - alpha) * ((re(alpha) >= 0.0) ? -y : y);  // 1/beta
                    K1 = tau * fast_rcp(abs2(K2));
                }
            }
            S f = K1 * (g + K2 * ri);
            if (!(live && l < i)) f = S(0.0);
            update(pv, i, f);
            if (gt == 0) {
                ring[(size_t)i * PLD + LPR * EP] = K1;
                ring[(size_t)i * PLD + LPR * EP + 1] = K2;
            }
            if (live && l == i - 1) write_pivot(i - 1, i);
            syncA();
            if (!NOB && gt == 0) st_release_cta(flag, i);  // stage i (pivot, K1, K2) complete
        }
        if constexpr (sizeof(S) != 8) {
            // stage 0: H_0 = I - tau e1 e1^* makes R~(0,0) real; P rows get row[0] *= (1 - tau)
            const S alpha = conjv(ring[0 * PLD]);
            S tau = S(0.0);
            if (im(alpha) != 0.0) {
                const double nrm = sqrt(abs2(alpha));
                const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
                tau = (S(beta) - alpha) * (1.0 / beta);
            }
            if (gt == 0) {
                ring[LPR * EP] = tau;
                if (!NOB) st_release_cta(flag, 0);
            }
        }
        if constexpr (NOB) {
            // uu = H_{m-1} ... H_1 H_0 e1 from the stored reflectors (one warp; H_0 first).
            // H_i = I - tau h h^*, h_c = conj(C[i][c]) / K2 (c < i), h_i = 1, tau = K1 |K2|^2.
            syncA();
            if (gt < 32) {
                const int lane = gt;
                constexpr int YL = (MAXM + 31) / 32;
                S y[YL];
#pragma unroll
                for (int s2 = 0; s2 < YL; ++s2) y[s2] = S((lane + 32 * s2) == 0 ? 1.0 : 0.0);
                if constexpr (sizeof(S) != 8) {
                    const S tau0 = ring[LPR * EP];
                    if (lane == 0) y[0] -= tau0 * y[0];
                }
                for (int i = 1; i <= m - 1; ++i) {
                    const S* pv = ring + (size_t)i * PLD;
                    const S K1 = pv[LPR * EP], K2 = pv[LPR * EP + 1];
                    if (is_zero(K1)) continue;  // uniform
                    S sacc = S(0.0);
                    S yi = S(0.0);
#pragma unroll
                    for (int s2 = 0; s2 < YL; ++s2) {
                        const int c = lane + 32 * s2;
                        if (c < i) sacc = fma_s(pv[(c % LPR) * EP + c / LPR], y[s2], sacc);
                        if (c == i) yi = y[s2];
                    }
                    sacc = warp_sum(sacc);
                    yi = warp_sum(yi);
                    const S inv = recip(K2);
                    const S d = sacc * conjv(inv) + yi;
                    const S tau = K1 * abs2(K2);
                    const S td = tau * d;
#pragma unroll
                    for (int s2 = 0; s2 < YL; ++s2) {
                        const int c = lane + 32 * s2;
                        if (c < i) y[s2] -= td * inv * conjv(pv[(c % LPR) * EP + c / LPR]);
                        else if (c == i) y[s2] -= td;
                    }
                }
#pragma unroll
                for (int s2 = 0; s2 < YL; ++s2)
                    if (lane + 32 * s2 < m) uu[lane + 32 * s2] = y[s2];
            }
        }
    } else {
        // ---------------- group B: P rows, trailing consumer ----------------
        for (int i = m - 1; i >= ilast; --i) {
            while (ld_acquire_cta(flag) > i) {
            }
            const S* pv = ring + (size_t)i * PLD;
            const S K1 = pv[LPR * EP], K2 = pv[LPR * EP + 1];
            if (i == 0) {  // complex stage 0 (see group A)
                if (live && part == 0) row[0] -= K1 * row[0];
                continue;
            }
            S g, ri;
            double nx;
            dots(pv, i, g, nx, ri);
            g = lpr_sum<S, LPR>(g);
            ri = lpr_sum<S, LPR>(ri);
            S f = K1 * (g + K2 * ri);
            if (!live) f = S(0.0);
            update(pv, i, f);
        }
        if (live && part == 0) uu[l] = row[0];
    }
}

// Fully unrolled variant for MAXM <= 32 (the common r <= 32 case): one thread per row (group A =
// warp 0 holds C, group B = warp 1 holds P), the stage index i is a compile-time constant in
// every unrolled copy, so column masks and the pick of row[i] cost nothing; scalars use the
// MUFU-seeded rsqrt / reciprocal (fast_rsqrt, fast_rcp).  Same mathematics as rq_direction.
template <typename S, int MAXM>
__device__ __forceinline__ void rq_direction_u(int m, const S* Cb, int LDC, S* ring, volatile int* flag, S* uu) {
    constexpr int PL = MAXM + 4;
    const int tid = threadIdx.x;
    const bool grpB = tid >= 32;
    const int l = tid & 31;
    const bool live = l < m && l < MAXM;
    S row[MAXM];
#pragma unroll
    for (int c = 0; c < MAXM; ++c) {
        S v = S(0.0);
        if (live && c < m) v = grpB ? S(l == c ? 1.0 : 0.0) : Cb[l + c * LDC];
        row[c] = v;
    }
    if (!grpB) {
        if (live && l == m - 1) {
#pragma unroll
            for (int c = 0; c < MAXM; ++c) ring[(size_t)(m - 1) * PL + c] = row[c];
        }
        __syncwarp();
#pragma unroll
        for (int i = MAXM - 1; i >= 1; --i) {
            if (i <= m - 1) {  // uniform
                const S* pv = ring + (size_t)i * PL;
                const S alpha = conjv(pv[i]);
                double n4[4] = {0.0, 0.0, 0.0, 0.0};
                S g4[4] = {S(0.0), S(0.0), S(0.0), S(0.0)};
#pragma unroll
                for (int c = 0; c < i; ++c) {
                    const S b = pv[c];
                    n4[c & 3] += abs2(b);
                    g4[c & 3] = fma_s(row[c], conjv(b), g4[c & 3]);
                }
                const double nx = (n4[0] + n4[1]) + (n4[2] + n4[3]);
                const S g = (g4[0] + g4[1]) + (g4[2] + g4[3]);
                S K1 = S(0.0), K2 = S(0.0);
                if (!(nx == 0.0 && im(alpha) == 0.0)) {
                    const double s2 = abs2(alpha) + nx;
                    const double y = fast_rsqrt(s2);
                    const double nrm = s2 * y;
                    const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
                    K2 = alpha - S(beta);
                    if constexpr (sizeof(S) == 8) {
                        K1 = S(fast_rcp(s2 + fabs(re(alpha)) * nrm));
                    } else {
                        const S tau = (S(beta) - alpha) * ((re(alpha) >= 0.0) ? -y : y);  // 1/beta
                        K1 = tau * fast_rcp(abs2(K2));
                    }
                }
                S f = K1 * (g + K2 * row[i]);
                if (!(live && l < i)) f = S(0.0);
#pragma unroll
                for (int c = 0; c < i; ++c) row[c] -= f * pv[c];
                if (l == 0) {
                    ring[(size_t)i * PL + MAXM] = K1;
                    ring[(size_t)i * PL + MAXM + 1] = K2;
                }
                if (live && l == i - 1) {
#pragma unroll
                    for (int c = 0; c < i; ++c) ring[(size_t)(i - 1) * PL + c] = row[c];
                }
                __syncwarp();
                if (l == 0) st_release_cta(flag, i);
            }
        }
        if constexpr (sizeof(S) != 8) {
            const S alpha = conjv(ring[0]);
            S tau = S(0.0);
            if (im(alpha) != 0.0) {
                const double nrm = sqrt(abs2(alpha));
                const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
                tau = (S(beta) - alpha) * (1.0 / beta);
            }
            if (l == 0) {
                ring[MAXM] = tau;
                st_release_cta(flag, 0);
            }
        }
    } else {
        constexpr int ILAST = (sizeof(S) == 8) ? 1 : 0;
#pragma unroll
        for (int i = MAXM - 1; i >= ILAST; --i) {
            if (i <= m - 1) {
                while (ld_acquire_cta(flag) > i) {
                }
                const S* pv = ring + (size_t)i * PL;
                const S K1 = pv[MAXM];
                if (i == 0) {
                    if (live) row[0] -= K1 * row[0];
                } else {
                    const S K2 = pv[MAXM + 1];
                    S g4[4] = {S(0.0), S(0.0), S(0.0), S(0.0)};
#pragma unroll
                    for (int c = 0; c < i; ++c) g4[c & 3] = fma_s(row[c], conjv(pv[c]), g4[c & 3]);
                    const S g = (g4[0] + g4[1]) + (g4[2] + g4[3]);
                    S f = K1 * (g + K2 * row[i]);
                    if (!live) f = S(0.0);
#pragma unroll
                    for (int c = 0; c < i; ++c) row[c] -= f * pv[c];
                }
            }
        }
        if (live) uu[l] = row[0];
    }
}

template <typename S, int MAXM>
__host__ __device__ constexpr bool rq_unrolled() { return MAXM * (int)sizeof(S) <= 256; }  // real <= 32, complex <= 16
template <typename S, int MAXM>
__host__ __device__ constexpr bool rq_warp_rows();
template <typename S, int MAXM>
__host__ __device__ constexpr int rq_nthr() {
    return rq_unrolled<S, MAXM>() ? 64 : (rq_warp_rows<S, MAXM>() ? 256 : RQCfg<S, MAXM>::NTHR);
}

// real 64 < m <= 128: the warp-row RQ of rqw.cuh (8 warps; the ring is its work storage, ld 132).
// Measured per RQ of a 128 x 128 block: 313k cycles alone / 444k inside the chase kernel against
// ~1M for rq_direction; at m = 64 (90k alone) it lost inside the chase kernel (103k RQ, slower
// other phases: register pressure) to rq_direction (~100k), which therefore stays for r <= 64.
template <typename S, int MAXM>
__host__ __device__ constexpr bool rq_warp_rows() {
#ifdef HT_RQW_OFF
    return false;
#else
#ifndef HT_RQW_MIN
#define HT_RQW_MIN 128
#endif
    return sizeof(S) == 8 && MAXM >= HT_RQW_MIN;
#endif
}

template <typename S, int MAXM>
__device__ __forceinline__ void rq_dir(int m, const S* Cb, int LDC, S* ring, volatile int* flag, S* uu,
                                       int ring_ld = 0, uint64_t* bars = nullptr, int par = 0) {
    if constexpr (rq_unrolled<S, MAXM>()) rq_direction_u<S, MAXM>(m, Cb, LDC, ring, flag, uu);
    else if constexpr (rq_warp_rows<S, MAXM>()) rq_direction_w<S, MAXM, 8>(m, Cb, LDC, ring, ring_ld, bars, par, uu);
    else rq_direction<S, MAXM>(m, Cb, LDC, ring, flag, uu);
}

// RQ ring slot length for the reflector length r (RQCfg<S,MAXM>::PLD of the MAXM that r uses;
// >= r + 4 also covers the unrolled variant's MAXM + 4)
__host__ __device__ inline int ring_pld(int r) { return r <= 32 ? r + 20 : (r <= 64 ? 68 : 132); }

// Dense catch-up operator (real r <= 32, complex r <= 16: the unrolled RQ leaves 6 warps idle):
// sweep t keeps M_t(k) (L x L) instead of records + WY factor; the idle warps form
// M_{t+1}(k) = (Q_k^j)^* M_t(k) during the RQ and store it for sweep t+1.
template <typename S>
__host__ __device__ constexpr bool chase_dense_catchup(int r) {
    return r <= 64 && r * (int)sizeof(S) <= 256;
}

// K1's RQ-update path (rqu.cuh): real fp64, 32 < r <= 64 (MAXM = 64)
template <typename S, int MAXM>
__host__ __device__ constexpr bool rqu_supported() { return sizeof(S) == 8 && (MAXM == 64 || MAXM == 128); }
template <typename S>
__host__ __device__ inline bool rqu_supported_r(int r) { return sizeof(S) == 8 && r > 32 && r <= 128; }
constexpr int CHASE_NT_RQU = 256;

template <typename S>
__host__ __device__ inline size_t chase_smem_elems(int r, int qp, int strip_cap, bool rqu = false) {
    const int w = qp + r - 1;
    const size_t XL = (size_t)(w + r + 8);
    const bool overlay = r > 64;         // the RQ ring (r slots of 132 for MAXM = 128) overlays the B block
    return 3 * XL +                      // x (2 buffers), y
           (overlay ? (size_t)r * 132 : (size_t)r * (r + 1)) +  // B block (| RQ ring)
           3 * (size_t)(r + 8) +         // vq, vz, uu
           (overlay ? 0 : (size_t)r * ring_pld(r)) +  // RQ ring (pivot rows + scalars per stage)
           16 +                          // scalars
           (size_t)qp * (r + 1) +        // catch-up records (Y)
           (size_t)qp * (qp + 1) +       // T factor of window k
           5 * (size_t)(qp + 8) +        // WY temporaries
           (overlay ? 0 : XL + (size_t)r * (r + 1) + (size_t)qp * (r + 1) + (size_t)qp * (qp + 1)) +  // prefetch set
           (chase_dense_catchup<S>(r) ? 2 * (size_t)w * (w | 1) + 2 * (size_t)(w + 1) : 0) +  // M_t, M_t(k+1), tmp
           (rqu ? (r <= 64 ? RQUCfg<CHASE_NT_RQU, 64>::extra : RQUCfg<CHASE_NT_RQU, 128>::extra) : 0) +  // RQ update
           (size_t)strip_cap * (r + 1);  // staged strip rows
}

// Far-strip helper of sweep t (one CTA per sweep): applies Z_k^j to the generate band's rows
// above b0(k-1) = j1+(k-1)r+1 -- A rows [i4, b0(k-1)) and B rows [i4, b0(k-1)) of columns
// i1..i2 -- which no step of the group reads before sweep j+1 reaches window k-1.  Order
// (the same per-row reflector order as Alg. 3): item (t,k) after sweep t's step k (its Z record)
// and after helper t-1's item k+1 (lag as the sweeps).  Sweep t+1 waits for helper t before its
// step k-1 (see chase_kernel).
// The helpers take the band rows above b0(k - hlag) (ChaseArgs::hlag).  Lag 0 also gives them
// the rows [b0(k-1), b0(k)): sweep j+1 first touches those rows of window k's columns at its
// step k-1 (one shared column: the last of its B block and its y column) after waiting for
// helper j's items <= k -- so with lag 0 the y column is loaded at the step start instead of
// being prefetched during step k-2 (the B block's last column is patched from the caught-up y
// anyway); sweep j itself never reads those rows again.
template <typename S, int NT, int MAXM, bool RQK>
__device__ __forceinline__ void far_strip_helper(const ChaseArgs<S>& a, int t, int h, S* sm, const RQUBufs& rb) {
    // this sweep's helpers: H of them at hprog[hb ..]; the previous sweep's: Hp at hprog[hbp ..]
    const int hb = a.lay ? __ldg(a.lay + t) : t * a.helpers;
    const int H = a.lay ? __ldg(a.lay + t + 1) - hb : a.helpers;
    const int hbp = t > 0 ? (a.lay ? __ldg(a.lay + t - 1) : (t - 1) * a.helpers) : 0;
    const int Hp = t > 0 ? hb - hbp : 0;
    constexpr int RB = 64;  // row block: helper h owns blocks h, h+H, ... (relative to j1)
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K;
    const int j = j1 + t;
    const int kcount = min(K, 2 + (n - j - 1) / r);
    const int kprev = (t > 0) ? min(K, 2 + (n - j) / r) : 0;
    int* hprog = a.prog + qp + 1;
    const int tid = threadIdx.x;
    S* zv = sm;
    constexpr int SPR = (MAXM * (int)sizeof(S) > 256) ? MAXM * (int)sizeof(S) / 256 : 1;
    constexpr int CPR = MAXM / SPR;
    const int part = tid % SPR, c0 = part * CPR;
    long long hw = 0, hx = 0, tc = clock64();  // profile: cycles waiting / working (helper 0)
    // rqu 2 (rqu.cuh): the RQ update of step (j,k) and its hand-over to sweep j+1 (helper k mod H).
    // MAXM 64: R0 and Q0 in their own buffers, Q rotated concurrently with the chain.  MAXM 128: R0
    // in the B block's buffer, R~ handed over first, then Q0 rotated in the same buffer; a sweep whose
    // solve failed requests the direction Q~(1,:) early (Freq) and waits for it (Fdirok).
    constexpr bool RQH = RQK && rqu_supported<S, MAXM>();
    constexpr bool RQU64 = RQH && MAXM == 64, RQU128 = RQH && MAXM == 128;
    __shared__ int hreq;
    int early_k = -1;  // step whose Q~ is already in shared memory (early request)
    auto fwork = [&](int k, int stage) {  // stage 0: all; 1: up to Q~ (early); 2: hand-over of W only
        if constexpr (RQH) {
            constexpr int RLD = RQUCfg<NT, MAXM>::RLD;
            const int i1 = j + k * r + 1, m = min(j + (k + 1) * r, n) - i1 + 1;
            const bool hasB = i1 + r - 1 <= n;
            const int f = hasB ? m - 1 : m;
            double* FR = a.Fg + (int64_t)k * a.fst;
            double* FW = FR + MAXM * MAXM;
            const double* qrec = reinterpret_cast<const double*>(a.Qr + ((int64_t)t * K + k) * (r + 1));
            const double* zrec = reinterpret_cast<const double*>(a.Zr + ((int64_t)t * K + k) * (r + 1));
            if (stage != 2) {
                if constexpr (RQU64) rqu_load_block<NT, MAXM>(rb.Qs, FW, f, false);
                rqu_load_block<NT, MAXM>(rb.Rs, FR, f, true);
                if (hasB)
                    for (int i = tid; i < m; i += NT) {
                        rb.Rs[i * RLD + (m - 1)] = ldcg(a.Fb + (int64_t)k * MAXM + i);
                        if constexpr (RQU64) {
                            rb.Qs[(m - 1) * RLD + i] = (i == m - 1) ? 1.0 : 0.0;
                            rb.Qs[i * RLD + (m - 1)] = (i == m - 1) ? 1.0 : 0.0;
                        }
                    }
                for (int c = tid; c < m; c += NT) rb.v[c] = ldcg(qrec + c);
                const double tau = ldcg(qrec + r);
                __syncthreads();
                rqu_direction<NT, MAXM>(m, rb.v, tau, rb.Rs, rb.Qs, rb.wpart, rb.cs1, rb.cs2, rb.uu);
                if constexpr (RQU128) {  // R~ out, then Q0 into the same buffer
                    rqu_handoff_R<NT, MAXM>(m, rb.Rs, FR);
                    __syncthreads();
                    rqu_load_block<NT, MAXM>(rb.Rs, FW, f, false);
                    if (hasB)
                        for (int i = tid; i < m; i += NT) {
                            rb.Rs[(m - 1) * RLD + i] = (i == m - 1) ? 1.0 : 0.0;
                            rb.Rs[i * RLD + (m - 1)] = (i == m - 1) ? 1.0 : 0.0;
                        }
                    __syncthreads();
                    rqu_q_apply<NT, MAXM>(m, rb.Rs, rb.cs1, rb.cs2, rb.uu);
                    for (int i = tid; i < MAXM; i += NT) rb.cs2[2 * i] = RQU_SENTINEL;
                    if (stage == 1) {  // the direction for the waiting sweep
                        for (int c = tid; c < m; c += NT) a.Fdir[(int64_t)k * MAXM + c] = rb.uu[c];
                        __syncthreads();
                        if (tid == 0) {
                            __threadfence();
                            st_release(&a.Fdirok[k], j + 1);
                        }
                        return;
                    }
                }
            }
            for (int c = tid; c < m; c += NT) rb.z[c] = ldcg(zrec + c);
            const double sig = ldcg(zrec + r);
            __syncthreads();
            if constexpr (RQU64) rqu_handoff<NT, MAXM>(m, rb.Rs, rb.Qs, rb.z, sig, FR, FW);
            else rqu_handoff_W<NT, MAXM>(m, rb.Rs, rb.z, sig, FW);
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                st_release(&a.Fdone[k], j + 1);
            }
        }
    };
    for (int k = 0; k < kcount; ++k) {
        if constexpr (RQU128) {
            // the designated helper also answers an early request of the sweep (its solve failed)
            if (a.rqu == 2 && k % H == h) {
                if (tid == 0) {
                    int req = 0;
                    while (ld_relaxed(&a.prog[t]) < k + 1)
                        if (ld_relaxed(&a.Freq[k]) >= j + 1) {
                            req = 1;
                            break;
                        }
                    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                    hreq = req;
                }
                __syncthreads();
                if (hreq) {
                    fwork(k, 1);
                    early_k = k;
                }
            }
        }
        if (tid == 0) {
            if (ld_acquire(&a.prog[t]) < k + 1)
                while (ld_relaxed(&a.prog[t]) < k + 1) {
                }
            if (t > 0) {  // every helper of sweep t-1 through item k+1 (their row blocks may differ)
                const int need = min(k + 2, kprev);
                for (int hh = 0; hh < Hp; ++hh)
                    while (ld_relaxed(&hprog[hbp + hh]) < need) {
                    }
            }
            (void)ld_acquire(&a.prog[t]);
            asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
            if (a.trace) a.trace[((int64_t)qp * K + ((int64_t)hb + h) * K + k) * 2] = gtimer();
        }
        __syncthreads();
        if (a.prof && tid == 0) {
            (void)*(volatile S*)sm;
            const long long now = clock64();
            hw += now - tc;
            tc = now;
        }
        const int i1 = j + k * r + 1;
        const int i2 = min(j + (k + 1) * r, n);
        const int i3 = min(j + (k + 2) * r, n);
        const int i4 = j1 + 1 + max(0, (k + t - qp + 1) * r);
        const int m = i2 - i1 + 1;
        const int cF = j1 + (k - a.hlag) * r + 1;  // rows above b0(k - lag) (see above)
        const int nAf = max(0, min(cF, i3 + 1) - i4), nBf = max(0, min(cF, i2 + 1) - i4);
        if (m >= 2 && nAf + nBf > 0) {
            const S* rec = a.Zr + ((int64_t)t * K + k) * (r + 1);
            for (int c = tid; c < MAXM; c += NT) zv[c] = (c < m) ? ldcg(rec + c) : S(0.0);  // (zero pad)
            if (tid == 0) zv[MAXM] = ldcg(rec + r);
            __syncthreads();
            const S sig = zv[MAXM];
            if (!is_zero(sig)) {
                // my row blocks intersected with the far rows [i4, i4 + nAf) (A) and [i4, i4 + nBf) (B);
                // a block has at most 2 RB = NT / SPR rows: one row per thread.  Two blocks in flight
                // (ping-pong registers): the next block's loads are issued before this block's dot.
                const int nfar = max(nAf, nBf);
                const int blk0 = (i4 - j1) / RB, blk1 = (i4 + nfar - 1 - j1) / RB;
                constexpr int RPT = (2 * RB + NT / SPR - 1) / (NT / SPR);  // rows per thread and block
                const int bfirst = blk0 + ((h - blk0 % H) + H) % H;
                const int nunits_ = bfirst <= blk1 ? ((blk1 - bfirst) / H + 1) * RPT : 0;
                // unit u: block bfirst + (u / RPT) H, row tid / SPR + (u % RPT) NT / SPR of it
                auto rowp = [&](int u, int64_t& ld) -> S* {  // my row of unit u (nullptr: none)
                    const int blk = bfirst + (u / RPT) * H;
                    const int eb = tid / SPR + (u % RPT) * (NT / SPR);
                    const int rlo = max(i4, j1 + blk * RB), rhi = min(i4 + nfar, j1 + (blk + 1) * RB);
                    const int nrA = max(0, min(rhi, i4 + nAf) - rlo), nrB = max(0, min(rhi, i4 + nBf) - rlo);
                    if (u >= nunits_ || blk > blk1 || eb >= nrA + nrB) return nullptr;
                    const bool isA = eb < nrA;
                    ld = isA ? a.lda : a.ldb;
                    return isA ? &IDX(a.A, a.lda, rlo + eb, i1) : &IDX(a.B, a.ldb, rlo + (eb - nrA), i1);
                };
                auto load = [&](const S* gp, int64_t ld, S* v) {
                    // all loads first: an FMA waiting on its load would hold back the next load's
                    // issue (in-order issue), one memory latency per element
                    if (gp) {
#pragma unroll
                        for (int c = 0; c < CPR; ++c) v[c] = (c0 + c < m) ? ldcg(gp + (c0 + c) * ld) : S(0.0);
                    }
                };
                auto finish = [&](S* gp, int64_t ld, const S* v) {  // (all threads: the shuffles)
                    S s0 = S(0.0), s1 = S(0.0);
                    if (gp) {
#pragma unroll
                        for (int c = 0; c < CPR; ++c) {
                            if (c & 1) s1 = fma_s(v[c], zv[c0 + c], s1);
                            else s0 = fma_s(v[c], zv[c0 + c], s0);
                        }
                    }
                    S sdot = s0 + s1;
                    if constexpr (SPR > 1) {
#pragma unroll
                        for (int o = 1; o < SPR; o <<= 1) sdot += shfl_xor(sdot, o);
                    }
                    if (gp) {
                        const S sv = sdot * sig;
#pragma unroll
                        for (int c = 0; c < CPR; ++c)
                            if (c0 + c < m) gp[(c0 + c) * ld] = v[c] - sv * conjv(zv[c0 + c]);
                    }
                };
                const int nunits = nunits_;
                S va[CPR];
                int64_t lda_ = 0, ldb_ = 0;
                if constexpr (sizeof(S) > 8) {  // complex: one row in flight (two spilled registers)
                    for (int u = 0; u < nunits; ++u) {
                        S* pa = rowp(u, lda_);
                        load(pa, lda_, va);
                        finish(pa, lda_, va);
                    }
                } else {
                S vb[CPR];
                S* pa = rowp(0, lda_);
                if (nunits > 0) load(pa, lda_, va);
                for (int u = 0; u < nunits; u += 2) {
                    S* pb = rowp(u + 1, ldb_);
                    if (u + 1 < nunits) load(pb, ldb_, vb);
                    finish(pa, lda_, va);
                    if (u + 1 >= nunits) break;
                    pa = rowp(u + 2, lda_);
                    if (u + 2 < nunits) load(pa, lda_, va);
                    finish(pb, ldb_, vb);
                }
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (a.trace) a.trace[((int64_t)qp * K + ((int64_t)hb + h) * K + k) * 2 + 1] = gtimer();
            st_release(&hprog[hb + h], k + 1);
        }
        if constexpr (RQH) {
            // rqu 2: the RQ update of step (j,k) and its hand-over (unless the sweep did it: MAXM 64)
            const int jb = j + max(0, (k - 1) * r + 1);
            if (a.rqu == 2 && k % H == h && m >= 2 && jb <= n && (RQU128 || ld_acquire(&a.Fdone[k]) < j + 1))
                fwork(k, early_k == k ? 2 : 0);
        }
        if (a.prof && tid == 0) {
            const long long now = clock64();
            hx += now - tc;
            tc = now;
        }
    }
    if (a.prof && tid == 0 && h == 0 && (a.prof_t0 < 0 || t == a.prof_t0)) {
        atomicAdd((unsigned long long*)&a.prof[14], (unsigned long long)hw);
        atomicAdd((unsigned long long*)&a.prof[15], (unsigned long long)hx);
    }
}

// RQK: the RQ-update instantiation (rqu.cuh; launched with a.rqu != 0) -- a separate kernel, so that
// neither path's register allocation carries the other's (the warp-row RQ of r > 64 needs 255)
template <typename S, int NT, int MAXM, bool RQK = false>
__global__ void __launch_bounds__(NT, 1) chase_kernel(ChaseArgs<S> a) {
    if (input_rejected(a.gate)) return;
    extern __shared__ __align__(16) unsigned char smraw[];
    S* sm = reinterpret_cast<S*>(smraw);
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K;
    const int w = qp + r - 1;
    const int SLD = r + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    const int XL = w + r + 8;
    const int TL = qp + 1;
    // column jb of this step / of the next step: sm + cur * XL (pointer arithmetic on the shared
    // base, not a pointer table, so accesses stay LDS/STS instead of generic loads)
    S* ys0 = sm + 2 * XL;
    constexpr bool OVERLAY = MAXM > 64;  // RQ ring overlays Cb (the block goes to HBM after Q^*)
    constexpr bool PF = !OVERLAY;        // next step's B block / records / T / y prefetched during the RQ
    S* Cb0 = ys0 + XL;         // r x (r+1) col-major
    static_assert(!OVERLAY || RQCfg<S, MAXM>::PLD <= 132, "ring slot of the overlay");
    S* vq = Cb0 + (OVERLAY ? (size_t)r * 132 : (size_t)r * (r + 1));
    S* vz = vq + (r + 8);
    S* uu = vz + (r + 8);
    S* ring = OVERLAY ? Cb0 : uu + (r + 8);  // RQ ring: r x ring_pld(r) (overlay: r x 132)
    static_assert(OVERLAY || RQCfg<S, MAXM>::PLD <= 68 || MAXM <= 32, "ring slot");
    S* scal = uu + (r + 8) + (OVERLAY ? 0 : (size_t)r * ring_pld(r));
    __shared__ int rq_flag;
    if (threadIdx.x == 0) rq_flag = 1 << 30;
    // warp-row RQ (rqw.cuh): one mbarrier per stage, one phase per RQ call
    constexpr bool RQW_ON = rq_warp_rows<S, MAXM>();
    __shared__ uint64_t rq_bars[RQW_ON ? MAXM : 1];
    if (RQW_ON && threadIdx.x < 32) rqw_bars_init(rq_bars, MAXM);
    int rq_calls = 0;
    S* rec0 = scal + 16;       // qp x (r+1): v of Q_k^{j1+s}, tau at [r]
    S* Tsm0 = rec0 + (size_t)qp * (r + 1);  // T(p, s) at Tsm[p*TL + s]
    S* wx = Tsm0 + (size_t)qp * TL;       // Y^* x, then T^* Y^* x
    S* wy = wx + (qp + 8);
    S* zx = wy + (qp + 8);
    S* zy = zx + (qp + 8);
    S* wu = zy + (qp + 8);                // Y^* v (T column build)
    S* ys1 = wu + (qp + 8);    // prefetch set (odd steps): y, B block, records, T
    S* Cb1 = PF ? ys1 + XL : ys1;
    S* rec1 = PF ? Cb1 + (size_t)r * (r + 1) : Cb1;
    S* Tsm1 = PF ? rec1 + (size_t)qp * (r + 1) : rec1;
    // (MAXM is the smallest of 8/16/32/64/128 >= r, so this is chase_dense_catchup<S>(r))
    constexpr bool MK = PF && rq_nthr<S, MAXM>() < NT && chase_dense_catchup<S>(MAXM);
    const int MLD = a.mld;
    S* Msm0 = PF ? Tsm1 + (size_t)qp * TL : ys1;  // M_t(k), even / odd steps (L x L, ld MLD)
    S* Msm1 = MK ? Msm0 + (size_t)w * MLD : Msm0;
    S* mtmp = MK ? Msm1 + (size_t)w * MLD : Msm0;  // 2 (w+1): catch-up outputs / M update row
    S* strip0 = MK ? mtmp + 2 * (size_t)(w + 1) : Msm0;
    // RQ update (rqu.cuh): R0 overlays the RQ ring (MAXM 64) or the B block (MAXM 128, after its
    // write-back); Q0 (MAXM 64) / w parts / rotations / x / b before the strip
    constexpr bool RQU_OK = RQK && rqu_supported<S, MAXM>();
    constexpr bool RQU64 = RQU_OK && MAXM == 64, RQU128 = RQU_OK && MAXM == 128;
    const bool rqu = RQU_OK && a.rqu != 0;
    constexpr int RQM = RQU_OK ? MAXM : 64;
    using RQC = RQUCfg<NT, RQM>;
    constexpr int RLD = RQC::RLD;
    double* const Rs = reinterpret_cast<double*>(RQU128 ? Cb0 : ring);
    double* const Qs = RQC::QCONC ? reinterpret_cast<double*>(strip0) : Rs;
    double* const wpart = reinterpret_cast<double*>(strip0) + (RQC::QCONC ? (size_t)RLD * RQM : 0);
    double* const cs1 = wpart + (size_t)RQC::NPART * RQM;
    double* const cs2 = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(cs1 + 2 * RQM) + 15) & ~(uintptr_t)15);
    double* const xs = cs2 + 2 * RQM;
    double* const bcol = xs + RQM;
    __shared__ int rqu_ok;
    if (rqu)
        for (int i = threadIdx.x; i < RQM; i += NT) cs2[2 * i] = RQU_SENTINEL;
    S* strip = rqu ? strip0 + RQC::extra : strip0;  // strip_cap rows x (r+1) (row-major)
    const int LDC = r + 1;
    // sweep index by ticket (not blockIdx): a CTA only ever waits on a sweep whose CTA already
    // started, so a normal (non-cooperative) launch cannot deadlock when SMs are shared
    __shared__ int t_sh;
    if (threadIdx.x == 0) t_sh = atomicAdd(&a.prog[qp], 1);
    __syncthreads();
    int role, t;  // tickets: sweep t, then its helpers
    if (a.lay) {
        if (t_sh >= qp + __ldg(a.lay + qp)) return;
        const int code = __ldg(a.lay + qp + 1 + t_sh);
        t = code >> 8;
        role = code & 255;
    } else {
        role = t_sh % (1 + a.helpers);
        t = t_sh / (1 + a.helpers);
    }
    if (t >= qp) return;
    if (role > 0) {
        far_strip_helper<S, NT, MAXM, RQK>(a, t, role - 1, sm,
                                      RQUBufs{Rs, Qs, wpart, cs1, cs2, xs, reinterpret_cast<double*>(vq),
                                              reinterpret_cast<double*>(vz), reinterpret_cast<double*>(uu)});
        return;
    }
    int* hprog = a.prog + qp + 1;
    const int j = j1 + t;
    const int kcount = min(K, 2 + (n - j - 1) / r);
    const int kprev = (t > 0) ? min(K, 2 + (n - j) / r) : 0;
    // the previous sweep's helpers: Hp of them at hprog[hbp ..] (at most 8)
    const int hbp = t > 0 ? (a.lay ? __ldg(a.lay + t - 1) : (t - 1) * a.helpers) : 0;
    const int Hp = t > 0 ? min(8, (a.lay ? __ldg(a.lay + t) : t * a.helpers) - hbp) : 0;
    int cur = 0;
    // K1 profile (HT_K1PROF): thread 0's cycle counts per phase, in shared memory (a register array
    // cost ~48 registers in every build)
    __shared__ long long pt[24];
    long long tc = clock64();  // (all threads: a tid-0-only branch here diverged warp 0 before its shuffles)
    if (tid == 0)
        for (int i = 0; i < 24; ++i) pt[i] = 0;
#define K1_TICK(slot)                         \
    do {                                      \
        if (a.prof) {                         \
            (void)*(volatile int*)&t_sh;      \
            const long long now_ = clock64(); \
            if (tid == 0) pt[slot] += now_ - tc; \
            tc = now_;                        \
        }                                     \
    } while (0)
    // sub-phase slot (16..23) that is also counted in its parent slot
#define K1_SUB(slot, parent)                  \
    do {                                      \
        if (a.prof) {                         \
            (void)*(volatile int*)&t_sh;      \
            const long long now_ = clock64(); \
            if (tid == 0) {                   \
                pt[slot] += now_ - tc;        \
                pt[parent] += now_ - tc;      \
            }                                 \
            tc = now_;                        \
        }                                     \
    } while (0)
    // cp.async of step kk's y column, catch-up records, T factor and B block into a buffer set
    auto issue_step_loads = [&](int kk, S* ysb, S* Cbb, S* recb, S* Tsmb, S* Mb, int th0, int nth, bool with_y) {
        const int me = tid - th0, mw = me >> 5, nw = nth >> 5;
        if (me < 0 || me >= nth) return;
        const int jbk = j + max(0, (kk - 1) * r + 1);
        const int i1k = j + kk * r + 1, i2k = min(j + (kk + 1) * r, n);
        const int b0k = j1 + kk * r + 1, mk = i2k - i1k + 1, nxk = i2k - b0k + 1;
        const int Lk = (t > 0) ? min(j - 1 + (kk + 1) * r, n) - b0k + 1 : 0;
        const int cBk = i1k + r - 1;
        if (!(jbk <= n && nxk > 0)) return;
        if (cBk <= n && with_y)
            for (int i = me; i < nxk; i += nth) k1_ld(&ysb[i], &IDX(a.B, a.ldb, b0k + i, cBk));
        if (MK && t > 0 && Lk >= 1) {
            const S* src = a.Mg + (int64_t)kk * a.mst;
            for (int i = mw; i < Lk; i += nw)
                for (int c = lane; c < Lk; c += 32) k1_ld(&Mb[i * MLD + c], src + (size_t)i * MLD + c);
        }
        if (!MK && t > 0 && Lk >= 1)
            for (int s2 = mw; s2 < t; s2 += nw) {  // warp per record / per T column
                const S* src = a.Qr + ((int64_t)s2 * K + kk) * (r + 1);
                for (int c = lane; c <= r; c += 32) k1_ld(&recb[s2 * (r + 1) + c], src + c);
                const S* tsrc = a.Tr + ((int64_t)s2 * K + kk) * a.TLD;
                for (int p = lane; p <= s2; p += 32) k1_ld(&Tsmb[p * TL + s2], tsrc + p);
            }
        if (mk >= 2)
            for (int cc = mw; cc < mk; cc += nw)
                for (int ii = lane; ii < mk; ii += 32) k1_ld(&Cbb[ii + cc * LDC], &IDX(a.B, a.ldb, i1k + ii, i1k + cc));
    };
    bool pf_next = false;  // step k's loads were issued during step k-1
    for (int k = 0; k < kcount; ++k) {
        bool rqu_fallback = false;  // rqu 2: the solve failed, the sweep did the RQ update itself
        const bool have = pf_next;
        pf_next = false;
        if (t > 0) {
            if (tid == 0) {
                // sweep t-1 through step k+2 and its helpers through item k+1 (their far strips of
                // (t-1, k+1) overlap rows >= b0(k-1)): the counters are read with relaxed loads
                // issued together (one L2 round trip, not one per counter), then one acquire fence
                const int need = min(k + 3, kprev), hneed = min(k + 2, kprev);
                const int* hp = hprog + hbp;
                int v = ld_relaxed(&a.prog[t - 1]);
                int hv[8];
#pragma unroll
                for (int h = 0; h < 8; ++h) hv[h] = (h < Hp) ? ld_relaxed(hp + h) : hneed;
                // rqu 2: sweep j-1's hand-over for window k (its helper's RQ update)
                const bool fw = RQU_OK && a.rqu == 2 && min(j + (k + 1) * r, n) - (j + k * r + 1) >= 1 &&
                                j + max(0, (k - 1) * r + 1) <= n;
                int fv = fw ? ld_relaxed(&a.Fdone[k]) : j;
                while (v < need) v = ld_relaxed(&a.prog[t - 1]);
                K1_TICK(0);
#pragma unroll
                for (int h = 0; h < 8; ++h)
                    while (hv[h] < hneed) hv[h] = ld_relaxed(hp + h);
                while (fv < j) fv = ld_relaxed(&a.Fdone[k]);
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                K1_TICK(9);
            }
            __syncthreads();
        }
        if (a.trace && tid == 0) a.trace[((int64_t)t * K + k) * 2] = gtimer();
        K1_TICK(0);
        S* const ys = (PF && (k & 1)) ? ys1 : ys0;
        S* const Cb = (PF && (k & 1)) ? Cb1 : Cb0;
        S* const rec = (PF && (k & 1)) ? rec1 : rec0;
        S* const Tsm = (PF && (k & 1)) ? Tsm1 : Tsm0;
        S* const Msm = (PF && (k & 1)) ? Msm1 : Msm0;
        const int jb = j + max(0, (k - 1) * r + 1);
        const int i1 = j + k * r + 1;
        const int i2 = min(j + (k + 1) * r, n);
        const int i3 = min(j + (k + 2) * r, n);
        const int i4g = j1 + 1 + max(0, (k + t - qp + 1) * r);
        // this CTA's part of the band: rows >= b0(k-1) when the helpers take the far rows
        const int i4 = a.helpers ? max(i4g, j1 + (k - a.hlag) * r + 1) : i4g;
        const int b0 = j1 + k * r + 1;
        const int m = i2 - i1 + 1;
        const int L = (t > 0) ? min(j - 1 + (k + 1) * r, n) - b0 + 1 : 0;
        const int nx = i2 - b0 + 1;
        const int cB = i1 + r - 1;  // == i2 when it exists
        const bool hasB = cB <= n;
        S* xcol = sm + (cur ? XL : 0);
        S* xnext = sm + (cur ? 0 : XL);
        const int nA = max(0, i3 - i4 + 1), nBs = max(0, i1 - i4);  // strip rows (B: above block)
        const int stA = min(nA, a.strip_cap), stB = min(nBs, a.strip_cap - stA);
        const bool gen = (m >= 2) && jb <= n && nx > 0;
        const bool cu = (t > 0) && L >= 1 && jb <= n && nx > 0;  // catch-up present
        // ---- (S1) all loads of the step at once ------------------------------------------
        // (y, records, T and the B block were prefetched during the previous step's RQ: they are
        // final once sweep j-1 finished step k+2, which step k-1 already waited for)
        if (jb <= n && nx > 0) {
            if (k == 0)
                for (int i = tid; i < nx; i += NT) k1_ld(&xcol[i], &IDX(a.A, a.lda, b0 + i, jb));
            if (!have) {
                issue_step_loads(k, ys, Cb, rec, Tsm, Msm, 0, NT, true);
            } else if (a.hlag == 0 && i1 + r - 1 <= n) {  // y was not prefetched (see far_strip_helper)
                for (int i = tid; i < nx; i += NT) k1_ld(&ys[i], &IDX(a.B, a.ldb, b0 + i, i1 + r - 1));
            }
        }
        k1_commit();
        K1_TICK(1);
        // the strip is only needed after the RQ: its own (newest) group, waited for there.  On the
        // dense path its loads are issued by warps 2.. during the fused catch-up (S2+S3) instead
        auto issue_strip = [&](int w0) {
            for (int cc = warp - w0; cc < m; cc += NW - w0) {
                for (int rr = lane; rr < stA; rr += 32) k1_ld(&strip[rr * SLD + cc], &IDX(a.A, a.lda, i4 + rr, i1 + cc));
                for (int rr = lane; rr < stB; rr += 32)
                    k1_ld(&strip[(stA + rr) * SLD + cc], &IDX(a.B, a.ldb, i4 + rr, i1 + cc));
            }
        };
        // (dense path: during the fused catch-up + left reflector; WY path: during the catch-up)
        const bool late_strip = gen && (MK || cu);
        if (jb <= n && nx > 0 && gen && !late_strip) issue_strip(0);
        if (!late_strip) k1_commit();
        K1_TICK(10);
        if (late_strip) k1_wait_group<0>();
        else k1_wait_group<1>();
        __syncthreads();
        K1_TICK(1);
        if constexpr (RQU_OK) {
            if (rqu) {  // sweep j-1's hand-over for window k (rqu.cuh), waited for before the RQ update
                if (RQU64 && gen && j > 1) {  // thread: column c, rows part, part + NP, ... (no divisions)
                    const int f = hasB ? m - 1 : m;
                    const double* FR = a.Fg + (int64_t)k * a.fst;
                    const double* FW = FR + MAXM * MAXM;
                    constexpr int NP = NT / RQM;
                    const int c = tid % RQM;
                    if (c < f)
                        for (int p = tid / RQM; p < f; p += NP) {
                            k1_ld(&Qs[p * RLD + c], FW + p * MAXM + c);
                            if (c >= p) k1_ld(&Rs[p * RLD + c], FR + p * MAXM + c);
                        }
                }
                k1_commit();
            }
        }
        if (jb <= n && nx > 0) {
            // ---- (S2) catch-up in WY form: x(0:L) <- x - Y T^* Y^* x (same for y) ----------------
            // (dense path with a reflector: merged with S3 below)
            if (cu && !(MK && gen)) {
                if constexpr (MK) {  // x <- M_t x, y <- M_t y (one round, thread per output row)
                    for (int e = tid; e < 2 * L; e += NT) {
                        const bool isy = e >= L;
                        if (isy && !hasB) continue;
                        const S* xv = isy ? ys : xcol;
                        const S* mr = Msm + (size_t)(isy ? e - L : e) * MLD;
                        S a0 = S(0.0), a1 = S(0.0), a2 = S(0.0), a3 = S(0.0);
                        int c = 0;
                        for (; c + 3 < L; c += 4) {
                            a0 = fma_s(mr[c], xv[c], a0);
                            a1 = fma_s(mr[c + 1], xv[c + 1], a1);
                            a2 = fma_s(mr[c + 2], xv[c + 2], a2);
                            a3 = fma_s(mr[c + 3], xv[c + 3], a3);
                        }
                        for (; c < L; ++c) a0 = fma_s(mr[c], xv[c], a0);
                        mtmp[e] = (a0 + a1) + (a2 + a3);
                    }
                    __syncthreads();
                    for (int e = tid; e < 2 * L; e += NT) {
                        const bool isy = e >= L;
                        if (isy && !hasB) continue;
                        (isy ? ys : xcol)[isy ? e - L : e] = mtmp[e];
                    }
                } else if (warp < 2 && (warp == 0 || hasB)) {
                    // warp 0 catches x up, warp 1 catches y up: three warp-synchronous rounds each
                    const bool isy = warp == 1;
                    S* xv = isy ? ys : xcol;
                    S* wv = isy ? wy : wx;
                    S* zv = isy ? zy : zx;
                    // round 1: w_s = Y(:,s)^* x, s < t
                    for (int s2 = lane; s2 < t; s2 += 32) {
                        const S* v = rec + (size_t)s2 * (r + 1);
                        const int ms = min(r, n - (j1 + s2 + k * r));
                        S d0 = S(0.0), d1 = S(0.0);
                        int i = 0;
                        for (; i + 1 < ms; i += 2) {
                            d0 += conj_mul(v[i], xv[s2 + i]);
                            d1 += conj_mul(v[i + 1], xv[s2 + i + 1]);
                        }
                        if (i < ms) d0 += conj_mul(v[i], xv[s2 + i]);
                        if (is_zero(v[r])) d0 = d1 = S(0.0);  // tau = 0: Q = I (record may be empty)
                        wv[s2] = d0 + d1;
                    }
                    __syncwarp();
                    // round 2: z = T^* w  (z_s = sum_{p<=s} conj(T(p,s)) w_p)
                    for (int s2 = lane; s2 < t; s2 += 32) {
                        S z = S(0.0);
                        for (int p = 0; p <= s2; ++p) z += conj_mul(Tsm[p * TL + s2], wv[p]);
                        zv[s2] = z;
                    }
                    __syncwarp();
                    // round 3: x(i) -= sum_s Y(i,s) z_s over reflectors covering row i
                    for (int i = lane; i < L; i += 32) {
                        S acc = S(0.0);
                        const int slo = max(0, i - r + 1), shi = min(t - 1, i);
                        for (int s2 = slo; s2 <= shi; ++s2) {
                            const int ms = min(r, n - (j1 + s2 + k * r));
                            if (i - s2 < ms) acc += rec[(size_t)s2 * (r + 1) + (i - s2)] * zv[s2];
                        }
                        xv[i] -= acc;
                    }
                } else if (late_strip && warp >= 2) {
                    issue_strip(2);  // (the warps the WY catch-up leaves idle)
                }
                if (late_strip) k1_commit();  // the strip group (empty for warps 0, 1)
                __syncthreads();
                if (hasB && gen)
                    for (int i = tid; i < m; i += NT)
                        if (t + i < L) Cb[i + (m - 1) * LDC] = ys[t + i];
            }
            if (!MK && hasB && gen && !cu)
                for (int i = tid; i < m; i += NT) Cb[i + (m - 1) * LDC] = ys[t + i];
            if (!gen) {  // catch-up only (no reflector at this step; Alg. 2 has m >= 2)
                for (int i = tid; i < L; i += NT) IDX(a.A, a.lda, b0 + i, jb) = xcol[i];
                if (hasB)
                    for (int i = tid; i < L; i += NT) IDX(a.B, a.ldb, b0 + i, cB) = ys[i];
                if (MK && t + 1 < qp) {  // M_{t+1}(k) = M_t(k) (Q = I), extended by identity
                    const int Ln = min(j + (k + 1) * r, n) - b0 + 1;
                    const int Lc = cu ? L : 0;
                    S* dst = a.Mg + (int64_t)k * a.mst;
                    for (int i = warp; i < Ln; i += NW)
                        for (int c = lane; c < Ln; c += 32)
                            dst[(size_t)i * MLD + c] = (i < Lc && c < Lc) ? Msm[i * MLD + c] : S(i == c ? 1.0 : 0.0);
                }
            } else {
                S tau;
                if constexpr (MK) {
                    // ---- (S2+S3) dense catch-up fused with the left reflector ------------------
                    // warp 0: caught-up rows t..t+m-1 of x, one per lane, straight into the reflector;
                    // warps 1..: rows 0..t-1 of x and rows 0..L-1 of y into mtmp ([0,t) / [L,2L)),
                    // y rows t..t+m-1 also into the B block's last column
                    auto mdot = [&](int row, const S* v) -> S {
                        const S* mr = Msm + (size_t)row * MLD;
                        S a0 = S(0.0), a1 = S(0.0), a2 = S(0.0), a3 = S(0.0);
                        int c = 0;
                        for (; c + 3 < L; c += 4) {
                            a0 = fma_s(mr[c], v[c], a0);
                            a1 = fma_s(mr[c + 1], v[c + 1], a1);
                            a2 = fma_s(mr[c + 2], v[c + 2], a2);
                            a3 = fma_s(mr[c + 3], v[c + 3], a3);
                        }
                        for (; c < L; ++c) a0 = fma_s(mr[c], v[c], a0);
                        return (a0 + a1) + (a2 + a3);
                    };
                    if (warp == 0) {
                        const int row = t + lane;
                        S xv = S(0.0);
                        if (lane < m) xv = (row < L) ? mdot(row, xcol) : xcol[row];
                        S tq;
                        double beta;
                        const S vl = larfg_reg(xv, m, tq, beta);
                        if (lane < m) vq[lane] = vl;
                        if (lane == 0) {
                            scal[0] = tq;
                            scal[1] = S(beta);
                        }
                    } else {
                        const int ny = hasB ? L : 0;
                        for (int e = tid - 32; e < t + ny; e += NT - 32) {
                            if (e < t) {
                                mtmp[e] = mdot(e, xcol);
                            } else {
                                const int i = e - t;
                                const S val = mdot(i, ys);
                                mtmp[L + i] = val;
                                if (gen && i >= t && i - t < m) Cb[(i - t) + (m - 1) * LDC] = val;
                            }
                        }
                        if (hasB && !cu)
                            for (int i = tid - 32; i < m; i += NT - 32) Cb[i + (m - 1) * LDC] = ys[t + i];
                        if (warp >= 2) issue_strip(2);
                    }
                    k1_commit();  // the strip group (empty for warps 0, 1)
                    __syncthreads();
                    K1_TICK(7);
                    tau = scal[0];
                    // (A(b0:i2, jb), B(b0:i1-1, cB) and the record are stored by the RQ's idle warps)
                } else {
                __syncthreads();
                K1_TICK(2);
                // ---- (S3) left reflector Q_k^j on A(i1:i2,jb) ----------------------------------
                if (warp == 0) {
                    S tq;
                    double beta;
                    if constexpr (MAXM <= 32) {
                        const S vl = larfg_reg(lane < m ? xcol[t + lane] : S(0.0), m, tq, beta);
                        if (lane < m) vq[lane] = vl;
                    } else {
                        larfg_regn<S, (MAXM + 31) / 32>(m, xcol + t, vq, tq, beta);
                    }
                    if (lane == 0) {
                        scal[0] = tq;
                        scal[1] = S(beta);
                    }
                }
                __syncthreads();
                K1_TICK(7);
                tau = scal[0];
                {
                    const S betaS = scal[1];
                    for (int i = tid; i < nx; i += NT) {
                        const S val = (i < t) ? xcol[i] : ((i == t) ? betaS : S(0.0));  // exact zeros (c5)
                        IDX(a.A, a.lda, b0 + i, jb) = val;
                    }
                    if (hasB)
                        for (int i = tid; i < t; i += NT) IDX(a.B, a.ldb, b0 + i, cB) = ys[i];
                    S* qr = a.Qr + ((int64_t)t * K + k) * (r + 1);
                    for (int c = tid; c < m; c += NT) qr[c] = vq[c];
                    if (tid == 0) qr[r] = tau;
                    if constexpr (RQU_OK) {
                        if (rqu) {  // R0 / Q0 from B0 (still unreduced in Cb): see rqu.cuh
                            if (j == 1) {  // T itself: R0 = B0 (upper triangular), Q0 = I
                                if constexpr (RQU64)
                                    for (int e = tid; e < m * m; e += NT) {
                                        const int p = e / m, c = e - p * m;
                                        Qs[p * RLD + c] = (p == c) ? 1.0 : 0.0;
                                        if (c >= p) Rs[p * RLD + c] = re(Cb[p + c * LDC]);
                                    }
                                if (a.rqu == 2) {  // the helper (and MAXM 128's sweep) read the hand-over form
                                    const int f = hasB ? m - 1 : m;
                                    double* FR = a.Fg + (int64_t)k * a.fst;
                                    for (int e = tid; e < f * f; e += NT) {
                                        const int p = e / f, c = e - p * f;
                                        FR[MAXM * MAXM + p * MAXM + c] = (p == c) ? 1.0 : 0.0;
                                        if (c >= p) FR[p * MAXM + c] = re(Cb[p + c * LDC]);
                                    }
                                }
                            } else if (RQU64 && hasB) {  // last column b = B0(:, m), Q0 = diag(W, 1)
                                for (int i = tid; i < m; i += NT) {
                                    Rs[i * RLD + (m - 1)] = re(Cb[i + (m - 1) * LDC]);
                                    Qs[(m - 1) * RLD + i] = (i == m - 1) ? 1.0 : 0.0;
                                    Qs[i * RLD + (m - 1)] = (i == m - 1) ? 1.0 : 0.0;
                                }
                            }
                            if (a.rqu == 2 && hasB)  // b for the helper's RQ update (and MAXM 128's R0)
                                for (int i = tid; i < m; i += NT) {
                                    const double b = re(Cb[i + (m - 1) * LDC]);
                                    a.Fb[(int64_t)k * MAXM + i] = b;
                                    if (RQU128) bcol[i] = b;
                                }
                        }
                    }
                }
                __syncthreads();
                K1_TICK(8);
                }
                // ---- (S4) B block <- Q^* B block (warps 0..NW/2-1) || T column t (others) ------
                if constexpr (MK) {
                    // m <= 32: a group of G lanes per column, one element per lane
                    if (!is_zero(tau)) {
                        const S ctau = conjv(tau);
                        const int G = m <= 8 ? 8 : (m <= 16 ? 16 : 32), CPW = 32 / G;
                        const int i = lane & (G - 1);
                        const S vi = i < m ? vq[i] : S(0.0);
                        for (int base = warp * CPW; base < m; base += NW * CPW) {
                            const int c = base + lane / G;
                            const bool ok = c < m && i < m;
                            const S e = ok ? Cb[i + c * LDC] : S(0.0);
                            S d = conj_mul(vi, e);
                            for (int o = 1; o < G; o <<= 1) d += shfl_xor(d, o);
                            if (ok) Cb[i + c * LDC] = e - vi * (d * ctau);
                        }
                    }
                } else if (warp < NW / 2) {
                    // warps 0..NW/2-1: warp per column, RPL rows per lane, U columns in flight
                    // (their shuffle reductions interleave)
                    if (!is_zero(tau)) {
                        const S ctau = conjv(tau);
                        constexpr int RPL = (MAXM + 31) / 32, U = 4, WG = NW / 2;
                        S vr[RPL];
#pragma unroll
                        for (int rr = 0; rr < RPL; ++rr) vr[rr] = (lane + 32 * rr < m) ? vq[lane + 32 * rr] : S(0.0);
                        for (int cb = warp; cb < m; cb += WG * U) {
                            S e[U][RPL], d[U];
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                const int c = cb + u * WG;
                                d[u] = S(0.0);
#pragma unroll
                                for (int rr = 0; rr < RPL; ++rr) {
                                    const int i = lane + 32 * rr;
                                    e[u][rr] = (c < m && i < m) ? Cb[i + c * LDC] : S(0.0);
                                    d[u] += conj_mul(vr[rr], e[u][rr]);
                                }
                            }
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                                for (int u = 0; u < U; ++u) d[u] += shfl_xor(d[u], o);
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                const int c = cb + u * WG;
                                const S sc = d[u] * ctau;
#pragma unroll
                                for (int rr = 0; rr < RPL; ++rr) {
                                    const int i = lane + 32 * rr;
                                    if (c < m && i < m) Cb[i + c * LDC] = e[u][rr] - vr[rr] * sc;
                                }
                            }
                        }
                    }
                } else if (!MK) {
                    const long long s4t0 = a.prof ? clock64() : 0;
                    // xLARFT column t: T(0:t,t) = -tau T(0:t,0:t) (Y(:,0:t)^* v), T(t,t) = tau
                    const int hn = NT - NT / 2, me = tid - NT / 2;
                    for (int s = me; s < t; s += hn) {
                        const S* v = rec + (size_t)s * (r + 1);
                        const int ms = min(r, n - (j1 + s + k * r));
                        const int hi = min(s + ms, t + m);
                        S d0 = S(0.0), d1 = S(0.0), d2 = S(0.0), d3 = S(0.0);
                        int ii = t;
                        for (; ii + 3 < hi; ii += 4) {
                            d0 += conj_mul(v[ii - s], vq[ii - t]);
                            d1 += conj_mul(v[ii + 1 - s], vq[ii + 1 - t]);
                            d2 += conj_mul(v[ii + 2 - s], vq[ii + 2 - t]);
                            d3 += conj_mul(v[ii + 3 - s], vq[ii + 3 - t]);
                        }
                        for (; ii < hi; ++ii) d0 += conj_mul(v[ii - s], vq[ii - t]);
                        S d = (d0 + d1) + (d2 + d3);
                        if (is_zero(v[r])) d = S(0.0);
                        wu[s] = d;
                    }
                    named_bar(2, hn);
                    S* tr = a.Tr + ((int64_t)t * K + k) * a.TLD;
                    for (int p = me; p <= t; p += hn) {
                        S val;
                        if (p == t) {
                            val = tau;
                        } else {
                            S acc = S(0.0);
                            for (int s = p; s < t; ++s) acc += Tsm[p * TL + s] * wu[s];
                            val = -(tau * acc);
                        }
                        tr[p] = val;
                    }
                    if (a.prof && tid == NT / 2) atomicAdd((unsigned long long*)&pt[23], (unsigned long long)(clock64() - s4t0));
                }
                K1_SUB(22, 3);
                __syncthreads();
                if constexpr (OVERLAY) {  // the block goes to HBM: the RQ ring reuses its smem
                    for (int cc = warp; cc < m; cc += NW)
                        for (int ii = lane; ii < m; ii += 32) IDX(a.B, a.ldb, i1 + ii, i1 + cc) = Cb[ii + cc * LDC];
                    __syncthreads();
                    if constexpr (RQU128) {
                        if (rqu) {  // R0 into the block's buffer: sweep j-1's hand-over (L2 reads) and b
                            const int f = hasB ? m - 1 : m;
                            rqu_load_block<NT, MAXM>(Rs, a.Fg + (int64_t)k * a.fst, f, true);
                            if (hasB)
                                for (int i = tid; i < m; i += NT) Rs[i * RLD + (m - 1)] = bcol[i];
                            __syncthreads();
                        }
                    }
                }
                K1_TICK(3);
                // ---- (S5) RQ of the block -> Z_k^j ---------------------------------------------
                if (rqu) {  // RQ update (rqu.cuh): the next step's prefetch first, then F / strip landed
                    if (PF && k + 1 < kcount) {
                        issue_step_loads(k + 1, (k & 1) ? ys0 : ys1, (k & 1) ? Cb0 : Cb1, (k & 1) ? rec0 : rec1,
                                         (k & 1) ? Tsm0 : Tsm1, (k & 1) ? Msm0 : Msm1, 0, NT, a.hlag != 0);
                        asm volatile("cp.async.commit_group;\n" ::: "memory");
                        pf_next = true;
                    }
                    if (pf_next) k1_wait_group<1>();
                    else k1_wait_group<0>();
                    __syncthreads();
                    K1_SUB(16, 6);
                    if constexpr (RQU64) {
                        const double* vd = reinterpret_cast<const double*>(vq);
                        double* ud = reinterpret_cast<double*>(uu);
                        const bool self = a.rqu == 2 && (k * a.rqu_self_num) % a.rqu_self_den < a.rqu_self_num;
                        if (a.rqu == 2 && !self)
                            rqu_fallback = !rqu_solve<NT, MAXM>(m, vd, re(tau), Rs, Qs, wpart, xs, ud, &rqu_ok,
                                                                a.prof ? pt : nullptr, &tc);
                        if (a.rqu != 2 || rqu_fallback || self)
                            rqu_direction<NT, MAXM>(m, vd, re(tau), Rs, Qs, wpart, cs1, cs2, ud, a.prof ? pt : nullptr, &tc);
                        if (self) rqu_fallback = true;  // the hand-over below, Fdone at the release
                    } else if constexpr (RQU128) {  // Q0 read from the hand-over in L2
                        const double* vd = reinterpret_cast<const double*>(vq);
                        double* ud = reinterpret_cast<double*>(uu);
                        const double* FW = a.Fg + (int64_t)k * a.fst + MAXM * MAXM;
                        if (!rqu_solve<NT, MAXM>(m, vd, re(tau), Rs, Qs, wpart, xs, ud, &rqu_ok, a.prof ? pt : nullptr, &tc,
                                                 FW, hasB)) {
                            // the designated helper runs the RQ update now and returns Q~(1,:)
                            if (tid == 0) {
                                __threadfence();
                                st_release(&a.Freq[k], j + 1);
                                while (ld_relaxed(&a.Fdirok[k]) < j + 1) {
                                }
                                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                            }
                            __syncthreads();
                            for (int c = tid; c < m; c += NT) ud[c] = ldcg(a.Fdir + (int64_t)k * MAXM + c);
                        }
                    }
                } else if constexpr (!RQU_OK) {
                if (PF && k + 1 < kcount) {  // next step's inputs land while the RQ runs (issued by
                    // the warps the RQ does not use, if any)
                    constexpr int RQT = rq_nthr<S, MAXM>();
                    issue_step_loads(k + 1, (k & 1) ? ys0 : ys1, (k & 1) ? Cb0 : Cb1, (k & 1) ? rec0 : rec1,
                                     (k & 1) ? Tsm0 : Tsm1, (k & 1) ? Msm0 : Msm1, RQT < NT ? RQT : 0, RQT < NT ? NT - RQT : NT,
                                     a.hlag != 0);
                    asm volatile("cp.async.commit_group;\n" ::: "memory");
                    pf_next = true;
                }
                if constexpr (MK) {
                    constexpr int RQT = rq_nthr<S, MAXM>();
                    if (tid >= RQT) {  // the step's stores of A(b0:i2, jb), B(b0:i1-1, cB), record
                        const int nth = NT - RQT, me = tid - RQT;
                        const S betaS = scal[1];
                        for (int i = me; i < nx; i += nth) {
                            const S val = (i < t) ? mtmp[i] : ((i == t) ? betaS : S(0.0));  // exact zeros (c5)
                            IDX(a.A, a.lda, b0 + i, jb) = val;
                        }
                        if (hasB)
                            for (int i = me; i < t; i += nth) IDX(a.B, a.ldb, b0 + i, cB) = mtmp[L + i];
                        S* qr = a.Qr + ((int64_t)t * K + k) * (r + 1);
                        for (int c = me; c < m; c += nth) qr[c] = vq[c];
                        if (me == 0) qr[r] = tau;
                    }
                    // the idle warps form M_{t+1}(k) = (Q_k^j)^* M_t(k) for sweep t+1 (in place in Mg)
                    if (t + 1 < qp && tid >= RQT) {
                        const int nth = NT - RQT, me = tid - RQT, mw = me >> 5, nw = nth >> 5;
                        const int Ln = min(j + (k + 1) * r, n) - b0 + 1;
                        const int Lc = cu ? L : 0;  // M_0 = I
                        auto base = [&](int i, int c) -> S {
                            return (i < Lc && c < Lc) ? Msm[i * MLD + c] : S(i == c ? 1.0 : 0.0);
                        };
                        const S ctau = conjv(tau);
                        for (int c = me; c < Ln; c += nth) {  // d_c = conj(tau) v^* M(t:t+m, c)
                            S d0 = S(0.0), d1 = S(0.0);
                            int p2 = 0;
                            for (; p2 + 1 < m; p2 += 2) {
                                d0 += conj_mul(vq[p2], base(t + p2, c));
                                d1 += conj_mul(vq[p2 + 1], base(t + p2 + 1, c));
                            }
                            if (p2 < m) d0 += conj_mul(vq[p2], base(t + p2, c));
                            wx[c] = (d0 + d1) * ctau;
                        }
                        named_bar(3, nth);
                        S* dst = a.Mg + (int64_t)k * a.mst;
                        for (int i = mw; i < Ln; i += nw) {
                            const bool upd = i >= t && i < t + m;
                            const S vi = upd ? vq[i - t] : S(0.0);
                            for (int c = lane; c < Ln; c += 32) {
                                S val = base(i, c);
                                if (upd) val -= vi * wx[c];
                                dst[(size_t)i * MLD + c] = val;
                            }
                        }
                    }
                }
                if (tid < rq_nthr<S, MAXM>())
                    rq_dir<S, MAXM>(m, Cb, LDC, ring, &rq_flag, uu, OVERLAY ? 132 : ring_pld(r), rq_bars, rq_calls & 1);
                ++rq_calls;
                }
                if (pf_next) k1_wait_group<1>();  // the strip (the prefetch group may stay in flight)
                else k1_wait_group<0>();
                __syncthreads();
                if (tid == 0) rq_flag = 1 << 30;
                K1_TICK(6);
                if (warp == 0) {
                    S sig;
                    double b2;
                    if constexpr (MAXM <= 32) {  // register form (fast rsqrt / reciprocal)
                        const S vl = larfg_reg(lane < m ? uu[lane] : S(0.0), m, sig, b2);
                        if (lane < m) vz[lane] = vl;
                    } else {
                        larfg_regn<S, (MAXM + 31) / 32>(m, uu, vz, sig, b2);
                    }
                    if (lane == 0) scal[2] = sig;
                } else if (hasB && cu) {
                    // caught-up rows b0..i1-1 of column i2 are also rows of the staged B strip
                    for (int i = tid - 32; i < t && i < L; i += NT - 32) {
                        const int rr = (b0 + i) - i4;
                        if (rr >= 0 && rr < stB) strip[(stA + rr) * SLD + (m - 1)] = MK ? mtmp[L + i] : ys[i];
                    }
                }
                __syncthreads();
                K1_TICK(4);
                const S sig = scal[2];
                // ---- (S6) right reflector Z_k^j on the band, next column ----------------------
                const int nBb = max(0, i2 - i4 + 1);  // B rows i4..i2 (block rows i1..i2 from Cb)
                const int bn = b0 + r;                 // first row of the next step's column
                // SPR threads per row (adjacent lanes), CPR columns each, dot by shuffle-xor
#ifndef HT_STRIP_SPR_BYTES
#define HT_STRIP_SPR_BYTES 256
#endif
                constexpr int SPR = (MAXM * (int)sizeof(S) > HT_STRIP_SPR_BYTES) ? MAXM * (int)sizeof(S) / HT_STRIP_SPR_BYTES : 1;
                constexpr int CPR = MAXM / SPR;
                const int part = tid % SPR, c0 = part * CPR;
                const int nrows = nA + nBb;
                for (int eb = tid / SPR; eb - tid / SPR < nrows; eb += NT / SPR) {  // uniform trip count per warp
                    const int e = eb;
                    const bool act = e < nrows;
                    const bool isA = e < nA;
                    const int row = isA ? i4 + e : i4 + (e - nA);
                    S v[CPR];
                    S* gp = isA ? &IDX(a.A, a.lda, row, i1) : &IDX(a.B, a.ldb, row, i1);
                    const int64_t ld = isA ? a.lda : a.ldb;
                    if (act) {
                        if (isA && e < stA) {
#pragma unroll
                            for (int c = 0; c < CPR; ++c)
                                if (c0 + c < m) v[c] = strip[e * SLD + c0 + c];
                        } else if (!OVERLAY && !isA && row >= i1) {
#pragma unroll
                            for (int c = 0; c < CPR; ++c)
                                if (c0 + c < m) v[c] = Cb[(row - i1) + (c0 + c) * LDC];
                        } else if (!isA && row < i1 && (e - nA) < stB) {
#pragma unroll
                            for (int c = 0; c < CPR; ++c)
                                if (c0 + c < m) v[c] = strip[(stA + e - nA) * SLD + c0 + c];
                        } else {
#pragma unroll
                            for (int c = 0; c < CPR; ++c)
                                if (c0 + c < m) v[c] = ldcg(gp + (c0 + c) * ld);
                        }
                    }
                    S s0 = S(0.0), s1 = S(0.0);
                    if (act && !is_zero(sig)) {
#pragma unroll
                        for (int c = 0; c < CPR; ++c)
                            if (c0 + c < m) {
                                if (c & 1) s1 = fma_s(v[c], vz[c0 + c], s1);
                                else s0 = fma_s(v[c], vz[c0 + c], s0);
                            }
                    }
                    S sdot = s0 + s1;
                    if constexpr (SPR > 1) {
#pragma unroll
                        for (int o = 1; o < SPR; o <<= 1) sdot += shfl_xor(sdot, o);
                    }
                    if (act) {
                        if (!is_zero(sig)) {
                            const S sv = sdot * sig;
#pragma unroll
                            for (int c = 0; c < CPR; ++c)
                                if (c0 + c < m) v[c] -= sv * conjv(vz[c0 + c]);
                        }
                        if (!isA && row > i1 && part == 0) v[0] = S(0.0);  // B(i1+1:i2,i1) = 0 (reading c5)
#pragma unroll
                        for (int c = 0; c < CPR; ++c)
                            if (c0 + c < m) gp[(c0 + c) * ld] = v[c];
                        if (isA && row >= bn && part == 0) xnext[row - bn] = v[0];  // column jb of step k+1
                    }
                }
                S* zr = a.Zr + ((int64_t)t * K + k) * (r + 1);
                for (int c = tid; c < m; c += NT) zr[c] = vz[c];
                if (tid == 0) zr[r] = sig;
                if constexpr (RQU64)
                    if (rqu && (a.rqu == 1 || rqu_fallback)) {  // hand-over to sweep j+1 (read at its step k)
                        K1_TICK(5);
                        double* FR = a.Fg + (int64_t)k * a.fst;
                        rqu_handoff<NT, MAXM>(m, Rs, Qs, reinterpret_cast<const double*>(vz), re(sig), FR, FR + MAXM * MAXM);
                        K1_SUB(20, 5);
                    }
            }
        }
        // the next step's column jb must come from global if this step did not produce it
        __syncthreads();
        K1_TICK(5);
        if (!gen && k + 1 < kcount) {
            const int bn = b0 + r, jbn = j + k * r + 1, nxn = min(j + (k + 2) * r, n) - bn + 1;
            for (int i = tid; i < nxn; i += NT) xnext[i] = ldcg(&IDX(a.A, a.lda, bn + i, jbn));
            __syncthreads();
        }
        if (tid == NT - 32) {  // (not thread 0: it spins on the previous sweep meanwhile)
            __threadfence();
            if (RQU_OK && rqu_fallback) st_release(&a.Fdone[k], j + 1);  // (rqu 2: the sweep did the hand-over)
            if (a.trace) a.trace[((int64_t)t * K + k) * 2 + 1] = gtimer();
            st_release(&a.prog[t], k + 1);
        }
        cur ^= 1;
        if (tid == 0) pt[11] += 1;  // step count (not a time slot)
    }
    if (a.prof && tid == 0 && (a.prof_t0 < 0 || t == a.prof_t0))
        for (int i = 0; i < 24; ++i) atomicAdd((unsigned long long*)&a.prof[i], (unsigned long long)pt[i]);
#undef K1_TICK
#undef K1_SUB
}
