// rqu.cuh -- K1's opposite reflector from an UPDATED RQ factorisation (real fp64), O(m^2) per
// step instead of the O(m^3) Householder RQ of the block ("the r^2 n^2 cost of the RQ
// factorizations can be significant if r is large", model: tests/rqu_ref.py).
//
// Step (j,k) reduces B' = Q^* B0 with B0 = B(i1:i2, i1:i2) before the left reflector
// Q = I - tau v v^*.  B0's leading (m-1) x (m-1) block is rows/columns 2..m of the block sweep j-1
// reduced at the same k, B'_prev Z_prev = R~ (Q~ Z_prev) -- so sweep j-1 hands over
// R1 = R~(2:m, 2:m) and W = (Q~ Z_prev)(2:m, 2:m) with B0(1:m-1, 1:m-1) = R1 W, and
//     B0 = R0 Q0,  R0 = [[R1, b'], [0, beta]],  Q0 = diag(W, 1)   (b = the caught-up column i2;
//                                                                 the last row of B0 is 0 left of it)
//     Q^* B0 = (R0 - v w^T) Q0,  w = tau R0^T v.
// The RQ of the rank-one-modified triangle is 2(m-1) Givens column rotations (Golub-Van Loan's
// rank-one update, column form): (B) rotations G_0..G_{m-2} reduce w^T to ||w|| e_{m-1}^T (they
// depend on w alone: prefix norms); (C) applied to R0 they make it upper Hessenberg, then the
// rank-one part only changes the last column; (D) rotations G'_{m-2}..G'_0 restore the triangle
// bottom-up (a sequential chain: each needs the diagonal entry the previous one produced).
// Q~ = G'_0^T ... G'_{m-2}^T G_{m-2}^T ... G_0^T Q0 (row rotations of Q0), and as in reading c3
// Z_k^j = larfg(Q~(1,:)^T); the hand-over for sweep j+1 is R~(2:m,2:m) and (Q~ Z_k^j)(2:m,2:m).
// When the block is clipped at n (no column i2 = i1+r-1), B0 is the whole m x m hand-over.
// The first sweep (j = 1) starts from T itself: R1 = B0(1:m-1, 1:m-1) (upper triangular), W = I.
//
// Thread roles (NT threads): (A) all threads form w (column dots of R0 in NPART row parts);
// warp 0 then runs (B), (C) on its rows (lane + 32e) and the chain (D), broadcasting each
// rotation by shuffles; warps 1..QW own Q0's columns: the forward rotations after (B), then the
// backward ones trailing the chain through a shared progress counter.
#pragma once
#include <type_traits>
#include "scalar.cuh"

// [a, b] [[c, s], [-s, c]] = [0, hypot(a, b)]
__device__ __forceinline__ void giv_rot(double a, double b, double& c, double& s) {
    const double r2 = fma(a, a, b * b);
    if (r2 > 1e-280 && r2 < 1e280) {
        const double inv = fast_rsqrt(r2);
        c = b * inv;
        s = a * inv;
    } else if (a == 0.0 && b == 0.0) {
        c = 1.0;
        s = 0.0;
    } else {  // (tiny / huge: no squares)
        const double rho = hypot(a, b);
        c = b / rho;
        s = a / rho;
    }
}
__device__ __forceinline__ double sqrt_nn(double x) { return x > 0.0 ? x * fast_rsqrt(x) : 0.0; }

// 32-bit shared-window addresses, formed once per call: generic shared pointers inside the loops
// made the compiler re-derive the window base (S2UR SR_CgaCtaId) on every access, on the chain
__device__ __forceinline__ unsigned rq_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
// an address the compiler cannot rematerialise (it re-derived symbol addresses via S2UR per use)
__device__ __forceinline__ unsigned opaque_u32(unsigned x) {
    unsigned y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ double lds64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ double lds64v(unsigned a) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
// predicated load (0 when !pred; no branch around it)
__device__ __forceinline__ double lds64_if(bool pred, unsigned a) {
    double v;
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n mov.b64 %0, 0;\n @p ld.shared.f64 %0, [%1];\n}"
                 : "=d"(v)
                 : "r"(a), "r"((int)pred));
    return v;
}
// predicated store (no branch: a divergent if around a store costs a BSSY/BSYNC pair per use)
__device__ __forceinline__ void sts64_if(bool pred, unsigned a, double v) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.shared.f64 [%0], %1;\n}" ::"r"(a), "d"(v), "r"((int)pred));
}
__device__ __forceinline__ void sts64v_if(bool pred, unsigned a, double v) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.volatile.shared.f64 [%0], %1;\n}" ::"r"(a), "d"(v),
                 "r"((int)pred));
}
__device__ __forceinline__ void sts32v_if(bool pred, unsigned a, int v) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.volatile.shared.s32 [%0], %1;\n}" ::"r"(a), "r"(v),
                 "r"((int)pred));
}
__device__ __forceinline__ void sts128v_if(bool pred, unsigned a, double x, double y) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n @p st.volatile.shared.v2.f64 [%0], {%1, %2};\n}" ::"r"(a), "d"(x),
                 "d"(y), "r"((int)pred));
}
__device__ __forceinline__ void lds128v(unsigned a, double& x, double& y) {
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
// a rotation slot of (D) not yet written (|c| <= 1)
#define RQU_SENTINEL 4.0
__device__ __forceinline__ void sts64v(unsigned a, double v) { asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }
__device__ __forceinline__ int lds32v(unsigned a) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts32v(unsigned a, int v) { asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(a), "r"(v)); }

template <int NT, int MAXM>
struct RQUCfg {
    static constexpr int RLD = MAXM + 1;           // row-major ld of R0 / Q0 in shared memory (odd)
    static constexpr int RPL = (MAXM + 31) / 32;   // chain rows per lane (warp 0)
    static constexpr int NPART = NT / MAXM;        // (A) row parts
    // MAXM <= 64: Q0 has its own buffer and warps 1..QW rotate it concurrently with the chain (D);
    // MAXM = 128: R0 and Q0 do not both fit -- Q0 reuses R0's buffer after the hand-over of R~
    static constexpr bool QCONC = MAXM <= 64;
    static constexpr int QW = QCONC ? (MAXM + 31) / 32 : 0;
    // shared memory besides R0 (which overlays the RQ ring / the B block): Q0 (QCONC), w parts,
    // rotations (B) and (D) (+2: cs2 alignment), x of the solve, the column b
    static constexpr size_t extra =
        (QCONC ? (size_t)MAXM * RLD : 0) + (size_t)NPART * MAXM + 4 * (size_t)MAXM + 2 + 2 * (size_t)MAXM;
    static_assert(NPART >= 1 && NT >= 32 * (1 + QW) && NT >= MAXM, "RQU thread roles");
};

// In: Rs = R0 (row-major, ld RLD, upper triangle rows/cols < m), Qs = Q0 (m x m), v (v[0] = 1),
// tau.  Out: Rs = R~ (upper triangle; the subdiagonal holds stale values), Qs = Q~, uu = Q~(0,:)^T.
// Called by all NT threads; ends with a barrier.  cs2 (16-byte aligned) must hold the sentinel in its
// even slots at entry (initialise once; every call restores it).
// (profile: thread 0's cycles into K1 sub-slot `slot`, also counted in slot 6)
__device__ __forceinline__ void rqu_tick(long long* pt, long long* tc0, int slot) {
    if (pt) {  // (all threads: tc0 is per thread; only thread 0 records)
        const long long now = clock64();
        if (threadIdx.x == 0) {
            pt[slot] += now - *tc0;
            pt[6] += now - *tc0;
        }
        *tc0 = now;
    }
}

// (A) w = tau R0^T v in NPART row parts: wpart[part][c] (w = tau * sum of the parts).  All threads;
// ends with a barrier.
template <int NT, int MAXM>
__device__ __forceinline__ void rqu_phase_w(int m, const double* v, const double* Rs, double* wpart) {
    using C = RQUCfg<NT, MAXM>;
    constexpr int RLD = C::RLD, NPART = C::NPART, RPP = MAXM / NPART;
    const int tid = threadIdx.x;
    const int c = tid % MAXM, part = tid / MAXM;
    if (part < NPART) {
        double s0 = 0.0, s1 = 0.0;
        if (c < m) {
            const int p0 = part * RPP, p1 = min(p0 + RPP, c + 1);
            int p = p0;
            for (; p + 1 < p1; p += 2) {
                s0 = fma(Rs[p * RLD + c], v[p], s0);
                s1 = fma(Rs[(p + 1) * RLD + c], v[p + 1], s1);
            }
            if (p < p1) s0 = fma(Rs[p * RLD + c], v[p], s0);
        }
        wpart[part * MAXM + c] = s0 + s1;
    }
    __syncthreads();
}

template <int NT, int MAXM>
__device__ __forceinline__ void rqu_direction(int m, const double* v, double tau, double* Rs, double* Qs, double* wpart,
                                              double* cs1, double* cs2, double* uu,
                                              long long* pt = nullptr, long long* tc0 = nullptr) {
    using C = RQUCfg<NT, MAXM>;
    constexpr int RLD = C::RLD, RPL = C::RPL, NPART = C::NPART, QW = C::QW;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto tick = [&](int slot) { rqu_tick(pt, tc0, slot); };
    rqu_phase_w<NT, MAXM>(m, v, Rs, wpart);
    tick(17);
    if (warp == 0) {
        // ---- (B) G_i (i = 0..m-2) zero w_i into w_{i+1}: p_0 = w_0, p_i = ||w(0:i)||, rotation
        // (p_i, w_{i+1}); lane l holds w_{RPL l + e}
        double wl[RPL], Sl[RPL];
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
            const int i = RPL * lane + e;
            double x = 0.0;
            if (i < m) {
#pragma unroll
                for (int p = 0; p < NPART; ++p) x += wpart[p * MAXM + i];
                x *= tau;
            }
            wl[e] = x;
            acc = fma(x, x, acc);
            Sl[e] = acc;
        }
        double P = acc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, P, o);
            if (lane >= o) P += y;
        }
        double E = __shfl_up_sync(0xffffffffu, P, 1);
        if (lane == 0) E = 0.0;
#pragma unroll
        for (int e = 0; e < RPL; ++e) Sl[e] += E;
        const double wnext = __shfl_down_sync(0xffffffffu, wl[0], 1);
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
            const int i = RPL * lane + e;
            if (i <= m - 2) {
                const double pi = (i == 0) ? wl[0] : sqrt_nn(Sl[e]);
                const double bi = (e + 1 < RPL) ? wl[(e + 1) % RPL] : wnext;
                double c, s;
                giv_rot(pi, bi, c, s);
                cs1[2 * i] = c;
                cs1[2 * i + 1] = s;
            }
        }
        // gamma = ||w|| = sqrt(S_{m-1})
        double Sm = Sl[0];
#pragma unroll
        for (int e = 1; e < RPL; ++e)
            if ((m - 1) % RPL == e) Sm = Sl[e];
        const double gamma = sqrt_nn(__shfl_sync(0xffffffffu, Sm, (m - 1) / RPL));
        __syncwarp();
        if constexpr (C::QCONC) asm volatile("bar.arrive 4, %0;" ::"r"(32 * (1 + QW)) : "memory");  // cs1 -> the Q warps
        // ---- (C) R0 G_0 ... G_{m-2} (upper Hessenberg), minus v gamma e_{m-1}^T
        // (loops unrolled by two with ping-pong register sets: a loop-carried copy of a prefetched
        // value made the compiler place the copy right behind the load, stalling on it)
        const unsigned rs0 = opaque_u32(rq_smem_u32(Rs)), c1a = opaque_u32(rq_smem_u32(cs1)),
                       c2a = opaque_u32(rq_smem_u32(cs2));
        unsigned ra[RPL];  // address of row p = lane + 32e
#pragma unroll
        for (int e = 0; e < RPL; ++e) ra[e] = rs0 + 8u * (unsigned)((lane + 32 * e) * RLD);
        double carry[RPL];
#pragma unroll
        for (int e = 0; e < RPL; ++e) carry[e] = (lane + 32 * e == 0) ? lds64(rs0) : 0.0;
        {
            double xa[RPL], xb[RPL], ca = 0.0, sa = 0.0, cb = 0.0, sb = 0.0;
            auto load = [&](int i, double* x, double& c, double& s) {  // rotation i, column i + 1
                c = lds64(c1a + 16u * i);
                s = lds64(c1a + 16u * i + 8);
#pragma unroll
                for (int e = 0; e < RPL; ++e) x[e] = lds64_if(lane + 32 * e < m, ra[e] + 8u * (i + 1));
            };
            auto body = [&](int i, const double* xj, double c, double s) {
#pragma unroll
                for (int e = 0; e < RPL; ++e) {
                    const int p = lane + 32 * e;
                    const bool act = p < m && i >= p - 1;
                    const double xi = carry[e];
                    sts64_if(act, ra[e] + 8u * i, fma(xi, c, -xj[e] * s));
                    const double nc = fma(xi, s, xj[e] * c);
                    carry[e] = act ? nc : xi;
                }
            };
            if (m >= 2) load(0, xa, ca, sa);
            for (int i = 0; i <= m - 2; i += 2) {
                if (i + 1 <= m - 2) load(i + 1, xb, cb, sb);
                body(i, xa, ca, sa);
                if (i + 1 > m - 2) break;
                if (i + 2 <= m - 2) load(i + 2, xa, ca, sa);
                body(i + 1, xb, cb, sb);
            }
        }
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
            const int p = lane + 32 * e;
            if (p < m) carry[e] = fma(-v[p], gamma, carry[e]);
        }
        tick(18);
        // ---- (D) Hessenberg -> triangle: G'_j (j = m-2..0) zeroes H(j+1, j) against the current
        // H(j+1, j+1) (row j+1's carry); rows p <= j+1 rotate columns (j, j+1).  The lead's
        // subdiagonal entry comes by a broadcast load (prefetched), only its carry by shuffles; a
        // rotation goes to the Q warps as one 16-byte store (its slot holds a sentinel until then).
        {
            double xa[RPL], xb[RPL], aa = 0.0, ab = 0.0;
            auto load = [&](int j, double* x, double& al) {  // column j of the rows p <= j + 1
#pragma unroll
                for (int e = 0; e < RPL; ++e) x[e] = lds64_if(lane + 32 * e <= j + 1, ra[e] + 8u * j);
                al = lds64(rs0 + 8u * ((j + 1) * RLD + j));
            };
            auto body = [&](int j, const double* xj, double a, auto ne) {  // ne: rows per lane still active
                constexpr int NE = decltype(ne)::value;
                const int L = (j + 1) & 31, eL = (j + 1) >> 5;
                double b = carry[0];
#pragma unroll
                for (int e = 1; e < NE; ++e)
                    if (eL == e) b = carry[e];
                b = __shfl_sync(0xffffffffu, b, L);
                double c, s;
                giv_rot(a, b, c, s);  // (every lane: no second broadcast)
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    const int p = lane + 32 * e;
                    const bool act = p < m && p <= j + 1;
                    sts64_if(act, ra[e] + 8u * (j + 1), fma(xj[e], s, carry[e] * c));
                    carry[e] = fma(xj[e], c, -carry[e] * s);  // (rows past their lead rotation: dead)
                }
                sts128v_if(lane == 0, c2a + 16u * j, c, s);
            };
            auto run = [&](int jhi, int jlo, auto ne) {  // rotations jhi down to jlo, NE rows per lane
                if (jhi < jlo) return;
                load(jhi, xa, aa);
                for (int j = jhi; j >= jlo; j -= 2) {
                    if (j - 1 >= jlo) load(j - 1, xb, ab);  // (column j-1 is untouched until rotation j-1)
                    body(j, xa, aa, ne);
                    if (j - 1 < jlo) break;
                    if (j - 2 >= jlo) load(j - 2, xa, aa);
                    body(j - 1, xb, ab, ne);
                }
            };
            // rows >= 32 e drop out once j + 1 < 32 e
            if constexpr (RPL == 1) {
                run(m - 2, 0, std::integral_constant<int, 1>());
            } else if constexpr (RPL == 2) {
                run(m - 2, 31, std::integral_constant<int, 2>());
                run(min(m - 2, 30), 0, std::integral_constant<int, 1>());
            } else {
                static_assert(RPL == 4, "MAXM 128");
                run(m - 2, 95, std::integral_constant<int, 4>());
                run(min(m - 2, 94), 63, std::integral_constant<int, 3>());
                run(min(m - 2, 62), 31, std::integral_constant<int, 2>());
                run(min(m - 2, 30), 0, std::integral_constant<int, 1>());
            }
        }
        if (lane == 0) sts64(rs0, carry[0]);
        tick(21);
    } else if (C::QCONC && warp <= QW) {
        // ---- Q~ = G'^T G^T Q0, one column per thread: forward rotations (B), then the chain's
        asm volatile("bar.sync 4, %0;" ::"r"(32 * (1 + QW)) : "memory");
        const int c = tid - 32;
        if (c < m) {
            const unsigned qa = opaque_u32(rq_smem_u32(Qs)) + 8u * c, c1a = opaque_u32(rq_smem_u32(cs1)),
                           c2a = opaque_u32(rq_smem_u32(cs2));
            double carry = lds64(qa);
            {
                double ya, yb, ca, sa, cb, sb;
                auto load = [&](int i, double& y, double& cc, double& ss) {
                    y = lds64(qa + 8u * (RLD * (i + 1)));
                    cc = lds64(c1a + 16u * i);
                    ss = lds64(c1a + 16u * i + 8);
                };
                auto body = [&](int i, double yj, double cc, double ss) {
                    sts64(qa + 8u * (RLD * i), fma(cc, carry, -ss * yj));
                    carry = fma(ss, carry, cc * yj);
                };
                load(0, ya, ca, sa);
                for (int i = 0; i <= m - 2; i += 2) {
                    if (i + 1 <= m - 2) load(i + 1, yb, cb, sb);
                    body(i, ya, ca, sa);
                    if (i + 1 > m - 2) break;
                    if (i + 2 <= m - 2) load(i + 2, ya, ca, sa);
                    body(i + 1, yb, cb, sb);
                }
            }
            for (int j = m - 2; j >= 0; --j) {
                const double yj = lds64(qa + 8u * (RLD * j));
                double cc, ss;
                do {
                    lds128v(c2a + 16u * j, cc, ss);
                } while (cc == RQU_SENTINEL);
                sts64(qa + 8u * (RLD * (j + 1)), fma(ss, yj, cc * carry));
                carry = fma(cc, yj, -ss * carry);
            }
            Qs[c] = carry;
            uu[c] = carry;
        }
    }
    __syncthreads();
    if constexpr (C::QCONC)  // (before the next call's barriers; QCONC off: rqu_q_apply still reads them)
        for (int j = tid; j < MAXM; j += NT) cs2[2 * j] = RQU_SENTINEL;
    tick(19);
}

// The direction of Z_k^j by a triangular solve (the RQ update's Givens chain stays off the critical
// path: the sweep's far-strip helper runs it for the hand-over).  With M = R0 - v w^T, rows 2..m of
// M are [-w_1 v_2, R22 - v_2 w_2^T]; their null vector is x = [1 - w_2^T u; w_1 u] with
// u = R22^{-1} v_2 (back substitution), and Z e1 is proportional to Q0^T x.  The residual of the
// zeroed column is w_1 (R22 u - v_2) + (rounding of x_1): bounded by O(m u ||R0||) ||x|| for a
// backward-stable substitution, whatever R22's condition; an exactly singular R22 (a non-finite or
// zero x) returns false and the caller falls back to the Givens chain (rqu_direction).
// Out (ok): uu = Q0^T x (unnormalised).  All threads; the caller's barrier publishes uu.
template <int NT, int MAXM>
__device__ __forceinline__ bool rqu_solve(int m, const double* v, double tau, const double* Rs, const double* Qs,
                                          double* wpart, double* xs, double* uu, volatile int* okflag,
                                          long long* pt = nullptr, long long* tc0 = nullptr,
                                          const double* FWg = nullptr, bool hasB = false) {
    using C = RQUCfg<NT, MAXM>;
    constexpr int RLD = C::RLD, RPL = C::RPL, NPART = C::NPART, RPP = MAXM / NPART;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    rqu_phase_w<NT, MAXM>(m, v, Rs, wpart);
    rqu_tick(pt, tc0, 17);
    if (warp == 0) {
        const unsigned rs0 = opaque_u32(rq_smem_u32(Rs));
        // rows p = RPL lane + e (consecutive): one lane's RPL columns per step of the back
        // substitution -- the lead lane solves its RPL x RPL triangle, one broadcast, then every
        // lane updates its rows for RPL columns (half / a quarter of the shuffle chain)
        double w[RPL], rhs[RPL], rinv[RPL], u[RPL];
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
            const int p = RPL * lane + e;
            double x = 0.0;
            if (p < m) {
#pragma unroll
                for (int q = 0; q < NPART; ++q) x += wpart[q * MAXM + p];
                x *= tau;
            }
            w[e] = x;
            const bool row = p >= 1 && p < m;
            rhs[e] = row ? v[p] : 0.0;
            rinv[e] = row ? fast_rcp(lds64(rs0 + 8u * (p * RLD + p))) : 0.0;  // (0 pivot: inf -> fallback)
            u[e] = 0.0;
        }
        // col[e][f] = R(RPL lane + e, RPL L + f) for the step's lane-block L (0 outside rows 1..m-1
        // and below the diagonal)
        double ca[RPL][RPL], cb[RPL][RPL];
        auto load = [&](int L, double (*col)[RPL]) {
#pragma unroll
            for (int e = 0; e < RPL; ++e)
#pragma unroll
                for (int f = 0; f < RPL; ++f) {
                    const int p = RPL * lane + e, c = RPL * L + f;
                    col[e][f] = lds64_if(p >= 1 && p < c && c < m, rs0 + 8u * (p * RLD + c));
                }
        };
        auto body = [&](int L, double (*col)[RPL]) {
            double ub[RPL];  // the lead's solve of its triangle (every lane computes its own; lane L's is used)
#pragma unroll
            for (int e = RPL - 1; e >= 0; --e) {
                double t = rhs[e];
#pragma unroll
                for (int f = e + 1; f < RPL; ++f) t = fma(-col[e][f], ub[f], t);
                ub[e] = t * rinv[e];
            }
#pragma unroll
            for (int f = 0; f < RPL; ++f) ub[f] = __shfl_sync(0xffffffffu, ub[f], L);
            if (lane == L) {
#pragma unroll
                for (int e = 0; e < RPL; ++e) u[e] = ub[e];
            }
#pragma unroll
            for (int e = 0; e < RPL; ++e)
#pragma unroll
                for (int f = 0; f < RPL; ++f) rhs[e] = fma(-col[e][f], ub[f], rhs[e]);
        };
        const int Ltop = (m - 1) / RPL;
        if (m >= 2) load(Ltop, ca);
        __syncwarp();  // (converged before the shuffle chain: a diverged warp takes BRA.DIV's slow shuffles)
        for (int L = Ltop; L >= 0; L -= 2) {
            if (L - 1 >= 0) load(L - 1, cb);
            body(L, ca);
            if (L - 1 < 0) break;
            if (L - 2 >= 0) load(L - 2, ca);
            body(L - 1, cb);
        }
        double dot = 0.0;
#pragma unroll
        for (int e = 0; e < RPL; ++e) dot = fma(w[e], u[e], dot);  // (u = 0 outside rows 1..m-1)
        dot = warp_sum(dot);
        const double w0 = __shfl_sync(0xffffffffu, w[0], 0);
        bool fin = true, nz = false;
        if (lane == 0) {
            const double x0 = 1.0 - dot;
            xs[0] = x0;
            fin = isfinite(x0);
            nz = x0 != 0.0;
        }
#pragma unroll
        for (int e = 0; e < RPL; ++e) {
            const int p = RPL * lane + e;
            if (p >= 1 && p < m) {
                const double xp = w0 * u[e];
                xs[p] = xp;
                fin = fin && isfinite(xp);
                nz = nz || xp != 0.0;
            }
        }
        const bool ok = __all_sync(0xffffffffu, fin) && __any_sync(0xffffffffu, nz);
        if (lane == 0) *okflag = ok ? 1 : 0;
    }
    __syncthreads();
    rqu_tick(pt, tc0, 18);
    const bool ok = *okflag != 0;
    if (ok) {  // uu = Q0^T x: column dots in NPART row parts
        const int c = tid % MAXM, part = tid / MAXM;
        if (part < NPART) {
            double s0 = 0.0, s1 = 0.0;
            if (c < m) {
                if (FWg) {  // Q0 = diag(W, 1) (hasB) or W, W row-major (ld MAXM) in global memory
                    const int f = hasB ? m - 1 : m;
                    const int p0 = part * RPP, p1 = min(p0 + RPP, f);
                    if (c < f) {
                        int p = p0;
                        for (; p + 3 < p1; p += 4) {  // (independent loads first)
                            const double q0 = ldcg(FWg + p * MAXM + c), q1 = ldcg(FWg + (p + 1) * MAXM + c);
                            const double q2 = ldcg(FWg + (p + 2) * MAXM + c), q3 = ldcg(FWg + (p + 3) * MAXM + c);
                            s0 = fma(q0, xs[p], s0);
                            s1 = fma(q1, xs[p + 1], s1);
                            s0 = fma(q2, xs[p + 2], s0);
                            s1 = fma(q3, xs[p + 3], s1);
                        }
                        for (; p < p1; ++p) s0 = fma(ldcg(FWg + p * MAXM + c), xs[p], s0);
                    } else if (part == (m - 1) / RPP) {
                        s0 = xs[m - 1];  // (hasB: the identity row / column)
                    }
                } else {
                    const int p0 = part * RPP, p1 = min(p0 + RPP, m);
                    int p = p0;
                    for (; p + 1 < p1; p += 2) {
                        s0 = fma(Qs[p * RLD + c], xs[p], s0);
                        s1 = fma(Qs[(p + 1) * RLD + c], xs[p + 1], s1);
                    }
                    if (p < p1) s0 = fma(Qs[p * RLD + c], xs[p], s0);
                }
            }
            wpart[part * MAXM + c] = s0 + s1;
        }
        __syncthreads();
        for (int c2 = tid; c2 < m; c2 += NT) {
            double z = 0.0;
#pragma unroll
            for (int q = 0; q < NPART; ++q) z += wpart[q * MAXM + c2];
            uu[c2] = z;
        }
    }
    rqu_tick(pt, tc0, 19);
    return ok;
}

// dst(p, c) = src[p MAXM + c] for p, c < f (upper: c >= p only), dst row-major with ld RLD; L2 reads,
// eight rows in flight per thread (a load-store loop serialised one L2 latency per element).
// All threads; no barrier.
template <int NT, int MAXM>
__device__ __forceinline__ void rqu_load_block(double* dst, const double* src, int f, bool upper) {
    constexpr int RLD = RQUCfg<NT, MAXM>::RLD, NP = NT / MAXM;
    const int c = threadIdx.x % MAXM, part = threadIdx.x / MAXM;
    if (part >= NP || c >= f) return;
    for (int p0 = part; p0 < f; p0 += 8 * NP) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int p = p0 + u * NP;
            v[u] = (p < f && (!upper || c >= p)) ? ldcg(src + p * MAXM + c) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int p = p0 + u * NP;
            if (p < f && (!upper || c >= p)) dst[p * RLD + c] = v[u];
        }
    }
}

// Q~ = G'^T G^T Q0 after the chain (QCONC off): one column per thread, all rotations in cs1 / cs2;
// uu = Q~(0,:)^T.  All threads; ends with a barrier.
template <int NT, int MAXM>
__device__ __forceinline__ void rqu_q_apply(int m, double* Qs, const double* cs1, const double* cs2, double* uu) {
    constexpr int RLD = RQUCfg<NT, MAXM>::RLD;
    const int c = threadIdx.x;
    if (c < m) {
        const unsigned qa = opaque_u32(rq_smem_u32(Qs)) + 8u * c;
        double carry = lds64(qa);
        for (int i = 0; i <= m - 2; ++i) {
            const double cc = cs1[2 * i], ss = cs1[2 * i + 1], yj = lds64(qa + 8u * (RLD * (i + 1)));
            sts64(qa + 8u * (RLD * i), fma(cc, carry, -ss * yj));
            carry = fma(ss, carry, cc * yj);
        }
        for (int j = m - 2; j >= 0; --j) {
            const double cc = cs2[2 * j], ss = cs2[2 * j + 1], yj = lds64(qa + 8u * (RLD * j));
            sts64(qa + 8u * (RLD * (j + 1)), fma(ss, yj, cc * carry));
            carry = fma(cc, yj, -ss * carry);
        }
        sts64(qa, carry);
        uu[c] = carry;
    }
    __syncthreads();
}

// Hand-over parts: FR = R~(1:m-1, 1:m-1) (upper triangle) and FW = (Q~ Z)(1:m-1, 1:m-1),
// Z = I - sig z z^T, row-major with ld MAXM (0-based ranges)
template <int NT, int MAXM>
__device__ __forceinline__ void rqu_handoff_R(int m, const double* Rs, double* FR) {
    constexpr int RLD = RQUCfg<NT, MAXM>::RLD, NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = 1 + warp; i < m; i += NW)
        for (int c = i + lane; c < m; c += 32) FR[(i - 1) * MAXM + (c - 1)] = Rs[i * RLD + c];
}
template <int NT, int MAXM>
__device__ __forceinline__ void rqu_handoff_W(int m, const double* Qs, const double* z, double sig, double* FW) {
    constexpr int RLD = RQUCfg<NT, MAXM>::RLD, NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = 1 + warp; i < m; i += NW) {
        double d = 0.0;
        for (int c = lane; c < m; c += 32) d = fma(Qs[i * RLD + c], z[c], d);
        d = warp_sum(d) * sig;
        for (int c = 1 + lane; c < m; c += 32) FW[(i - 1) * MAXM + (c - 1)] = fma(-d, z[c], Qs[i * RLD + c]);
    }
}

// Hand-over of step (j,k) to sweep j+1 (same k): FR = R~(1:m-1, 1:m-1) (upper triangle),
// FW = (Q~ Z)(1:m-1, 1:m-1) with Z = I - sig z z^T -- row-major, ld MAXM (0-based ranges).
template <int NT, int MAXM>
__device__ __forceinline__ void rqu_handoff(int m, const double* Rs, const double* Qs, const double* z, double sig,
                                            double* FR, double* FW) {
    constexpr int RLD = RQUCfg<NT, MAXM>::RLD, NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = 1 + warp; i < m; i += NW) {
        double d = 0.0;
        for (int c = lane; c < m; c += 32) d = fma(Qs[i * RLD + c], z[c], d);
        d = warp_sum(d) * sig;
        for (int c = 1 + lane; c < m; c += 32) {
            FW[(i - 1) * MAXM + (c - 1)] = fma(-d, z[c], Qs[i * RLD + c]);
            if (c >= i) FR[(i - 1) * MAXM + (c - 1)] = Rs[i * RLD + c];
        }
    }
}
