// chase.cuh -- K1: the generate phase of one group of q sweeps (PAPER.md:1843-1877,
// Alg. 3 "Generate phase of stage two", with the index corrections of DESIGN.md §3 / c8),
// run as a wavefront: CTA t owns sweep j = j1+t; step (j,k) starts once sweep j-1 has
// finished step k+2 (lag 3, SURVEY App. A.4 [V7][V11]), so up to q bulges are in flight.
//
// Per step (j,k), 1-based as in the paper:
//   jb = j + max(0,(k-1)r+1), i1 = j+kr+1, i2 = min(j+(k+1)r,n), i3 = min(j+(k+2)r,n),
//   i4 = j1 + 1 + max(0,(k+j-j1-q+1)r)                                 (corrected, c8)
//   (a) catch-up of Q_k^{j1..j-1} on A(.,jb) and B(.,i1+r-1)  (Alg. 3 lines 9-16) as ONE
//       mat-vec with the partial product U_k = Q_k^{j1}...Q_k^{j-1} (kept dense; K2 fused)
//   (b) Q_k^j reduces A(i1:i2,jb); B(i1:i2,i1:i2) <- Q^* B           (lines 17-19)
//   (c) RQ of B(i1:i2,i1:i2); Z_k^j from the first row of Q~          (lines 20-21)
//   (d) A(i4:i3,i1:i2) <- A Z ; B(i4:i2,i1:i2) <- B Z                   (lines 22-23)
//   U_k <- U_k Q_k^j and V_k <- V_k Z_k^j ("Form compact WY", kept as
//   dense w x w blocks for the DMMA chains); Z_k^j stored for the staircase (K4).
//
// Latency design: every input of a step is final once (j-1,k+2) is done, except column jb,
// which the same CTA produced in step k-1 and keeps in shared memory; so a step issues all
// of its loads at once (cp.async: U_k, V_k, the B block and catch-up column, and as much of
// the tall strip as fits), then runs a chain of one-reduction phases.  The RQ runs on
// NWR warps with the stacked [B_blk; P] rows in registers (one row per lane slot): each
// Householder stage broadcasts row i through shared memory and needs ONE reduction-free
// pass (all dot products with row i at once, the norm included), P accumulating
// H_m...H_2 so that P e1 = Q~^* e1 comes out without a second sweep.
#pragma once
#include "scalar.cuh"

#ifndef IDX
#define IDX(p, ld, i, j) (p)[((int64_t)(i) - 1) + ((int64_t)(j) - 1) * (int64_t)(ld)]
#endif

template <typename S>
struct ChaseArgs {
    int n, r, qp, j1, K, WP, LDB;
    S* A;
    int64_t lda;
    S* B;
    int64_t ldb;
    S* U;       // K dense blocks, row-major: (l, c) at U[k*WP*LDB + l*LDB + c]
    S* V;       // (rows/cols >= w_k are zero; U_k, V_k start as I_{w_k})
    S* Zr;      // (qp*K) records of (r+1): Z_k^j vector (m entries), sigma at [r]
    int* prog;  // qp counters: steps completed by each sweep of the group
    int strip_cap;  // strip rows (A then B) staged in shared memory per step
    long long* prof;  // optional: per-CTA cycle counts of the step phases (8 slots)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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

// RQ-based opposite reflector direction (readings c3/c4) on NWR warps.
// In: Cb (m x m, col-major, ld LDC) = B(i1:i2,i1:i2) after Q_k^j.  Out: uu[0..m) = Q~^* e1.
// Householder RQ, rows bottom-up (xGERQ2 order): stage i uses h = scal*(conj(row_i) - beta e_i)
// (h_i = 1), so every row's dot with h is scal*(g_l - beta*C[l,i]) with g_l = <row_l, row_i>:
// one pass per stage.  Rows of P (= H_m...H_2 accumulated, P e1 = Q~^* e1) ride along.
template <typename S, int MAXM, int NWR>
__device__ __forceinline__ void rq_direction(int m, const S* Cb, int LDC, S* bc, S* uu) {
    constexpr int ROWS = 32 * NWR;
    constexpr int RPL = (2 * MAXM + ROWS - 1) / ROWS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    S row[RPL][MAXM];
    int rho[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
        rho[s] = s * ROWS + warp * 32 + lane;
#pragma unroll
        for (int c = 0; c < MAXM; ++c) {
            S v = S(0.0);
            if (c < m) {
                if (rho[s] < m) v = Cb[rho[s] + c * LDC];
                else if (rho[s] < 2 * m) v = S((rho[s] - m) == c ? 1.0 : 0.0);
            }
            row[s][c] = v;
        }
    }
    int par = 0;
    for (int i = m - 1; i >= 1; --i) {
        // broadcast row i of C (its owner: slot i / ROWS, warp (i % ROWS) / 32, lane i % 32)
        S b[MAXM];
        if (NWR == 1) {
            const int src = i & 31, sl = i / ROWS;
#pragma unroll
            for (int c = 0; c < MAXM; ++c) {
                S v = row[0][c];
#pragma unroll
                for (int s = 1; s < RPL; ++s)
                    if (sl == s) v = row[s][c];
                b[c] = shfl_idx(v, src);
            }
        } else {
            S* bs = bc + par * (MAXM + 1);
#pragma unroll
            for (int s = 0; s < RPL; ++s)
                if (rho[s] == i) {
#pragma unroll
                    for (int c = 0; c < MAXM; ++c) bs[c] = row[s][c];
                }
            named_bar(1, 32 * NWR);
#pragma unroll
            for (int c = 0; c < MAXM; ++c) b[c] = bs[c];
        }
        // scalars of stage i (every lane redundantly): alpha = conj(C[i,i]), x = conj(C[i,0:i))
        double n4[4] = {0.0, 0.0, 0.0, 0.0};
        S bi = S(0.0);
#pragma unroll
        for (int c = 0; c < MAXM; ++c) {
            if (c < i) n4[c & 3] += abs2(b[c]);
            if (c == i) bi = b[c];
        }
        const double nx = (n4[0] + n4[1]) + (n4[2] + n4[3]);
        const S alpha = conjv(bi);
        if (!(nx == 0.0 && im(alpha) == 0.0)) {
            const double nrm = sqrt(abs2(alpha) + nx);
            const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
            // tau |scal|^2 = ((beta-alpha)/beta) / |alpha-beta|^2 = -1 / (beta conj(alpha-beta))
            const S ts = -recip(beta * conjv(alpha - S(beta)));
            // rows >= i of C are finished (never read again), so they may be updated too:
            // every lane runs the same straight-line code (no divergence)
#pragma unroll
            for (int s = 0; s < RPL; ++s) {
                S g4[4] = {S(0.0), S(0.0), S(0.0), S(0.0)};
                S cli = S(0.0);
#pragma unroll
                for (int c = 0; c < MAXM; ++c) {
                    const S bc_ = (c <= i) ? b[c] : S(0.0);
                    g4[c & 3] = fma_s(row[s][c], conjv(bc_), g4[c & 3]);
                    if (c == i) cli = row[s][c];
                }
                const S coef = ts * (((g4[0] + g4[1]) + (g4[2] + g4[3])) - beta * cli);
#pragma unroll
                for (int c = 0; c < MAXM; ++c) {
                    const S d = (c < i) ? b[c] : ((c == i) ? b[c] - S(beta) : S(0.0));
                    row[s][c] -= coef * d;
                }
            }
        }
        par ^= 1;
    }
#pragma unroll
    for (int s = 0; s < RPL; ++s)
        if (rho[s] >= m && rho[s] < 2 * m) uu[rho[s] - m] = row[s][0];
}

template <typename S>
__host__ __device__ inline size_t chase_smem_elems(int r, int w, int strip_cap) {
    // xcol (2 buffers), ys, tx/ty, U, V (w x (w+1)), Cb r x (r+1), vectors, strip
    return 2 * (size_t)(w + r + 8) + (size_t)(w + r + 8) + 2 * (size_t)(w + r + 8) +
           2 * (size_t)w * (w + 1) + (size_t)r * (r + 1) + 4 * (size_t)(r + 8) + 2 * (size_t)(r + 9) +
           16 + (size_t)strip_cap * (r + 1);
}

template <typename S, int NT, int MAXM, int NWR>
__global__ void __launch_bounds__(NT, 1) chase_kernel(ChaseArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    S* sm = reinterpret_cast<S*>(smraw);
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K, LDB = a.LDB;
    const int w = qp + r - 1;
    const int LU = (w & 1) ? w : w + 1;  // odd ld of the U/V copies (conflict-free rows)
    const int SLD = r + 1;               // odd-ish ld of the strip rows
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    const int XL = w + r + 8;
    S* xc[2] = {sm, sm + XL};  // column jb of this step / of the next step
    S* ys = sm + 2 * XL;
    S* tx = ys + XL;
    S* ty = tx + XL;
    S* Ub = ty + XL;           // U_k rows/cols [0, t+m)
    S* Vb = Ub + (size_t)w * LU;
    S* Cb = Vb + (size_t)w * LU;  // r x (r+1)
    S* vq = Cb + (size_t)r * (r + 1);
    S* vz = vq + (r + 8);
    S* uu = vz + (r + 8);
    S* xs2 = uu + (r + 8);     // spare
    S* bc = xs2 + (r + 8);     // 2 x (r+9) RQ broadcast rows
    S* scal = bc + 2 * (r + 9);  // 16 scalars
    S* strip = scal + 16;      // strip_cap rows x (r+1) (row-major)
    const int LDC = r + 1;
    const int t = blockIdx.x;
    if (t >= qp) return;
    const int j = j1 + t;
    const int kcount = min(K, 2 + (n - j - 1) / r);
    const int kprev = (t > 0) ? min(K, 2 + (n - j) / r) : 0;
    int cur = 0;
    long long pt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc = clock64();
#define K1_TICK(slot)                         \
    do {                                      \
        const long long now_ = clock64();     \
        pt[slot] += now_ - tc;                \
        tc = now_;                            \
    } while (0)
    for (int k = 0; k < kcount; ++k) {
        K1_TICK(7);
        if (t > 0) {
            if (tid == 0) {
                const int need = min(k + 3, kprev);
                while (ld_acquire(&a.prog[t - 1]) < need) {
                }
            }
            __syncthreads();
        }
        K1_TICK(0);
        const int jb = j + max(0, (k - 1) * r + 1);
        const int i1 = j + k * r + 1;
        const int i2 = min(j + (k + 1) * r, n);
        const int i3 = min(j + (k + 2) * r, n);
        const int i4 = j1 + 1 + max(0, (k + t - qp + 1) * r);
        const int b0 = j1 + k * r + 1;
        const int m = i2 - i1 + 1;
        const int L = (t > 0) ? min(j - 1 + (k + 1) * r, n) - b0 + 1 : 0;
        const int nx = i2 - b0 + 1;
        const int cB = i1 + r - 1;  // == i2 when it exists
        const bool hasB = cB <= n;
        const int tm = t + max(m, 0);  // U/V square needed: [0, t+m)
        S* Uk = a.U + (int64_t)k * a.WP * LDB;
        S* Vk = a.V + (int64_t)k * a.WP * LDB;
        S* xcol = xc[cur];
        S* xnext = xc[cur ^ 1];
        const int nA = max(0, i3 - i4 + 1), nBs = max(0, i1 - i4);  // strip rows (B: above block)
        const int stA = min(nA, a.strip_cap), stB = min(nBs, a.strip_cap - stA);
        const bool gen = (m >= 2) && jb <= n && nx > 0;
        // ---- (S1) all loads of the step at once ------------------------------------------
        if (jb <= n && nx > 0) {
            if (k == 0)
                for (int i = tid; i < nx; i += NT) k1_ld(&xcol[i], &IDX(a.A, a.lda, b0 + i, jb));
            if (hasB)
                for (int i = tid; i < nx; i += NT) k1_ld(&ys[i], &IDX(a.B, a.ldb, b0 + i, cB));
            if (t > 0)
                for (int e = tid; e < tm * tm; e += NT) {
                    const int l = e / tm, c = e % tm;
                    k1_ld(&Ub[l * LU + c], &Uk[(int64_t)l * LDB + c]);
                }
            if (gen) {
                if (t > 0)
                    for (int e = tid; e < tm * tm; e += NT) {
                        const int l = e / tm, c = e % tm;
                        k1_ld(&Vb[l * LU + c], &Vk[(int64_t)l * LDB + c]);
                    }
                for (int e = tid; e < m * m; e += NT) {
                    const int ii = e % m, cc = e / m;
                    k1_ld(&Cb[ii + cc * LDC], &IDX(a.B, a.ldb, i1 + ii, i1 + cc));
                }
                for (int e = tid; e < (stA + stB) * m; e += NT) {
                    const int rr = e % (stA + stB), cc = e / (stA + stB);
                    const S* src = rr < stA ? &IDX(a.A, a.lda, i4 + rr, i1 + cc)
                                            : &IDX(a.B, a.ldb, i4 + (rr - stA), i1 + cc);
                    k1_ld(&strip[rr * SLD + cc], src);
                }
            }
        }
        if (t == 0 && gen)
            for (int e = tid; e < tm * tm; e += NT) {
                const int l = e / tm, c = e % tm;
                Ub[l * LU + c] = S(l == c ? 1.0 : 0.0);
                Vb[l * LU + c] = S(l == c ? 1.0 : 0.0);
            }
        k1_commit_wait();
        __syncthreads();
        K1_TICK(1);
        if (jb <= n && nx > 0) {
            // ---- (S2) catch-up: x(0:L) <- U^* x(0:L), same for the B column --------------------
            if (L >= 1) {
                for (int o = tid; o < L; o += NT) {
                    S s0 = S(0.0), s1 = S(0.0), y0 = S(0.0), y1 = S(0.0);
                    int l = 0;
                    for (; l + 1 < L; l += 2) {
                        const S u0 = Ub[l * LU + o], u1 = Ub[(l + 1) * LU + o];
                        s0 += conj_mul(u0, xcol[l]);
                        s1 += conj_mul(u1, xcol[l + 1]);
                        if (hasB) {
                            y0 += conj_mul(u0, ys[l]);
                            y1 += conj_mul(u1, ys[l + 1]);
                        }
                    }
                    if (l < L) {
                        const S u0 = Ub[l * LU + o];
                        s0 += conj_mul(u0, xcol[l]);
                        if (hasB) y0 += conj_mul(u0, ys[l]);
                    }
                    tx[o] = s0 + s1;
                    ty[o] = y0 + y1;
                }
                __syncthreads();
                for (int i = tid; i < L; i += NT) {
                    xcol[i] = tx[i];
                    if (hasB) ys[i] = ty[i];
                }
                if (hasB && gen) {  // catch-up column also feeds the block and the B strip
                    for (int i = tid; i < t && i < L; i += NT) {
                        const int rr = (b0 + i) - i4;  // strip row of B row b0+i (>= 0)
                        if (rr >= 0 && rr < stB) strip[(stA + rr) * SLD + (m - 1)] = ty[i];
                    }
                    for (int i = tid; i < m; i += NT)
                        if (t + i < L) Cb[i + (m - 1) * LDC] = ty[t + i];
                }
                __syncthreads();
            }
            if (hasB && gen && !(L >= 1))
                for (int i = tid; i < m; i += NT) Cb[i + (m - 1) * LDC] = ys[t + i];
            if (!gen) {  // catch-up only (no reflector at this step; Alg. 2 has m >= 2)
                for (int i = tid; i < L; i += NT) IDX(a.A, a.lda, b0 + i, jb) = xcol[i];
                if (hasB)
                    for (int i = tid; i < L; i += NT) IDX(a.B, a.ldb, b0 + i, cB) = ys[i];
            } else {
                K1_TICK(2);
                // ---- (S3) left reflector Q_k^j on A(i1:i2,jb) ----------------------------------
                if (warp == 0) {
                    S tau;
                    double beta;
                    warp_larfg(m, xcol + t, vq, tau, beta);
                    if (lane == 0) {
                        scal[0] = tau;
                        scal[1] = S(beta);
                    }
                }
                __syncthreads();
                const S tau = scal[0];
                {
                    const S betaS = scal[1];
                    for (int i = tid; i < nx; i += NT) {
                        const S val = (i < t) ? xcol[i] : ((i == t) ? betaS : S(0.0));  // exact zeros (c5)
                        IDX(a.A, a.lda, b0 + i, jb) = val;
                    }
                    if (hasB)
                        for (int i = tid; i < t; i += NT) IDX(a.B, a.ldb, b0 + i, cB) = ys[i];
                }
                // ---- (S4) B block <- Q^* B block ---------------------------------------------------
                if (!is_zero(tau)) {
                    const S ctau = conjv(tau);
                    for (int c = warp; c < m; c += NW) {
                        S s = S(0.0);
                        for (int i = lane; i < m; i += 32) s += conj_mul(vq[i], Cb[i + c * LDC]);
                        s = warp_sum(s) * ctau;
                        for (int i = lane; i < m; i += 32) Cb[i + c * LDC] -= vq[i] * s;
                    }
                }
                __syncthreads();
                K1_TICK(3);
                // ---- (S5) RQ on warps [0,NWR) || U_k <- U_k Q_k^j on the other warps --------------
                if (warp < NWR) {
                    rq_direction<S, MAXM, NWR>(m, Cb, LDC, bc, uu);
                    if (NWR == 1) __syncwarp();
                    else named_bar(1, 32 * NWR);
                    K1_TICK(6);
                    if (warp == 0) {
                        S sig;
                        double b2;
                        warp_larfg(m, uu, vz, sig, b2);
                        if (lane == 0) scal[2] = sig;
                    }
                } else if (!is_zero(tau)) {
                    const int nth = NT - 32 * NWR, me = tid - 32 * NWR;
                    for (int l = me; l < tm; l += nth) {
                        S s = S(0.0);
                        for (int c = 0; c < m; ++c) s = fma_s(Ub[l * LU + t + c], vq[c], s);
                        s = s * tau;
                        for (int c = 0; c < m; ++c) {
                            const S v = Ub[l * LU + t + c] - s * conjv(vq[c]);
                            Ub[l * LU + t + c] = v;
                            Uk[(int64_t)l * LDB + t + c] = v;
                        }
                    }
                }
                __syncthreads();
                K1_TICK(4);
                const S sig = scal[2];
                // ---- (S6) right reflector Z_k^j on the band, V_k update, next column --------------
                const int nBb = max(0, i2 - i4 + 1);  // B rows i4..i2 (block rows i1..i2 from Cb)
                const int bn = b0 + r;                 // first row of the next step's column
                for (int e = tid; e < nA + nBb; e += NT) {
                    const bool isA = e < nA;
                    const int row = isA ? i4 + e : i4 + (e - nA);
                    S v[MAXM];
                    S* gp = isA ? &IDX(a.A, a.lda, row, i1) : &IDX(a.B, a.ldb, row, i1);
                    const int64_t ld = isA ? a.lda : a.ldb;
                    if (isA && e < stA) {
#pragma unroll
                        for (int c = 0; c < MAXM; ++c)
                            if (c < m) v[c] = strip[e * SLD + c];
                    } else if (!isA && row >= i1) {
#pragma unroll
                        for (int c = 0; c < MAXM; ++c)
                            if (c < m) v[c] = Cb[(row - i1) + c * LDC];
                    } else if (!isA && (e - nA) < stB) {
#pragma unroll
                        for (int c = 0; c < MAXM; ++c)
                            if (c < m) v[c] = strip[(stA + e - nA) * SLD + c];
                    } else {
#pragma unroll
                        for (int c = 0; c < MAXM; ++c)
                            if (c < m) v[c] = ldcg(gp + c * ld);
                    }
                    if (!is_zero(sig)) {
                        S s0 = S(0.0), s1 = S(0.0);
#pragma unroll
                        for (int c = 0; c < MAXM; ++c)
                            if (c < m) {
                                if (c & 1) s1 = fma_s(v[c], vz[c], s1);
                                else s0 = fma_s(v[c], vz[c], s0);
                            }
                        const S s = (s0 + s1) * sig;
#pragma unroll
                        for (int c = 0; c < MAXM; ++c)
                            if (c < m) v[c] -= s * conjv(vz[c]);
                    }
                    if (!isA && row > i1) v[0] = S(0.0);  // B(i1+1:i2,i1) = 0 (reading c5)
#pragma unroll
                    for (int c = 0; c < MAXM; ++c)
                        if (c < m) gp[c * ld] = v[c];
                    if (isA && row >= bn) xnext[row - bn] = v[0];  // column jb of step k+1
                }
                if (!is_zero(sig)) {
                    for (int l = tid; l < tm; l += NT) {  // V_k <- V_k Z_k^j
                        S s = S(0.0);
                        for (int c = 0; c < m; ++c) s = fma_s(Vb[l * LU + t + c], vz[c], s);
                        s = s * sig;
                        for (int c = 0; c < m; ++c) Vk[(int64_t)l * LDB + t + c] = Vb[l * LU + t + c] - s * conjv(vz[c]);
                    }
                }
                S* zr = a.Zr + ((int64_t)t * K + k) * (r + 1);
                for (int c = tid; c < m; c += NT) zr[c] = vz[c];
                if (tid == 0) zr[r] = sig;
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
        if (tid == 0) {
            __threadfence();
            st_release(&a.prog[t], k + 1);
        }
        cur ^= 1;
    }
    if (a.prof && tid == 0)
        for (int i = 0; i < 8; ++i) atomicAdd((unsigned long long*)&a.prof[i], (unsigned long long)pt[i]);
#undef K1_TICK
}
