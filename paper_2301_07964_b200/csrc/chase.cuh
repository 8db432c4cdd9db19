// chase.cuh -- K1: the generate phase of one group of q sweeps (PAPER.md:1843-1877,
// Alg. 3 "Generate phase of stage two", with the index corrections of DESIGN.md §3 / c8),
// run as a wavefront: CTA b owns sweeps t = b, b+P, ...; step (j,k) starts once sweep
// j-1 has finished step k+2 (lag 3, SURVEY App. A.4 [V7][V11]).
//
// Per step (j,k), 1-based as in the paper:
//   jb = j + max(0,(k-1)r+1), i1 = j+kr+1, i2 = min(j+(k+1)r,n), i3 = min(j+(k+2)r,n),
//   i4 = j1 + 1 + max(0,(k+j-j1-q+1)r)                                 (corrected, c8)
//   (a) catch-up of Q_k^{j1..j-1} on A(.,jb) and B(.,i1+r-1)  (Alg. 3 lines 9-16) -- one
//       mat-vec with the partial product U_k = Q_k^{j1}...Q_k^{j-1} (kept dense, K2 fused)
//   (b) Q_k^j reduces A(i1:i2,jb); B(i1:i2,i1:i2) <- Q^* B           (lines 17-19)
//   (c) RQ of B(i1:i2,i1:i2); Z_k^j from the first row of Q~          (lines 20-21)
//   (d) A(i4:i3,i1:i2) <- A Z ; B(i4:i2,i1:i2) <- B Z                   (lines 22-23)
//   U_k <- U_k Q_k^j and V_k <- V_k Z_k^j on local columns t..t+m-1 (PAPER.md:1894/1903,
//   "Form compact WY", kept as dense w x w blocks); Z_k^j stored for the staircase (K4).
#pragma once
#include "scalar.cuh"

#define IDX(p, ld, i, j) (p)[((int64_t)(i) - 1) + ((int64_t)(j) - 1) * (int64_t)(ld)]

template <typename S>
struct ChaseArgs {
    int n, r, qp, j1, K, WP, LDB;
    S* A;
    int64_t lda;
    S* B;
    int64_t ldb;
    S* U;     // K dense blocks, row-major: (l, c) at U[k*WP*LDB + l*LDB + c]
    S* V;     // (rows/cols >= w_k are zero; U_k, V_k start as I_{w_k})
    S* Zr;    // (qp*K) records of (r+1): Z_k^j vector (m entries), sigma at [r]
    int* prog;  // qp counters: steps completed by each sweep of the group
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

template <typename S>
__host__ __device__ inline size_t chase_smem_elems(int r, int w) {
    return 4 * (size_t)(w + r) + 5 * (size_t)r + 1 + (size_t)r * (r + 1) + 8;
}

template <typename S, int NT>
__global__ void __launch_bounds__(NT, 1) chase_kernel(ChaseArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    S* sm = reinterpret_cast<S*>(smraw);
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K, LDB = a.LDB;
    const int w = qp + r - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NT / 32;
    S* xs = sm;             // w + r : column jb, rows b0..
    S* ys = xs + (w + r);   // w + r : column i1+r-1 of B, rows b0..
    S* tx = ys + (w + r);   // w + r : mat-vec outputs
    S* ty = tx + (w + r);   // w + r
    S* vq = ty + (w + r);   // r     : left reflector v
    S* vz = vq + r;         // r     : right reflector w
    S* uu = vz + r;         // r     : Q~^* e1
    S* taus = uu + r;       // r     : RQ taus
    S* hv = taus + r;       // r + 1 : RQ reflector
    S* scal = hv + (r + 1); // 8     : broadcast scalars
    S* Cb = scal + 8;       // r x (r+1)
    const int LDC = r + 1;

    for (int t = blockIdx.x; t < qp; t += gridDim.x) {
        const int j = j1 + t;
        const int kcount = min(K, 2 + (n - j - 1) / r);
        const int kprev = (t > 0) ? min(K, 2 + (n - j) / r) : 0;
        for (int k = 0; k < kcount; ++k) {
            if (t > 0) {  // wavefront dependency: sweep j-1 finished step k+2 (lag 3)
                if (tid == 0) {
                    const int need = min(k + 3, kprev);
                    while (ld_acquire(&a.prog[t - 1]) < need) __nanosleep(20);
                }
                __syncthreads();
            }
            const int jb = j + max(0, (k - 1) * r + 1);
            const int i1 = j + k * r + 1;
            const int i2 = min(j + (k + 1) * r, n);
            const int i3 = min(j + (k + 2) * r, n);
            const int i4 = j1 + 1 + max(0, (k + t - qp + 1) * r);
            const int b0 = j1 + k * r + 1;
            const int m = i2 - i1 + 1;
            const int wk = min(w, n - b0 + 1);
            S* Uk = a.U + (int64_t)k * a.WP * LDB;
            S* Vk = a.V + (int64_t)k * a.WP * LDB;
            const int L = (t > 0) ? min(j - 1 + (k + 1) * r, n) - b0 + 1 : 0;
            const int nx = i2 - b0 + 1;
            const int cB = i1 + r - 1;  // == i2 when it exists
            const bool hasB = cB <= n;
            if (jb <= n && nx > 0) {
                // ---- (a) load + catch-up --------------------------------------------------
                for (int i = tid; i < nx; i += NT) xs[i] = ldcg(&IDX(a.A, a.lda, b0 + i, jb));
                if (hasB)
                    for (int i = tid; i < nx; i += NT) ys[i] = ldcg(&IDX(a.B, a.ldb, b0 + i, cB));
                __syncthreads();
                if (L >= 1) {
                    for (int o = warp; o < L; o += NW) {
                        S s = S(0.0), s2 = S(0.0);
                        for (int l = lane; l < L; l += 32) {
                            const S u = ldcg(&Uk[(int64_t)l * LDB + o]);
                            s += conj_mul(u, xs[l]);
                            if (hasB) s2 += conj_mul(u, ys[l]);
                        }
                        s = warp_sum(s);
                        if (hasB) s2 = warp_sum(s2);
                        if (lane == 0) {
                            tx[o] = s;
                            ty[o] = s2;
                        }
                    }
                    __syncthreads();
                    for (int i = tid; i < L; i += NT) {
                        xs[i] = tx[i];
                        if (hasB) ys[i] = ty[i];
                    }
                    __syncthreads();
                }
                if (m < 2) {  // catch-up only (no reflector at this step; Alg. 2 has m >= 2)
                    for (int i = tid; i < L; i += NT) IDX(a.A, a.lda, b0 + i, jb) = xs[i];
                    if (hasB)
                        for (int i = tid; i < L; i += NT) IDX(a.B, a.ldb, b0 + i, cB) = ys[i];
                } else {
                    // ---- (b) left reflector Q_k^j on A(i1:i2,jb) ------------------------------
                    if (warp == 0) {
                        S tau;
                        double beta;
                        warp_larfg(m, xs + t, vq, tau, beta);
                        if (lane == 0) {
                            scal[0] = tau;
                            scal[1] = S(beta);
                        }
                    }
                    __syncthreads();
                    const S tau = scal[0];
                    const S betaS = scal[1];
                    for (int i = tid; i < nx; i += NT) {
                        const S val = (i < t) ? xs[i] : ((i == t) ? betaS : S(0.0));  // exact zeros (c5)
                        IDX(a.A, a.lda, b0 + i, jb) = val;
                    }
                    if (hasB)
                        for (int i = tid; i < t; i += NT) IDX(a.B, a.ldb, b0 + i, cB) = ys[i];
                    for (int e = tid; e < m * m; e += NT) {
                        const int ii = e % m, cc = e / m;
                        Cb[ii + cc * LDC] = (hasB && cc == m - 1) ? ys[t + ii]
                                                                  : ldcg(&IDX(a.B, a.ldb, i1 + ii, i1 + cc));
                    }
                    __syncthreads();
                    if (!is_zero(tau)) {
                        const S ctau = conjv(tau);
                        for (int c = warp; c < m; c += NW) {
                            S s = S(0.0);
                            for (int i = lane; i < m; i += 32) s += conj_mul(vq[i], Cb[i + c * LDC]);
                            s = warp_sum(s) * ctau;
                            for (int i = lane; i < m; i += 32) Cb[i + c * LDC] -= vq[i] * s;
                        }
                        for (int l = tid; l < wk; l += NT) {  // U_k <- U_k Q_k^j
                            S s = S(0.0);
                            for (int c = 0; c < m; ++c) s += ldcg(&Uk[(int64_t)l * LDB + t + c]) * vq[c];
                            s = s * tau;
                            for (int c = 0; c < m; ++c) {
                                S* p = &Uk[(int64_t)l * LDB + t + c];
                                *p = ldcg(p) - s * conjv(vq[c]);
                            }
                        }
                    }
                    __syncthreads();
                    for (int e = tid; e < m * m; e += NT) {
                        const int ii = e % m, cc = e / m;
                        IDX(a.B, a.ldb, i1 + ii, i1 + cc) = Cb[ii + cc * LDC];
                    }
                    // ---- (c) RQ of the block (rows bottom-up, xGERQ2 order; reading c4) -------
                    for (int i = m - 1; i >= 1; --i) {
                        if (warp == 0) {
                            double s = 0.0;
                            for (int c = lane; c < i; c += 32) s += abs2(Cb[i + c * LDC]);
                            s = warp_sum(s);
                            const S alpha = conjv(Cb[i + i * LDC]);
                            S ti, sc;
                            if (s == 0.0 && im(alpha) == 0.0) {
                                ti = S(0.0);
                                sc = S(0.0);
                            } else {
                                const double nrm = sqrt(abs2(alpha) + s);
                                const double bi = (re(alpha) >= 0.0) ? -nrm : nrm;
                                ti = divr(S(bi) - alpha, bi);
                                sc = recip(alpha - S(bi));
                            }
                            for (int c = lane; c < i; c += 32) hv[c] = conjv(Cb[i + c * LDC]) * sc;
                            if (lane == 0) {
                                hv[i] = S(1.0);
                                taus[i] = ti;
                            }
                        }
                        __syncthreads();
                        const S ti = taus[i];
                        if (!is_zero(ti)) {
                            for (int l = warp; l < i; l += NW) {
                                S s = S(0.0);
                                for (int c = lane; c <= i; c += 32) s += Cb[l + c * LDC] * hv[c];
                                s = warp_sum(s) * ti;
                                for (int c = lane; c <= i; c += 32) Cb[l + c * LDC] -= s * conjv(hv[c]);
                            }
                        }
                        for (int c = tid; c < i; c += NT) Cb[i + c * LDC] = hv[c];
                        __syncthreads();
                    }
                    // u = H_m ... H_2 e1 = Q~^* e1 = conj(Q~(1,:))^T  (reading c3)
                    if (warp == 0) {
                        for (int c = lane; c < m; c += 32) uu[c] = S(c == 0 ? 1.0 : 0.0);
                        __syncwarp();
                        for (int i = 1; i < m; ++i) {
                            const S ti = taus[i];
                            if (is_zero(ti)) continue;
                            S s = S(0.0);
                            for (int c = lane; c <= i; c += 32) {
                                const S h = (c == i) ? S(1.0) : Cb[i + c * LDC];
                                s += conj_mul(h, uu[c]);
                            }
                            s = warp_sum(s) * ti;
                            for (int c = lane; c <= i; c += 32) {
                                const S h = (c == i) ? S(1.0) : Cb[i + c * LDC];
                                uu[c] -= h * s;
                            }
                            __syncwarp();
                        }
                        S sig;
                        double b2;
                        warp_larfg(m, uu, vz, sig, b2);
                        if (lane == 0) scal[2] = sig;
                    }
                    __syncthreads();
                    const S sig = scal[2];
                    // ---- (d) right reflector on the band: A(i4:i3,i1:i2), B(i4:i2,i1:i2) --------
                    const int nA = max(0, i3 - i4 + 1), nB = max(0, i2 - i4 + 1);
                    for (int e = tid; e < nA + nB; e += NT) {
                        const bool isA = e < nA;
                        S* M = isA ? a.A : a.B;
                        const int64_t ld = isA ? a.lda : a.ldb;
                        const int row = i4 + (isA ? e : e - nA);
                        S* p = &IDX(M, ld, row, i1);
                        if (!is_zero(sig)) {
                            S s = S(0.0);
                            for (int c = 0; c < m; ++c) s += ldcg(p + c * ld) * vz[c];
                            s = s * sig;
                            for (int c = 0; c < m; ++c) p[c * ld] = ldcg(p + c * ld) - s * conjv(vz[c]);
                        }
                        if (!isA && row > i1) p[0] = S(0.0);  // B(i1+1:i2,i1) = 0 (reading c5)
                    }
                    if (!is_zero(sig)) {
                        for (int l = tid; l < wk; l += NT) {  // V_k <- V_k Z_k^j
                            S s = S(0.0);
                            for (int c = 0; c < m; ++c) s += ldcg(&Vk[(int64_t)l * LDB + t + c]) * vz[c];
                            s = s * sig;
                            for (int c = 0; c < m; ++c) {
                                S* p = &Vk[(int64_t)l * LDB + t + c];
                                *p = ldcg(p) - s * conjv(vz[c]);
                            }
                        }
                    }
                    S* zr = a.Zr + ((int64_t)t * K + k) * (r + 1);
                    for (int c = tid; c < m; c += NT) zr[c] = vz[c];
                    if (tid == 0) zr[r] = sig;
                }
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                st_release(&a.prog[t], k + 1);
            }
        }
    }
}
