// chain.cuh -- K3/K4: the apply phase of one group (Alg. 4
// "Application phase of stage two", corrected per DESIGN.md §3 / c8), as fused
// descending-k chains:
//
//   row chain  (right updates, row-independent):  M(rows, C_k) <- M(rows, C_k) X_k,
//              k = K-1 ... 0, X_k = V_k (A, B, Z) or U_k (Q).  One CTA owns a tile of
//              BM rows and streams the windows right-to-left, keeping the q-1 overlap
//              columns of consecutive windows on chip (each entry read/written once per
//              group).  For A and B the tile rows split per window into the dense block
//              region (rows <= i5), the staircase (rows i5s..i4, reflector by reflector,
//              Alg. 4 lines 4-9), and untouched rows.
//   col chain  (left updates, column-independent): M(R_k, cols) <- U_k^* M(R_k, cols)
//              for columns > i5 (A) / > i6 (B), Alg. 4 lines 16-25.
//
// Windows: C_k = R_k = [j1+kr+1, min(j1+q-1+(k+1)r, n)], width wk <= w = q+r-1.
#pragma once
#include "scalar.cuh"
#include "chase.cuh"

template <typename S>
struct ChainArgs {
    int n, r, qp, j1, K, W;
    S* M0;
    int64_t ld0;
    S* M1;
    int64_t ld1;
    const S* Blk0;  // blocks for M0 (U or V)
    const S* Blk1;  // blocks for M1
    const S* Zr;    // staircase reflectors (row chain on A/B)
    int kcnt_base;  // unused (reserved)
};

__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------------------
// Row chain.  AB = true: A/B right updates (masks + staircase).  AB = false: Q or Z.
// grid.x = row tiles, grid.y = matrix (0 -> M0/Blk0, 1 -> M1/Blk1).
// smem: X [BM x W] (column slot = global col mod W, ld BM), Y [BM x W], Vs [W x W].
template <typename S, int BM, int NT, bool AB>
__global__ void __launch_bounds__(NT) row_chain_kernel(ChainArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    S* X = reinterpret_cast<S*>(smraw);
    const int W = a.W;
    S* Y = X + (size_t)BM * W;
    S* Vs = Y + (size_t)BM * W;
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K;
    const int w = qp + r - 1;
    S* M = blockIdx.y == 0 ? a.M0 : a.M1;
    const int64_t ld = blockIdx.y == 0 ? a.ld0 : a.ld1;
    const S* Blk = blockIdx.y == 0 ? a.Blk0 : a.Blk1;
    const int R0 = blockIdx.x * BM + 1;
    if (R0 > n) return;
    const int nr = min(BM, n - R0 + 1);
    const int tid = threadIdx.x;
    // rows touched by window k in the apply phase (A/B): block rows <= i5b(k), staircase
    // rows <= max_t i4(k,t) = j1 + k r (q >= 2)
    auto rowmax = [&](int k) {
        return (qp >= 2) ? j1 + imax(0, k * r) : j1 + imax(0, (k - qp + 1) * r);
    };
    if (AB && rowmax(K - 1) < R0) return;
    int pc0 = 0, pwk = 0;
    for (int k = K - 1; k >= 0; --k) {
        if (AB && rowmax(k) < R0) break;
        const int c0 = j1 + k * r + 1;
        const int wk = min(w, n - c0 + 1);
        // write out columns leaving the window, then load the entering ones
        if (pwk > 0) {
            for (int e = tid; e < nr * (pc0 + pwk - (c0 + wk)); e += NT) {
                const int i = e % nr, c = c0 + wk + e / nr;
                IDX(M, ld, R0 + i, c) = X[i + (c % W) * BM];
            }
            __syncthreads();
        }
        const int cin1 = (pwk > 0) ? pc0 : c0 + wk;  // entering columns [c0, cin1)
        for (int e = tid; e < nr * (cin1 - c0); e += NT) {
            const int i = e % nr, c = c0 + e / nr;
            X[i + (c % W) * BM] = IDX(M, ld, R0 + i, c);
        }
        const S* Bk = Blk + (int64_t)k * W * W;
        for (int e = tid; e < wk * wk; e += NT) {
            const int l = e % wk, c = e / wk;
            Vs[l + c * W] = Bk[l + (int64_t)c * W];
        }
        __syncthreads();
        // Y = X(:, window) * Vs
        const int i5b = j1 + imax(0, (k - qp + 1) * r);
        for (int e = tid; e < nr * wk; e += NT) {
            const int i = e % nr, c = e / nr;
            S acc = S(0.0);
            for (int l = 0; l < wk; ++l) acc = fma_s(X[i + ((c0 + l) % W) * BM], Vs[l + c * W], acc);
            Y[i + c * BM] = acc;
        }
        __syncthreads();
        for (int e = tid; e < nr * wk; e += NT) {
            const int i = e % nr, c = e / nr;
            if (!AB || R0 + i <= i5b) X[i + ((c0 + c) % W) * BM] = Y[i + c * BM];
        }
        __syncthreads();
        if (AB) {  // staircase (Alg. 4 lines 4-9, corrected): rows i5s..i4(k,j), j = j1+1..j1+q-1
            const int i5s = j1 + 1 + imax(0, (k - qp + 1) * r);
            const int rlo = imax(i5s, R0), rhi = min(rowmax(k), R0 + nr - 1);
            if (rlo <= rhi) {
                for (int i = tid; i < nr; i += NT) {  // one thread per row: sequential in t
                    const int row = R0 + i;
                    if (row < rlo || row > rhi) continue;
                    for (int t = 1; t < qp; ++t) {
                        const int j = j1 + t;
                        const int i1 = j + k * r + 1, i2 = min(j + (k + 1) * r, n);
                        const int m = i2 - i1 + 1;
                        if (m < 2) continue;
                        const int i4a = j1 + imax(0, (k + t - qp + 1) * r);
                        if (row > i4a) continue;
                        const S* zr = a.Zr + ((int64_t)t * K + k) * (r + 1);
                        const S sig = zr[r];
                        if (is_zero(sig)) continue;
                        S s = S(0.0);
                        for (int c = 0; c < m; ++c) s = fma_s(X[i + ((i1 + c) % W) * BM], zr[c], s);
                        s = s * sig;
                        for (int c = 0; c < m; ++c) X[i + ((i1 + c) % W) * BM] -= s * conjv(zr[c]);
                    }
                }
                __syncthreads();
            }
        }
        pc0 = c0;
        pwk = wk;
    }
    if (pwk > 0) {
        for (int e = tid; e < nr * pwk; e += NT) {
            const int i = e % nr, c = pc0 + e / nr;
            IDX(M, ld, R0 + i, c) = X[i + (c % W) * BM];
        }
    }
}

// ---------------------------------------------------------------------------------------
// Column chain (left updates of A (M0, cols > i5) and B (M1, cols > i6)).
// grid.x = column tiles of BN, grid.y = matrix.  smem: X [W x BN] (row slot = row mod W,
// ld W+1), Y [W x BN], Us [W x W].
template <typename S, int BN, int NT>
__global__ void __launch_bounds__(NT) col_chain_kernel(ChainArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int W = a.W;
    const int LDX = W + 1;
    S* X = reinterpret_cast<S*>(smraw);
    S* Y = X + (size_t)LDX * BN;
    S* Us = Y + (size_t)LDX * BN;
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K;
    const int w = qp + r - 1;
    const bool isA = blockIdx.y == 0;
    S* M = isA ? a.M0 : a.M1;
    const int64_t ld = isA ? a.ld0 : a.ld1;
    const S* Blk = a.Blk0;
    const int C0 = blockIdx.x * BN + 1;
    if (C0 > n) return;
    const int nc = min(BN, n - C0 + 1);
    const int C1 = C0 + nc - 1;
    const int tid = threadIdx.x;
    auto cstart = [&](int k) {  // columns > cstart(k) receive U_k^*  (corrected i5 / i6)
        return isA ? j1 + qp - 1 + imax(0, (k - 1) * r + 1) : j1 + qp + (k + 1) * r - 1;
    };
    int kmax = K - 1;
    while (kmax >= 0 && cstart(kmax) >= C1) --kmax;
    if (kmax < 0) return;
    int pc0 = 0, pwk = 0;
    for (int k = kmax; k >= 0; --k) {
        const int c0 = j1 + k * r + 1;
        const int wk = min(w, n - c0 + 1);
        if (pwk > 0) {
            const int nl = pc0 + pwk - (c0 + wk);
            for (int e = tid; e < nl * nc; e += NT) {
                const int i = c0 + wk + e % nl, c = e / nl;
                IDX(M, ld, i, C0 + c) = X[(i % W) + c * LDX];
            }
            __syncthreads();
        }
        const int rin1 = (pwk > 0) ? pc0 : c0 + wk;
        const int ne = rin1 - c0;
        for (int e = tid; e < ne * nc; e += NT) {
            const int i = c0 + e % ne, c = e / ne;
            X[(i % W) + c * LDX] = IDX(M, ld, i, C0 + c);
        }
        const S* Bk = Blk + (int64_t)k * W * W;
        for (int e = tid; e < wk * wk; e += NT) {
            const int l = e % wk, c = e / wk;
            Us[l + c * W] = Bk[l + (int64_t)c * W];
        }
        __syncthreads();
        const int cs = cstart(k);
        for (int e = tid; e < nc * wk; e += NT) {
            const int c = e % nc, i = e / nc;
            S acc = S(0.0);
            for (int l = 0; l < wk; ++l) acc += conj_mul(Us[l + i * W], X[((c0 + l) % W) + c * LDX]);
            Y[i + c * LDX] = acc;
        }
        __syncthreads();
        for (int e = tid; e < nc * wk; e += NT) {
            const int c = e % nc, i = e / nc;
            if (C0 + c > cs) X[((c0 + i) % W) + c * LDX] = Y[i + c * LDX];
        }
        __syncthreads();
        pc0 = c0;
        pwk = wk;
    }
    for (int e = tid; e < pwk * nc; e += NT) {
        const int i = pc0 + e % pwk, c = e / pwk;
        IDX(M, ld, i, C0 + c) = X[(i % W) + c * LDX];
    }
}
