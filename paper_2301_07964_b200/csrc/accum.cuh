// accum.cuh -- K2: fold each window's reflectors into the dense window blocks of the apply
// phase ("Q_k = Q_k^{j1} Q_k^{j2} ... Q_k^{j1+q-1}", PAPER.md:1903 likewise for
// Z_k; "Form compact WY" -- north_star keeps them as dense w x w blocks U_k, V_k).
//
// Grid (K, 2): block (k, 0) builds U_k from the left-reflector records Qr, block (k, 1) builds
// V_k from the right-reflector records Zr.  Record (t, k) holds v (v[0] = 1) of length
// m = min(r, n - (j1+t+kr)) and tau at [r]; a zero tau is the identity (steps that generate
// no reflector are left zero by the host).  Reflector t acts on window-local columns
// t .. t+m-1, so X <- X (I - tau v v^*) touches only rows 0 .. t+m-1 of X = I (initially).
// Output layout (read by the chain kernels): block k at Out + k*WP*LDB, row-major, (l, c) at
// [l*LDB + c], rows/cols >= w_k zero (so padded DMMA K-steps contribute nothing).
#pragma once
#include "scalar.cuh"

template <typename S>
struct AccumArgs {
    int n, r, qp, j1, K, WP, LDB;
    const S* Qr;
    const S* Zr;
    S* U;
    S* V;
};

template <typename S>
__host__ __device__ inline size_t accum_smem_bytes(int r, int qp) {
    const int w = qp + r - 1;
    return ((size_t)w * (w | 1) + (size_t)(r + 8)) * sizeof(S);
}

template <typename S, int NT>
__global__ void __launch_bounds__(NT) accum_kernel(AccumArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    S* X = reinterpret_cast<S*>(smraw);
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K;
    const int k = blockIdx.x;
    const bool isV = blockIdx.y != 0;
    const S* R = isV ? a.Zr : a.Qr;
    S* Out = (isV ? a.V : a.U) + (size_t)k * a.WP * a.LDB;
    const int w = qp + r - 1;
    const int wk = min(w, n - (j1 + k * r + 1) + 1);
    const int LX = wk | 1;  // odd row stride: thread-per-row access is conflict-free
    S* vs = X + (size_t)wk * LX;
    const int tid = threadIdx.x;
    for (int e = tid; e < wk * LX; e += NT) {
        const int l = e / LX, c = e % LX;
        X[e] = S(l == c ? 1.0 : 0.0);
    }
    __syncthreads();
    for (int t = 0; t < qp; ++t) {
        const S* rec = R + ((size_t)t * K + k) * (r + 1);
        const S tau = rec[r];
        if (is_zero(tau)) continue;  // uniform across the block
        const int m = min(r, min(n - (j1 + t + k * r), wk - t));
        for (int c = tid; c < m; c += NT) vs[c] = rec[c];
        __syncthreads();
        const int rows = min(t + m, wk);
        for (int l = tid; l < rows; l += NT) {
            S* xr = X + (size_t)l * LX + t;
            S s0 = S(0.0), s1 = S(0.0);
            int c = 0;
            for (; c + 1 < m; c += 2) {
                s0 = fma_s(xr[c], vs[c], s0);
                s1 = fma_s(xr[c + 1], vs[c + 1], s1);
            }
            if (c < m) s0 = fma_s(xr[c], vs[c], s0);
            const S s = (s0 + s1) * tau;
            for (c = 0; c < m; ++c) xr[c] -= s * conjv(vs[c]);
        }
        __syncthreads();
    }
    for (int e = tid; e < a.WP * a.LDB; e += NT) {
        const int l = e / a.LDB, c = e % a.LDB;
        Out[e] = (l < wk && c < wk) ? X[(size_t)l * LX + c] : S(0.0);
    }
}

// ---------------------------------------------------------------------------------------
// K2m: merged window blocks for the apply chains.  Consecutive windows overlap in q-1 columns,
// so P of them (k = klo .. khi) act on W = q + P r - 1 columns and, applied in the chain's
// descending order, compose to ONE W x W block
//     M = V'_khi V'_{khi-1} ... V'_klo      (V'_k = V_k embedded at column offset (k-klo) r),
// the same for U.  A merged chain step costs W^2 per row against P w^2 for P single steps
// (about equal for P ~ 4 at q ~ 2r) but syncs and streams once instead of P times.
// Grid (ceil(K/P), 2); group mg covers windows [mg P, min(K-1, mg P + P - 1)].  Real fp64 only.
template <typename S>
struct MergeArgs {
    int n, r, qp, j1, K, P, WP, LDB;
    const S* U;  // single blocks (chain layout: WP x LDB row-major, zero padded)
    const S* V;
    S* MU;       // merged blocks, same layout
    S* MV;
};

template <typename S>
__host__ __device__ inline size_t merge_smem_bytes(int W, int w) {
    return (2 * (size_t)W * (W | 1) + (size_t)w * (w | 1)) * sizeof(S);
}

template <typename S, int NT>
__global__ void __launch_bounds__(NT) merge_kernel(MergeArgs<S> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K, P = a.P;
    const int mg = blockIdx.x;
    const bool isV = blockIdx.y != 0;
    const S* Blk = isV ? a.V : a.U;
    S* Out = (isV ? a.MV : a.MU) + (size_t)mg * a.WP * a.LDB;
    const int w = qp + r - 1;
    const int klo = mg * P, khi = min(K - 1, klo + P - 1);
    const int c0 = j1 + klo * r + 1;
    const int W = min(qp + (khi - klo + 1) * r - 1, n - c0 + 1);
    const int LM = W | 1;
    S* M = reinterpret_cast<S*>(smraw);
    S* M2 = M + (size_t)W * LM;
    S* Vs = M2 + (size_t)W * LM;  // the current window block (w x (w|1))
    const int LV = w | 1;
    const int tid = threadIdx.x;
    // M = V'_khi (identity outside its columns)
    {
        const int o = (khi - klo) * r;
        const int wk = min(w, n - (j1 + khi * r + 1) + 1);
        const S* B = Blk + (size_t)khi * a.WP * a.LDB;
        for (int e = tid; e < W * LM; e += NT) {
            const int l = e / LM, c = e % LM;
            S v = S(0.0);
            if (c < W) {
                if (l >= o && l < o + wk && c >= o && c < o + wk) v = B[(size_t)(l - o) * a.LDB + (c - o)];
                else if (l == c) v = S(1.0);
            }
            M[e] = v;
        }
    }
    __syncthreads();
    for (int k = khi - 1; k >= klo; --k) {  // M <- M V'_k (columns o .. o+wk)
        const int o = (k - klo) * r;
        const int wk = min(w, n - (j1 + k * r + 1) + 1);
        const S* B = Blk + (size_t)k * a.WP * a.LDB;
        for (int e = tid; e < wk * wk; e += NT) {
            const int l = e / wk, c = e % wk;
            Vs[(size_t)l * LV + c] = B[(size_t)l * a.LDB + c];
        }
        __syncthreads();
        for (int e = tid; e < W * LM; e += NT) {
            const int l = e / LM, c = e % LM;
            S v = M[e];
            if (c >= o && c < o + wk) {
                S s0 = S(0.0), s1 = S(0.0), s2 = S(0.0), s3 = S(0.0);
                const S* mr = M + (size_t)l * LM + o;
                const S* vc = Vs + (c - o);
                int cc = 0;
                for (; cc + 3 < wk; cc += 4) {
                    s0 = fma_s(mr[cc], vc[(size_t)cc * LV], s0);
                    s1 = fma_s(mr[cc + 1], vc[(size_t)(cc + 1) * LV], s1);
                    s2 = fma_s(mr[cc + 2], vc[(size_t)(cc + 2) * LV], s2);
                    s3 = fma_s(mr[cc + 3], vc[(size_t)(cc + 3) * LV], s3);
                }
                for (; cc < wk; ++cc) s0 = fma_s(mr[cc], vc[(size_t)cc * LV], s0);
                v = (s0 + s1) + (s2 + s3);
            }
            M2[e] = v;
        }
        __syncthreads();
        S* tmp = M;
        M = M2;
        M2 = tmp;
    }
    for (int e = tid; e < a.WP * a.LDB; e += NT) {
        const int l = e / a.LDB, c = e % a.LDB;
        Out[e] = (l < W && c < W) ? M[(size_t)l * LM + c] : S(0.0);
    }
}
