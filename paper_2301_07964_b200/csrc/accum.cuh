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
