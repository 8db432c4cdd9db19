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
#include "chain.cuh"  // chain_ldb / chain_wy_ldy: the block strides the chains read

template <typename S>
struct AccumArgs {
    int n, r, qp, j1, K, WP, LDB;
    int pre;  // 1: all records of the window staged at once (else one at a time: large w)
    const S* Qr;
    const S* Zr;
    S* U;
    S* V;
    const unsigned long long* gate;  // input-check verdict (input_rejected)
};

template <typename S>
__host__ __device__ inline size_t accum_smem_bytes(int r, int qp, bool pre) {
    const int w = qp + r - 1;
    return ((size_t)w * (w | 1) + (pre ? (size_t)qp * (r + 1) : (size_t)(r + 1))) * sizeof(S);
}

template <typename S, int NT>
__global__ void __launch_bounds__(NT) accum_kernel(AccumArgs<S> a) {
    if (input_rejected(a.gate)) return;
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
    S* recs = X + (size_t)wk * LX;  // all qp records of the window, loaded at once
    const int tid = threadIdx.x;
    for (int l = tid / 32; l < wk; l += NT / 32)  // (warp per row, lanes along it: no division)
        for (int c = tid % 32; c < LX; c += 32) X[(size_t)l * LX + c] = S(l == c ? 1.0 : 0.0);
    if (a.pre)
        for (int t = tid / 32; t < qp; t += NT / 32)  // warp per record (one latency for all of them)
            for (int c = tid % 32; c <= r; c += 32) recs[(size_t)t * (r + 1) + c] = R[((size_t)t * K + k) * (r + 1) + c];
    __syncthreads();
    for (int t = 0; t < qp; ++t) {
        const S* vs = recs + (a.pre ? (size_t)t * (r + 1) : 0);
        if (!a.pre) {
            const S* rec = R + ((size_t)t * K + k) * (r + 1);
            for (int c = tid; c <= r; c += NT) recs[c] = rec[c];
            __syncthreads();
        }
        const S tau = vs[r];
        if (is_zero(tau)) continue;  // uniform across the block
        const int m = min(r, min(n - (j1 + t + k * r), wk - t));
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
    for (int l = tid / 32; l < a.WP; l += NT / 32)
        for (int c = tid % 32; c < a.LDB; c += 32)
            Out[(size_t)l * a.LDB + c] = (l < wk && c < wk) ? X[(size_t)l * LX + c] : S(0.0);
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
    const unsigned long long* gate;  // input-check verdict (input_rejected)
};

template <typename S>
__host__ __device__ inline size_t merge_smem_bytes(int W, int w) {
    return ((size_t)W * (W | 1) + (size_t)W * (w + 4) + (size_t)w * (w + 4)) * sizeof(S);
}

template <typename S, int NT>
__global__ void __launch_bounds__(NT) merge_kernel(MergeArgs<S> a) {
    if (input_rejected(a.gate)) return;
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
    // M (W x LM); Tm = M(:, o:o+wk) V'_k (W x LT), then copied back; Vs = the window block (w x LT)
    const int LT = w + 4;
    S* M = reinterpret_cast<S*>(smraw);
    S* Tm = M + (size_t)W * LM;
    S* Vs = Tm + (size_t)W * LT;
    const int tid = threadIdx.x;
    // M = V'_khi (identity outside its columns)
    {
        const int o = (khi - klo) * r;
        const int wk = min(w, n - (j1 + khi * r + 1) + 1);
        const S* B = Blk + (size_t)khi * a.WP * a.LDB;
        for (int l = tid / 32; l < W; l += NT / 32)
            for (int c = tid % 32; c < LM; c += 32) {
                S v = S(0.0);
                if (c < W) {
                    if (l >= o && l < o + wk && c >= o && c < o + wk) v = B[(size_t)(l - o) * a.LDB + (c - o)];
                    else if (l == c) v = S(1.0);
                }
                M[(size_t)l * LM + c] = v;
            }
    }
    for (int k = khi - 1; k >= klo; --k) {  // M <- M V'_k (columns o .. o+wk)
        const int o = (k - klo) * r;
        const int wk = min(w, n - (j1 + k * r + 1) + 1);
        const S* B = Blk + (size_t)k * a.WP * a.LDB;
        for (int l = tid / 32; l < wk; l += NT / 32)
            for (int c = tid % 32; c < wk; c += 32) Vs[(size_t)l * LT + c] = B[(size_t)l * a.LDB + c];
        __syncthreads();
        // register tiles of 4 rows x 4 columns: 8 shared loads per 16 FMAs (lanes of a warp share
        // the row tile: the M loads broadcast, the Vs loads are consecutive)
        const int nct = (wk + 3) / 4, nrt = (W + 3) / 4;
        for (int id = tid; id < nct * nrt; id += NT) {
            const int l0 = (id / nct) * 4, cb = (id % nct) * 4;
            S acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) acc[i][jj] = S(0.0);
            const S* mr = M + (size_t)l0 * LM + o;
            for (int cc = 0; cc < wk; ++cc) {
                S mv[4], vv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) mv[i] = (l0 + i < W) ? mr[(size_t)i * LM + cc] : S(0.0);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) vv[jj] = Vs[(size_t)cc * LT + cb + jj];  // (cols >= wk: LT pad)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fma_s(mv[i], vv[jj], acc[i][jj]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    if (l0 + i < W && cb + jj < wk) Tm[(size_t)(l0 + i) * LT + cb + jj] = acc[i][jj];
        }
        __syncthreads();
        for (int l = tid / 32; l < W; l += NT / 32)
            for (int c = tid % 32; c < wk; c += 32) M[(size_t)l * LM + o + c] = Tm[(size_t)l * LT + c];
        __syncthreads();
    }
    for (int l = tid / 32; l < a.WP; l += NT / 32)
        for (int c = tid % 32; c < a.LDB; c += 32)
            Out[(size_t)l * a.LDB + c] = (l < W && c < W) ? M[(size_t)l * LM + c] : S(0.0);
}

// ---------------------------------------------------------------------------------------
// K2w: the window blocks in compact WY form for the apply chains ("compact WY
// representation", "Form compact WY").  The window's reflectors
// in sweep order, H_t = I - tau_t y_t y_t^* with y_t = v_t at window offset t (m_t entries), give
// H_0 H_1 ... H_{qp-1} = I - Y T Y^* (forward, columnwise xLARFT: T(t,t) = tau_t,
// T(s,t) = -tau_t sum_{l=s}^{t-1} T(s,l) (y_l^* y_t)).  Stored per window (chain_wy_stride):
// Y (WP x (QP + 8), row-major, zero outside the staircase) then T Y^* (QP x (WP + 8)).
// Grid (K, 2): block (k, 0) from the left reflectors (U_k), (k, 1) from the right ones (V_k).
template <typename S>
struct AccumWYArgs {
    int n, r, qp, j1, K, WP, QP;
    const S* Qr;
    const S* Zr;
    S* U;
    S* V;
    const unsigned long long* gate;
};

template <typename S>
__host__ __device__ inline size_t accum_wy_smem_bytes(int r, int qp, int QP) {
    return ((size_t)qp * (r + 1) + 2 * (size_t)QP * (QP + 1)) * sizeof(S);
}

template <typename S, int NT>
__global__ void __launch_bounds__(NT) accum_wy_kernel(AccumWYArgs<S> a) {
    if (input_rejected(a.gate)) return;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int n = a.n, r = a.r, qp = a.qp, j1 = a.j1, K = a.K, WP = a.WP, QP = a.QP;
    const int LDY = chain_wy_ldy<S>(QP), LDB = chain_ldb<S>(WP);
    const int k = blockIdx.x;
    const bool isV = blockIdx.y != 0;
    const S* R = isV ? a.Zr : a.Qr;
    S* Out = (isV ? a.V : a.U) + (size_t)k * ((size_t)WP * LDY + (size_t)QP * LDB);
    const int w = qp + r - 1;
    const int wk = min(w, n - (j1 + k * r + 1) + 1);
    S* recs = reinterpret_cast<S*>(smraw);       // qp records (r + 1)
    S* G = recs + (size_t)qp * (r + 1);          // QP x (QP+1): y_l^* y_t (l < t)
    S* T = G + (size_t)QP * (QP + 1);            // QP x (QP+1)
    const int tid = threadIdx.x;
    for (int t = tid / 32; t < qp; t += NT / 32)
        for (int c = tid % 32; c <= r; c += 32) recs[(size_t)t * (r + 1) + c] = R[((size_t)t * K + k) * (r + 1) + c];
    __syncthreads();
    auto msz = [&](int t) { return min(r, min(n - (j1 + t + k * r), wk - t)); };  // entries of y_t in the window
    auto tau = [&](int t) { return recs[(size_t)t * (r + 1) + r]; };
    // Y (row-major), zero outside the staircase and the padding
    for (int e = tid; e < WP * LDY; e += NT) {
        const int i = e / LDY, t = e % LDY;
        S v = S(0.0);
        if (t < qp && i < wk && i >= t && i - t < msz(t) && !is_zero(tau(t))) v = recs[(size_t)t * (r + 1) + (i - t)];
        Out[e] = v;
    }
    // Gram entries G(l, t) = y_l^* y_t, l < t (rows t .. l + m_l - 1 overlap)
    for (int e = tid; e < qp * qp; e += NT) {
        const int l = e / qp, t = e % qp;
        S g = S(0.0);
        if (l < t && !is_zero(tau(l)) && !is_zero(tau(t))) {
            const S* yl = recs + (size_t)l * (r + 1);
            const S* yt = recs + (size_t)t * (r + 1);
            const int hi = min(l + msz(l), t + msz(t));
            for (int i = t; i < hi; ++i) g += conj_mul(yl[i - l], yt[i - t]);
        }
        G[(size_t)l * (QP + 1) + t] = g;
    }
    __syncthreads();
    // T rows are independent given G: T(s, t) = -tau_t sum_{l=s}^{t-1} T(s, l) G(l, t)
    for (int s2 = tid; s2 < QP; s2 += NT) {
        S* Ts = T + (size_t)s2 * (QP + 1);
        for (int t = 0; t < QP; ++t) {
            S v = S(0.0);
            if (s2 < qp && t < qp) {
                const S tt = tau(t);
                if (t == s2) {
                    v = tt;
                } else if (t > s2 && !is_zero(tt)) {
                    S acc = S(0.0);
                    for (int l = s2; l < t; ++l) acc += Ts[l] * G[(size_t)l * (QP + 1) + t];
                    v = -(tt * acc);
                }
            }
            Ts[t] = v;
        }
    }
    __syncthreads();
    // T Y^* (QP x LDB): row s, column c = sum_{t >= s} T(s, t) conj(Y(c, t))
    S* Bw = Out + (size_t)WP * LDY;
    for (int e = tid; e < QP * LDB; e += NT) {
        const int s2 = e / LDB, c = e % LDB;
        S v = S(0.0);
        if (s2 < qp && c < wk) {
            const int tlo = max(s2, c - r + 1), thi = min(qp - 1, c);  // y_t covers rows t .. t + m_t - 1
            for (int t = tlo; t <= thi; ++t)
                if (c - t < msz(t) && !is_zero(tau(t)))
                    v += T[(size_t)s2 * (QP + 1) + t] * conjv(recs[(size_t)t * (r + 1) + (c - t)]);
        }
        Bw[e] = v;
    }
}
