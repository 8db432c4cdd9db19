// dev micro-benchmark (not product code): per-phase cycles of one RQ stage (copy of rq_direction with clocks)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2301_07964_b200/csrc/chase.cuh"

template <int MAXM>
__device__ void rq_timed(int m, const double* Cb, int LDC, double* piv, double* uu, long long* ph) {
    using S = double;
    using CF = RQCfg<S, MAXM>;
    constexpr int SB = CF::SB, NSB = CF::NSB, E = NSB * SB, PL = E + 2;
    const int tid = threadIdx.x;
    const bool isP = tid >= MAXM;
    const int l = isP ? tid - MAXM : tid;
    const bool live = tid < 2 * MAXM && l < m;
    S row[E];
#pragma unroll
    for (int c = 0; c < E; ++c) { S v = 0; if (live && c < m) v = isP ? (l == c ? 1.0 : 0.0) : Cb[l + c * LDC]; row[c] = v; }
    int par = 0;
    if (live && !isP && l == m - 1) for (int c = 0; c < E; ++c) piv[c] = row[c];
    __syncwarp();
    long long t0 = clock64(), t1, t2, t3, t4;
    for (int i = m - 1; i >= 1; --i) {
        const S* pv = piv + par * PL;
        double n0 = 0, n1 = 0, g0 = 0, g1 = 0, ri = 0;
        const int sbi = i / SB, ei = i % SB;
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb) {
            if (sb < sbi) {
#pragma unroll
                for (int e = 0; e < SB; ++e) { const S b = pv[sb * SB + e]; if (e & 1) { n1 += b * b; g1 = fma(row[sb * SB + e], b, g1); } else { n0 += b * b; g0 = fma(row[sb * SB + e], b, g0); } }
            } else if (sb == sbi) {
#pragma unroll
                for (int e = 0; e < SB; ++e) { const S b = (e < ei) ? pv[sb * SB + e] : 0.0; if (e & 1) { n1 += b * b; g1 = fma(row[sb * SB + e], b, g1); } else { n0 += b * b; g0 = fma(row[sb * SB + e], b, g0); } if (e == ei) ri = row[sb * SB + e]; }
            }
        }
        const double nx = n0 + n1, g = g0 + g1;
        const double alpha = pv[i];
        t1 = clock64(); ph[0] += t1 - t0;
        double f = 0;
        if (nx != 0.0) {
            const double nrm = sqrt(alpha * alpha + nx);
            const double beta = (alpha >= 0.0) ? -nrm : nrm;
            const double amb = alpha - beta;
            f = -(g + ri * amb) / (beta * amb);
        }
        if (!(live && (isP || l < i))) f = 0.0;
        t2 = clock64(); ph[1] += t2 - t1;
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb) {
            if (sb < sbi) {
#pragma unroll
                for (int e = 0; e < SB; ++e) row[sb * SB + e] -= f * pv[sb * SB + e];
            } else if (sb == sbi) {
#pragma unroll
                for (int e = 0; e < SB; ++e) if (e < ei) row[sb * SB + e] -= f * pv[sb * SB + e];
            }
        }
        t3 = clock64(); ph[2] += t3 - t2;
        par ^= 1;
        if (live && !isP && l == i - 1) {
#pragma unroll
            for (int sb = 0; sb < NSB; ++sb) if (sb <= sbi)
#pragma unroll
                for (int e = 0; e < SB; ++e) piv[par * PL + sb * SB + e] = row[sb * SB + e];
        }
        __syncwarp();
        t4 = clock64(); ph[3] += t4 - t3;
        t0 = t4;
    }
    if (live && isP) uu[l] = row[0];
}

template <int MAXM>
__global__ void bench(const double* C0, double* out, long long* cyc, int m) {
    __shared__ double Cb[64 * 65];
    __shared__ double piv[2 * 66];
    __shared__ double uu[80];
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Cb[(e % m) + (e / m) * (m + 1)] = C0[e];
    __syncthreads();
    long long ph[4] = {0, 0, 0, 0};
    for (int it = 0; it < 10; ++it) if (threadIdx.x < 32) rq_timed<MAXM>(m, Cb, m + 1, piv, uu, ph);
    if (threadIdx.x == 0) for (int i = 0; i < 4; ++i) cyc[i] = ph[i] / 10 / (m - 1);
    if (threadIdx.x < m) out[threadIdx.x] = uu[threadIdx.x];
}

__global__ void lat(double* out, long long* cyc, double x0) {
    __shared__ double sh[64];
    if (threadIdx.x < 64) sh[threadIdx.x] = threadIdx.x * 1e-3;
    __syncwarp();
    double a = x0;
    long long t0 = clock64();
    for (int i = 0; i < 100; ++i) a = sqrt(a + 2.0);
    long long t1 = clock64();
    for (int i = 0; i < 100; ++i) a = 1.0 / (a + 2.0);
    long long t2 = clock64();
    for (int i = 0; i < 100; ++i) a = __shfl_sync(0xffffffff, a, (threadIdx.x + 1) & 31) + 1e-3;
    long long t3 = clock64();
    for (int i = 0; i < 100; ++i) { if (threadIdx.x == 0) sh[1] = a; __syncwarp(); a = sh[1] + 1e-3; __syncwarp(); }
    long long t4 = clock64();
    for (int i = 0; i < 100; ++i) a = fma(a, 1.0000001, 1e-9);
    long long t5 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 100; cyc[1] = (t2 - t1) / 100; cyc[2] = (t3 - t2) / 100; cyc[3] = (t4 - t3) / 100; cyc[4] = (t5 - t4) / 100; }
}

int main() {
    double *C, *out; long long* cyc;
    cudaMallocManaged(&C, 64 * 64 * 8); cudaMallocManaged(&out, 64 * 8); cudaMallocManaged(&cyc, 64);
    for (int i = 0; i < 64 * 64; ++i) C[i] = (rand() / (double)RAND_MAX) - 0.5;
    lat<<<1, 32>>>(out, cyc, 1.0); cudaDeviceSynchronize();
    printf("sqrt+add=%lld div+add=%lld shfl+add=%lld sts-sync-lds+add=%lld dfma=%lld\n", cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
    bench<8><<<1, 256>>>(C, out, cyc, 8); cudaDeviceSynchronize();
    printf("m=8  per stage: dots=%lld scal=%lld upd=%lld wr+sync=%lld\n", cyc[0], cyc[1], cyc[2], cyc[3]);
    bench<16><<<1, 256>>>(C, out, cyc, 16); cudaDeviceSynchronize();
    printf("m=16 per stage: dots=%lld scal=%lld upd=%lld wr+sync=%lld  (%s)\n", cyc[0], cyc[1], cyc[2], cyc[3], cudaGetErrorString(cudaGetLastError()));
}
