// dev micro-benchmark (not product code): latency of the warp-row RQ's pieces on sm_100a
#include <cstdio>
#define RQW_TRACE 1
#include "../paper_2301_07964_b200/csrc/chase.cuh"
#include "../paper_2301_07964_b200/csrc/rqw.cuh"

template <int N>
__global__ void k_allreduce(double* out, long long* cyc, int iters) {
    double v[N];
    for (int k = 0; k < N; ++k) v[k] = threadIdx.x * 1e-3 + k;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        warp_allreduce_n<double, N>(v);
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] *= 1e-3;
    }
    long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < N; ++k) s += v[k];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
}
__global__ void k_scalars(double* out, long long* cyc, int iters) {
    double a = 0.3 + threadIdx.x, nx = 1.7, K1 = 0, K2 = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        rqw_scalars(a, nx, K1, K2);
        a = K2 * 0.5 + 1.0;
        nx = K1 + 1.0;
    }
    long long t1 = clock64();
    out[threadIdx.x] = a + nx;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
}
template <int NW>
__global__ void k_rq(const double* C0, double* out, long long* cyc, int m) {
    extern __shared__ double dyn[];
    const int LDC = 65, HLD = 68;
    double* Cb = dyn;
    double* hb = Cb + 64 * LDC;
    double* uu = hb + 64 * HLD;
    __shared__ int flag;
    __shared__ uint64_t bars[128];
    if (threadIdx.x < 32) rqw_bars_init(bars, 128);
    __syncthreads();
    long long tot = 0;
    for (int it = 0; it < 5; ++it) {
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) Cb[(e % m) + (e / m) * LDC] = C0[e];
        if (threadIdx.x == 0) flag = 1 << 30;
        __syncthreads();
        long long t0 = clock64();
        rq_direction_w<double, 64, NW>(m, Cb, LDC, hb, HLD, bars, it & 1, uu);
        __syncthreads();
        tot += clock64() - t0;
    }
    if (threadIdx.x < m) out[threadIdx.x] = uu[threadIdx.x];
    if (threadIdx.x == 0) cyc[0] = tot / 5;
}
int main(int argc, char** argv) {
    const bool only8 = argc > 1;
    double* out; long long* cyc; double* C;
    cudaMallocManaged(&out, 4096 * 8); cudaMallocManaged(&cyc, 64); cudaMallocManaged(&C, 64 * 64 * 8);
    for (int i = 0; i < 64 * 64; ++i) C[i] = (rand() / (double)RAND_MAX) - 0.5;
    k_allreduce<1><<<1, 32>>>(out, cyc, 1000); cudaDeviceSynchronize(); printf("allreduce N=1: %lld cyc\n", cyc[0]);
    k_allreduce<8><<<1, 32>>>(out, cyc, 1000); cudaDeviceSynchronize(); printf("allreduce N=8: %lld cyc\n", cyc[0]);
    k_allreduce<16><<<1, 32>>>(out, cyc, 1000); cudaDeviceSynchronize(); printf("allreduce N=16: %lld cyc\n", cyc[0]);
    k_allreduce<8><<<1, 256>>>(out, cyc, 1000); cudaDeviceSynchronize(); printf("allreduce N=8, 8 warps: %lld cyc\n", cyc[0]);
    k_allreduce<16><<<1, 256>>>(out, cyc, 1000); cudaDeviceSynchronize(); printf("allreduce N=16, 8 warps: %lld cyc\n", cyc[0]);
    k_scalars<<<1, 32>>>(out, cyc, 1000); cudaDeviceSynchronize(); printf("scalars: %lld cyc\n", cyc[0]);
    int b = (64 * 65 + 64 * 68 + 72) * 8;

    cudaFuncSetAttribute(k_rq<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(k_rq<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);

    if (!only8) k_rq<4><<<1, 128, b>>>(C, out, cyc, 64); cudaDeviceSynchronize(); printf("rq m=64 NW=4: %lld cyc\n", cyc[0]);
    for (int mm : {2, 8, 16, 32}) {
        if (only8 && mm != 8) continue;
        k_rq<8><<<1, 256, b>>>(C, out, cyc, mm); cudaDeviceSynchronize(); printf("rq m=%d NW=8: %lld cyc\n", mm, cyc[0]);
        long long tr0[4096];
        cudaMemcpyFromSymbol(tr0, rqw_trace, sizeof(tr0));
        printf("   stage starts rel. to stage m-1:");
        for (int i = mm - 1; i >= 1; --i) printf(" %d:%lld", i, tr0[i] - tr0[mm - 1]);
        printf(" | end own w0: %lld, bar: %lld, end: %lld\n", tr0[2048] - tr0[mm - 1], tr0[3072] - tr0[mm - 1], tr0[3100] - tr0[mm - 1]);
    }
    if (only8) return 0;
    k_rq<8><<<1, 256, b>>>(C, out, cyc, 64); cudaDeviceSynchronize(); printf("rq m=64 NW=8: %lld cyc\n", cyc[0]);
    long long tr[4096];
    cudaMemcpyFromSymbol(tr, rqw_trace, sizeof(tr));
    long long t0 = tr[1024 + 7];
    printf("stage starts (rel. to warp 7 block start):");
    for (int i = 63; i >= 1; --i) printf(" %d:%lld", i, tr[i] - t0);
    printf("\nblock start / end / bar per warp:");
    for (int w = 7; w >= 0; --w) printf(" w%d:%lld/%lld/%lld", w, tr[1024 + w] - t0, tr[2048 + w] - t0, tr[3072 + w] - t0);
    printf("\nend of reverse pass: %lld\n", tr[3100] - t0);
    printf("stage 60 substeps (rel. to its start):");
    for (int k = 0; k < 7; ++k) printf(" %d:%lld", k, tr[3200 + k] - tr[60]);
    printf("\n");
}
