// dev micro-benchmark: cycles of the K1 RQ direction routine on one warp (not product code)
#include <cstdio>
#include <cstdlib>
#include "../paper_2301_07964_b200/csrc/chase.cuh"

template <int MAXM, int NWR>
__global__ void bench(const double* C0, double* out, long long* cyc, int m, int reps) {
    __shared__ double Cb[64 * 65];
    __shared__ double bc[2 * 80];
    __shared__ double uu[80];
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Cb[(e % m) + (e / m) * (m + 1)] = C0[e];
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (threadIdx.x < 32 * NWR) rq_direction<double, MAXM, NWR>(m, Cb, m + 1, bc, uu);
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x < m) out[threadIdx.x] = uu[threadIdx.x];
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
    int ms[3] = {16, 32, 64};
    for (int mi = 0; mi < 3; ++mi) {
        int m = ms[mi];
        double *C, *out; long long* cyc;
        cudaMallocManaged(&C, m * m * 8); cudaMallocManaged(&out, 64 * 8); cudaMallocManaged(&cyc, 8);
        for (int i = 0; i < m * m; ++i) C[i] = (rand() / (double)RAND_MAX) - 0.5;
        if (m == 16) bench<16, 1><<<1, 256>>>(C, out, cyc, m, 20);
        if (m == 32) bench<32, 1><<<1, 256>>>(C, out, cyc, m, 20);
        if (m == 64) bench<64, 4><<<1, 256>>>(C, out, cyc, m, 20);
        cudaDeviceSynchronize();
        printf("m=%d cycles/RQ=%lld (%s) u0=%g\n", m, cyc[0], cudaGetErrorString(cudaGetLastError()), out[0]);
    }
}
