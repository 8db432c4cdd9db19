// dev micro-benchmark (not product code): cycles of K1 pieces on one CTA of 256 threads
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2301_07964_b200/csrc/chase.cuh"

template <int MAXM>
__global__ void bench(const double* C0, double* out, long long* cyc, int m, int reps) {
    extern __shared__ double dyn[];
    double* Cb = dyn;
    double* piv = dyn + 64 * 65;
    __shared__ int flag;
    if (threadIdx.x == 0) flag = 1 << 30;
    __syncthreads();
    __shared__ double uu[80];
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Cb[(e % m) + (e / m) * (m + 1)] = C0[e];
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (threadIdx.x < rq_nthr<double, MAXM>()) rq_dir<double, MAXM>(m, Cb, m + 1, piv, &flag, uu);
        __syncthreads();
        if (threadIdx.x == 0) flag = 1 << 30;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x < m) out[threadIdx.x] = uu[threadIdx.x];
    __syncthreads();
    double tau; double beta;
    for (int it = 0; it < reps; ++it) {
        if (threadIdx.x < 32) warp_larfg(m, uu, piv, tau, beta);
        __syncthreads();
    }
    long long t2 = clock64();
    
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; cyc[1] = (t2 - t1) / reps; }
}

int main() {
    int ms[4] = {8, 16, 32, 64};
    for (int mi = 0; mi < 4; ++mi) {
        int m = ms[mi];
        double *C, *out; long long* cyc;
        cudaMallocManaged(&C, m * m * 8); cudaMallocManaged(&out, 64 * 8); cudaMallocManaged(&cyc, 16);
        for (int i = 0; i < m * m; ++i) C[i] = (rand() / (double)RAND_MAX) - 0.5;
        if (m == 8) { cudaFuncSetAttribute(bench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); bench<8><<<1, 256, 100000>>>(C, out, cyc, m, 20); }
        if (m == 16) { cudaFuncSetAttribute(bench<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); bench<16><<<1, 256, 100000>>>(C, out, cyc, m, 20); }
        if (m == 32) { cudaFuncSetAttribute(bench<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); bench<32><<<1, 256, 100000>>>(C, out, cyc, m, 20); }
        if (m == 64) { cudaFuncSetAttribute(bench<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); bench<64><<<1, rq_nthr<double, 64>() > 256 ? rq_nthr<double, 64>() : 256, 100000>>>(C, out, cyc, m, 20); }
        cudaDeviceSynchronize();
        // residual of rows 1..m-1 of C u (must vanish) and |u|
        double res = 0, nu = 0, nc = 0;
        for (int i = 0; i < m; ++i) nu += out[i] * out[i];
        for (int i = 1; i < m; ++i) { double s = 0; for (int c = 0; c < m; ++c) s += C[i + c * m] * out[c]; res += s * s; }
        for (int i = 0; i < m * m; ++i) nc += C[i] * C[i];
        printf("m=%d cycles/RQ=%lld larfg=%lld (%s) |u|=%.15f res=%.3e\n", m, cyc[0], cyc[1], cudaGetErrorString(cudaGetLastError()), sqrt(nu), sqrt(res / nc));
    }
}
