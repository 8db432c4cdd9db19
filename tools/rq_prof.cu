// dev: long-running RQ loop (m=16) for ncu source-level stall sampling (not product code)
#include <cstdio>
#include <cstdlib>
#include "../paper_2301_07964_b200/csrc/chase.cuh"
__global__ void rqloop(const double* C0, double* out, int m, int reps) {
    extern __shared__ double dyn[];
    double* Cb = dyn; double* piv = dyn + 64 * 65; double* uu = piv + 64 * 84;
    __shared__ int flag;
    if (threadIdx.x == 0) flag = 1 << 30;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Cb[(e % m) + (e / m) * (m + 1)] = C0[e];
    __syncthreads();
    for (int it = 0; it < reps; ++it) {
        if (threadIdx.x < RQCfg<double, 16>::NTHR) rq_direction<double, 16>(m, Cb, m + 1, piv, &flag, uu);
        __syncthreads();
        if (threadIdx.x == 0) flag = 1 << 30;
        __syncthreads();
    }
    if (threadIdx.x < m) out[threadIdx.x] = uu[threadIdx.x];
}
int main() {
    double *C, *out;
    cudaMallocManaged(&C, 64 * 64 * 8); cudaMallocManaged(&out, 64 * 8);
    for (int i = 0; i < 64 * 64; ++i) C[i] = (rand() / (double)RAND_MAX) - 0.5;
    cudaFuncSetAttribute(rqloop, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    rqloop<<<1, 256, 100000>>>(C, out, 16, 3000);
    cudaDeviceSynchronize();
    printf("%s %g\n", cudaGetErrorString(cudaGetLastError()), out[0]);
}
