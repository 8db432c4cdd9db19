// dev micro-benchmark: larfg_regn latency (one warp)
#include <cstdio>
#include "chase.cuh"
__global__ void k(double* out, long long* cyc, int n, int m) {
    __shared__ double x[128], v[128];
    for (int i = threadIdx.x; i < 128; i += 32) x[i] = 1.0 + i * 1e-3;
    __syncwarp();
    double tau = 0, beta = 0, acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
        larfg_regn<double, 2>(m, x, v, tau, beta);
        acc += tau;
        if (threadIdx.x == 0) x[0] = 1.0 + 1e-9 * acc;
        __syncwarp();
    }
    long long t1 = clock64();
    for (int it = 0; it < n; ++it) {
        warp_larfg<double>(m, x, v, tau, beta);
        acc += tau;
        if (threadIdx.x == 0) x[0] = 1.0 + 1e-9 * acc;
        __syncwarp();
    }
    long long t2 = clock64();
    out[threadIdx.x] = acc + v[threadIdx.x];
    if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; }
}
int main() {
    double* out; long long* cyc;
    cudaMallocManaged(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
    k<<<1, 32>>>(out, cyc, 200, 64); cudaDeviceSynchronize();
    printf("larfg_regn(64)=%lld warp_larfg(64)=%lld cycles\n", cyc[0], cyc[1]);
}
