// dev micro-benchmark: the RQ-update chain step (shfl -> Givens -> carry update) in isolation
#include <cstdio>
#include "rqu.cuh"
#define STEP_BASE                                                                                   \
    const double xj = x;                                                                            \
    x = lds64(sa + 8u * (j & 63));                                                                  \
    double a = __shfl_sync(0xffffffffu, xj, j & 31), b = __shfl_sync(0xffffffffu, carry, j & 31);   \
    double c, s;                                                                                    \
    giv_rot(a, b, c, s);                                                                            \
    sts64(sa + 8u * ((j + 1) & 63), fma(xj, s, carry * c));                                         \
    carry = fma(xj, c, -carry * s) + 0.5;
__global__ void k(double* out, long long* cyc, int n) {
    __shared__ double sh[64 * 65 + 1024];
    const int lane = threadIdx.x & 31;
    double carry = 1.0 + lane * 1e-3, carry2 = 0.5 + lane * 1e-3, x = 0.3 + lane * 1e-4;
    for (int i = threadIdx.x; i < 64 * 65 + 1024; i += blockDim.x) sh[i] = i * 1e-3;
    __syncthreads();
    const unsigned sa = opaque_u32(rq_smem_u32(sh) + 8u * 65 * lane), ca = opaque_u32(rq_smem_u32(sh + 64 * 65));
    long long t[8];
    t[0] = clock64();
    for (int j = n; j > 0; --j) { STEP_BASE }
    t[1] = clock64();
    for (int j = n; j > 0; --j) { STEP_BASE sts64v_if(lane == 0, ca + 16u * (j & 31), c); sts64v_if(lane == 0, ca + 16u * (j & 31) + 8, s); sts32v_if(lane == 0, ca + 600, j); }
    t[2] = clock64();
    for (int j = n; j > 0; --j) { STEP_BASE sts64_if(lane == 0, ca + 16u * (j & 31), c); sts64_if(lane == 0, ca + 16u * (j & 31) + 8, s); }
    t[3] = clock64();
    for (int j = n; j > 0; --j) { STEP_BASE const double nc2 = fma(xj, c, -carry2 * s); sts64_if(lane < j % 40, sa + 8u * ((j + 2) & 63), fma(xj, s, carry2 * c)); carry2 = nc2; }
    t[4] = clock64();
    for (int j = n; j > 0; --j) { double c, s; giv_rot(x, carry, c, s); carry = c + 0.5; }
    t[5] = clock64();
    out[threadIdx.x] = carry + carry2 + x;
    if (threadIdx.x == 0) for (int i = 0; i < 5; ++i) cyc[i] = (t[i + 1] - t[i]) / n;
}
int main() {
    double* out; long long* cyc;
    cudaMallocManaged(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
    for (int w = 1; w <= 8; w *= 8) {
        k<<<1, 32 * w>>>(out, cyc, 1000); cudaDeviceSynchronize();
        printf("warps=%d base=%lld +vol-stores=%lld +pred-stores=%lld +row2=%lld giv-only=%lld\n", w, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
    }
}
