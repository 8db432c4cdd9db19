// dev micro-benchmark: back-substitution step chain (DMUL -> SHFL -> DFMA) variants
#include <cstdio>
#include "rqu.cuh"
__global__ void k(double* out, long long* cyc, int n) {
    __shared__ double sh[64 * 65];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 65; i += blockDim.x) sh[i] = 1e-3 * (i % 97);
    __syncthreads();
    const unsigned rs0 = opaque_u32(rq_smem_u32(sh));
    double rhs0 = 1.0 + lane, rhs1 = 2.0 + lane, rinv0 = 0.5, rinv1 = 0.25, u0 = 0, u1 = 0;
    long long t[8];
    t[0] = clock64();
    for (int i = n; i >= 1; --i) {  // V1: registers only
        const int L = i & 31;
        double ui = ((i >> 5) & 1) ? rhs1 * rinv1 : rhs0 * rinv0;
        ui = __shfl_sync(0xffffffffu, ui, L);
        rhs0 = fma(-0.001, ui, rhs0);
        rhs1 = fma(-0.002, ui, rhs1);
    }
    t[1] = clock64();
    for (int i = n; i >= 1; --i) {  // V2: + per-lane select of u
        const int L = i & 31;
        double ui = ((i >> 5) & 1) ? rhs1 * rinv1 : rhs0 * rinv0;
        ui = __shfl_sync(0xffffffffu, ui, L);
        if (lane == L) u0 = ui;
        if (lane + 32 == (i & 63)) u1 = ui;
        rhs0 = fma(-0.001, ui, rhs0);
        rhs1 = fma(-0.002, ui, rhs1);
    }
    t[2] = clock64();
    double c0 = 0, c1 = 0;
    for (int i = n; i >= 1; --i) {  // V3: + smem loads (current iteration)
        const int L = i & 31;
        c0 = lds64(rs0 + 8u * (lane * 65 + (i & 63)));
        c1 = lds64(rs0 + 8u * ((lane + 32) * 65 + (i & 63)));
        double ui = ((i >> 5) & 1) ? rhs1 * rinv1 : rhs0 * rinv0;
        ui = __shfl_sync(0xffffffffu, ui, L);
        rhs0 = fma(-c0, ui, rhs0);
        rhs1 = fma(-c1, ui, rhs1);
    }
    t[3] = clock64();
    double d0 = lds64(rs0), d1 = lds64(rs0 + 8);
    for (int i = n; i >= 1; --i) {  // V4: loads one iteration ahead
        const int L = i & 31;
        c0 = d0; c1 = d1;
        d0 = lds64(rs0 + 8u * (lane * 65 + ((i - 1) & 63)));
        d1 = lds64(rs0 + 8u * ((lane + 32) * 65 + ((i - 1) & 63)));
        double ui = ((i >> 5) & 1) ? rhs1 * rinv1 : rhs0 * rinv0;
        ui = __shfl_sync(0xffffffffu, ui, L);
        rhs0 = fma(-c0, ui, rhs0);
        rhs1 = fma(-c1, ui, rhs1);
    }
    t[4] = clock64();
    out[threadIdx.x] = rhs0 + rhs1 + u0 + u1 + c0 + c1;
    if (threadIdx.x == 0) for (int i = 0; i < 4; ++i) cyc[i] = (t[i + 1] - t[i]) / n;
}
int main() {
    double* out; long long* cyc;
    cudaMallocManaged(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
    k<<<1, 32>>>(out, cyc, 1000); cudaDeviceSynchronize();
    printf("regs=%lld +select=%lld +lds(same iter)=%lld +lds(prefetched)=%lld\n", cyc[0], cyc[1], cyc[2], cyc[3]);
}
