// dev micro-benchmark: dependent-chain latencies of the RQ-update chain's building blocks (sm_100a)
#include <cstdio>
#include "rqu.cuh"
__global__ void lat(double* out, long long* cyc, double x0, int n) {
    double a = x0 + threadIdx.x * 1e-9, b = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, 1e-9);
    long long t1 = clock64();
    double r = a;
    for (int i = 0; i < n; ++i) r = fast_rsqrt(r + 1.5);
    long long t2 = clock64();
    double s = r;
    for (int i = 0; i < n; ++i) s = __shfl_sync(0xffffffffu, s, (i + 1) & 31) + 1e-9;
    long long t3 = clock64();
    double c = s, ss = 0.3;
    for (int i = 0; i < n; ++i) { double c2, s2; giv_rot(c + 0.5, ss + 0.25, c2, s2); c = c2; ss = s2; }
    long long t4 = clock64();
    double m = ss;
    for (int i = 0; i < n; ++i) m = m * b;
    long long t5 = clock64();
    float f = (float)m;
    for (int i = 0; i < n; ++i) f = fmaf(f, 1.0001f, 1e-7f);
    long long t6 = clock64();
    out[threadIdx.x] = a + r + s + c + m + f;
    if (threadIdx.x == 0) { cyc[0] = (t1-t0)/n; cyc[1] = (t2-t1)/n; cyc[2] = (t3-t2)/n; cyc[3] = (t4-t3)/n; cyc[4] = (t5-t4)/n; cyc[5] = (t6-t5)/n; }
}
int main() {
    double* out; long long* cyc;
    cudaMallocManaged(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
    for (int w = 1; w <= 8; w *= 8) {
        lat<<<1, 32 * w>>>(out, cyc, 1.0, 2000); cudaDeviceSynchronize();
        printf("warps=%d dfma=%lld fast_rsqrt+dadd=%lld shfl64+dadd=%lld giv_rot(+2 dadd)=%lld dmul=%lld ffma=%lld cycles\n", w, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
    }
}
