// dev micro-benchmark: single-warp latencies on sm_100a (not product code)
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double x0, int n) {
    __shared__ double sh[64];
    double a = x0, b = 1.0000001;
    if (threadIdx.x < 64) sh[threadIdx.x] = threadIdx.x * 1e-3;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, 1e-9);
    long long t1 = clock64();
    double s = a;
    for (int i = 0; i < n; ++i) s = 1.0 / (s + 2.0);
    long long t2 = clock64();
    double q = s + 3;
    for (int i = 0; i < n; ++i) q = sqrt(q + 2.0);
    long long t3 = clock64();
    int idx = (int)q & 7;
    double v = 0;
    for (int i = 0; i < n; ++i) { v += sh[idx]; idx = ((int)v) & 7; }
    long long t4 = clock64();
    float f = (float)v;
    for (int i = 0; i < n; ++i) f = fmaf(f, 1.0001f, 1e-7f);
    long long t5 = clock64();
    out[threadIdx.x] = a + s + q + v + f;
    if (threadIdx.x == 0) { cyc[0] = (t1-t0)/n; cyc[1] = (t2-t1)/n; cyc[2] = (t3-t2)/n; cyc[3] = (t4-t3)/n; cyc[4] = (t5-t4)/n; }
}
int main() {
    double* out; long long* cyc;
    cudaMallocManaged(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
    for (int w = 1; w <= 8; w *= 8) {
        lat<<<1, 32 * w>>>(out, cyc, 1.0, 1000); cudaDeviceSynchronize();
        printf("warps=%d dfma=%lld div=%lld sqrt=%lld lds+dadd=%lld ffma=%lld cycles\n", w, cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
    }
}
