// dev check + micro-benchmark (not product code): the warp-row RQ (rqw.cuh) against the
// register RQ of chase.cuh on random, graded and singular m x m blocks: direction residual
// ||B(2:m,:) u|| / ||B||, |u| = 1, agreement with the old kernel's u, and cycles per RQ.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/rqw_test tools/rqw_test.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#ifndef REPS
#define REPS 10
#endif

#include "../paper_2301_07964_b200/csrc/chase.cuh"
#include "../paper_2301_07964_b200/csrc/rqw.cuh"

template <int MAXM, bool NEW>
__global__ void run(const double* C0, double* out, long long* cyc, int m, int reps) {
    extern __shared__ double dyn[];
    const int LDC = MAXM + 1, HLD = MAXM + 4;
    double* Cb = dyn;  // (MAXM = 128: the work rows overlay the block, as in the chase kernel)
    double* hb = MAXM > 64 ? Cb : Cb + MAXM * LDC;
    double* uu = hb + MAXM * HLD;
    __shared__ int flag;
    __shared__ uint64_t bars[128];
    if (threadIdx.x < 32) rqw_bars_init(bars, 128);
    __syncthreads();
    long long tot = 0;
    for (int it = 0; it < reps; ++it) {
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) Cb[(e % m) + (e / m) * LDC] = C0[e];
        if (threadIdx.x == 0) flag = 1 << 30;
        __syncthreads();
        long long t0 = clock64();
        if constexpr (NEW) {
            rq_direction_w<double, MAXM, 8>(m, Cb, LDC, hb, HLD, bars, it & 1, uu);
        } else {
            if (threadIdx.x < RQCfg<double, MAXM>::NTHR) rq_direction<double, MAXM>(m, Cb, LDC, hb, &flag, uu);
        }
        __syncthreads();
        tot += clock64() - t0;
    }
    if (threadIdx.x < m) out[threadIdx.x] = uu[threadIdx.x];
    if (threadIdx.x == 0) cyc[0] = tot / reps;
}

template <int MAXM, bool NEW>
void launch(const double* C, double* out, long long* cyc, int m, int reps) {
    const int bytes = ((MAXM > 64 ? 0 : MAXM * (MAXM + 1)) + MAXM * (MAXM + 4) + MAXM + 8) * 8;
    cudaFuncSetAttribute(run<MAXM, NEW>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    const int nt = NEW ? 256 : (RQCfg<double, MAXM>::NTHR > 256 ? RQCfg<double, MAXM>::NTHR : 256);
    run<MAXM, NEW><<<1, nt, bytes>>>(C, out, cyc, m, reps);
}

int main() {
    struct Case { int maxm, m, kind; };  // kind 0 random, 1 graded diag-dominant, 2 singular
    std::vector<Case> cases = {{64, 64, 0}, {64, 37, 0}, {64, 2, 0}, {64, 64, 1}, {64, 64, 2},
                               {128, 128, 0}, {128, 100, 0}, {128, 65, 0}, {128, 128, 1}, {128, 128, 2}};
    int bad = 0;
    for (auto cs : cases) {
        const int m = cs.m;
        double *C, *o1, *o2;
        long long *c1, *c2;
        cudaMallocManaged(&C, m * m * 8);
        cudaMallocManaged(&o1, 128 * 8);
        cudaMallocManaged(&o2, 128 * 8);
        cudaMallocManaged(&c1, 16);
        cudaMallocManaged(&c2, 16);
        srand(1234 + m + cs.kind);
        for (int i = 0; i < m * m; ++i) C[i] = (rand() / (double)RAND_MAX) - 0.5;
        if (cs.kind == 1)  // upper triangular-ish with graded diagonal + small fill
            for (int j = 0; j < m; ++j)
                for (int i = 0; i < m; ++i) {
                    if (i > j) C[i + j * m] *= 1e-3;
                    if (i == j) C[i + j * m] = pow(10.0, -3.0 * (rand() / (double)RAND_MAX));
                }
        if (cs.kind == 2)  // exactly singular: upper triangular with zero diagonal entries
            for (int j = 0; j < m; ++j)
                for (int i = 0; i < m; ++i) {
                    if (i > j) C[i + j * m] = 0.0;
                    if (i == j && j % 5 == 2) C[i + j * m] = 0.0;
                }
        if (cs.maxm == 64) {
            launch<64, true>(C, o1, c1, m, REPS);
            launch<64, false>(C, o2, c2, m, 10);
        } else {
            launch<128, true>(C, o1, c1, m, REPS);
            launch<128, false>(C, o2, c2, m, 10);
        }
        cudaError_t err = cudaDeviceSynchronize();
        double res1 = 0, res2 = 0, n1 = 0, n2 = 0, nc = 0, diff = 0;
        for (int i = 0; i < m; ++i) {
            n1 += o1[i] * o1[i];
            n2 += o2[i] * o2[i];
            diff += (o1[i] - o2[i]) * (o1[i] - o2[i]);
        }
        for (int i = 1; i < m; ++i) {
            double s1 = 0, s2 = 0;
            for (int c = 0; c < m; ++c) {
                s1 += C[i + c * m] * o1[c];
                s2 += C[i + c * m] * o2[c];
            }
            res1 += s1 * s1;
            res2 += s2 * s2;
        }
        for (int i = 0; i < m * m; ++i) nc += C[i] * C[i];
        const double r1 = sqrt(res1 / nc), r2 = sqrt(res2 / nc);
        const bool ok = err == cudaSuccess && fabs(sqrt(n1) - 1) < 1e-13 && r1 < 1e-14 * m;
        bad += !ok;
        printf("MAXM=%d m=%d kind=%d new: %lld cyc |u|-1=%.1e res=%.2e | old: %lld cyc |u|-1=%.1e res=%.2e | "
               "|u_new-u_old|=%.2e %s %s\n",
               cs.maxm, m, cs.kind, c1[0], sqrt(n1) - 1, r1, c2[0], sqrt(n2) - 1, r2, sqrt(diff),
               cudaGetErrorString(err), ok ? "OK" : "FAIL");
        cudaFree(C);
        cudaFree(o1);
        cudaFree(o2);
        cudaFree(c1);
        cudaFree(c2);
    }
    printf("%s\n", bad ? "SOME FAILED" : "ALL OK");
    return bad != 0;
}
