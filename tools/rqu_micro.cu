// rqu_micro.cu -- isolated timing + check of K1's RQ update (rqu.cuh) on one CTA (dev tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2301_07964_b200/csrc
//        -o tools/rqu_micro tools/rqu_micro.cu
//   tools/rqu_micro [m] [iters]
// Checks R~ Q~ = (R0 - v w^T) Q0 (w = tau R0^T v), Q~ Q~^T = I, R~ upper triangular, and prints
// cycles per call of the phases (A, B+C, D + Q tail) measured by thread 0.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rqu.cuh"

#ifndef MAXM_
#define MAXM_ 64
#endif
constexpr int NT = 256, MAXM = MAXM_;
using CF = RQUCfg<NT, MAXM>;

__global__ void micro(int mode, int m, int iters, const double* R0, const double* Q0, const double* v, double tau, double* Rout,
                      double* Qout, double* uout, long long* cyc) {
    extern __shared__ double sm[];
    constexpr int RLD = CF::RLD;
    double* Rs = sm;
    double* Qs = Rs + (CF::QCONC ? MAXM * RLD : 0);
    double* wpart = Qs + MAXM * RLD;
    double* cs1 = wpart + CF::NPART * MAXM;
    double* cs2 = cs1 + 2 * MAXM;
    double* vs = cs2 + 2 * MAXM;
    double* uu = vs + MAXM;
    double* xs = uu + MAXM;
    __shared__ int okf;
    long long pt[24] = {};
    long long tc = 0;
    for (int i = threadIdx.x; i < m; i += NT) vs[i] = v[i];
    for (int i = threadIdx.x; i < MAXM; i += NT) cs2[2 * i] = RQU_SENTINEL;
    for (int it = 0; it < iters; ++it) {
        for (int e = threadIdx.x; e < m * m; e += NT) {
            const int p = e / m, c = e % m;
            Rs[p * RLD + c] = R0[p * m + c];
            if (CF::QCONC) Qs[p * RLD + c] = Q0[p * m + c];
        }
        __syncthreads();
        tc = clock64();
        if (mode == 1) {
            rqu_direction<NT, MAXM>(m, vs, tau, Rs, Qs, wpart, cs1, cs2, uu, pt, &tc);
        } else {
            rqu_solve<NT, MAXM>(m, vs, tau, Rs, Qs, wpart, xs, uu, &okf, pt, &tc, CF::QCONC ? nullptr : Q0, false);
            __syncthreads();
        }
    }
    for (int e = threadIdx.x; e < m * m; e += NT) {
        const int p = e / m, c = e % m;
        Rout[p * m + c] = Rs[p * RLD + c];
        Qout[p * m + c] = Qs[p * RLD + c];
    }
    for (int i = threadIdx.x; i < m; i += NT) uout[i] = uu[i];
    if (threadIdx.x == 0)
        for (int i = 0; i < 24; ++i) cyc[i] = pt[i];
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 64;
    const int iters = argc > 2 ? atoi(argv[2]) : 200;
    const int mode = argc > 3 ? atoi(argv[3]) : 1;
    srand(7);
    auto rnd = [] { return 2.0 * rand() / RAND_MAX - 1.0; };
    std::vector<double> R0(m * m, 0.0), Q0(m * m, 0.0), v(m), Rt(m * m), Qt(m * m), uu(m);
    for (int p = 0; p < m; ++p)
        for (int c = p; c < m; ++c) R0[p * m + c] = rnd() + (p == c ? 2.0 : 0.0);
    // Q0: product of a few random reflectors (orthogonal)
    for (int i = 0; i < m; ++i) Q0[i * m + i] = 1.0;
    for (int h = 0; h < 4; ++h) {
        std::vector<double> x(m);
        double nn = 0;
        for (auto& t : x) nn += (t = rnd()) * t;
        for (int c = 0; c < m; ++c) {
            double d = 0;
            for (int i = 0; i < m; ++i) d += x[i] * Q0[i * m + c];
            for (int i = 0; i < m; ++i) Q0[i * m + c] -= 2.0 * x[i] * d / nn;
        }
    }
    // v, tau of a larfg
    std::vector<double> x(m);
    double s = 0;
    for (int i = 0; i < m; ++i) x[i] = rnd();
    for (int i = 1; i < m; ++i) s += x[i] * x[i];
    const double nrm = sqrt(x[0] * x[0] + s), beta = x[0] >= 0 ? -nrm : nrm, tau = (beta - x[0]) / beta;
    v[0] = 1.0;
    for (int i = 1; i < m; ++i) v[i] = x[i] / (x[0] - beta);
    double *dR, *dQ, *dv, *dRo, *dQo, *du;
    long long* dc;
    cudaMalloc(&dR, m * m * 8);
    cudaMalloc(&dQ, m * m * 8);
    cudaMalloc(&dv, m * 8);
    cudaMalloc(&dRo, m * m * 8);
    cudaMalloc(&dQo, m * m * 8);
    cudaMalloc(&du, m * 8);
    cudaMalloc(&dc, 24 * 8);
    cudaMemcpy(dR, R0.data(), m * m * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dQ, Q0.data(), m * m * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), m * 8, cudaMemcpyHostToDevice);
    const size_t smem = ((CF::QCONC ? 2 : 1) * MAXM * CF::RLD + CF::NPART * MAXM + 4 * MAXM + 3 * MAXM + 2) * 8;
    cudaFuncSetAttribute(micro, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    micro<<<1, NT, smem>>>(mode, m, iters, dR, dQ, dv, tau, dRo, dQo, du, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
    }
    long long cyc[24];
    cudaMemcpy(Rt.data(), dRo, m * m * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(Qt.data(), dQo, m * m * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(uu.data(), du, m * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(cyc, dc, 24 * 8, cudaMemcpyDeviceToHost);
    // check: M Q0 = R~ Q~ with M = R0 - v w^T
    std::vector<double> w(m, 0.0);
    for (int c = 0; c < m; ++c)
        for (int p = 0; p <= c; ++p) w[c] += tau * R0[p * m + c] * v[p];
    double err = 0, ref = 0, orth = 0, low = 0, urow = 0;
    for (int p = 0; p < m; ++p)
        for (int c = 0; c < m; ++c) {
            double a = 0, b = 0, o = 0;
            for (int k = 0; k < m; ++k) {
                a += (R0[p * m + k] - v[p] * w[k]) * Q0[k * m + c];
                if (k >= p) b += Rt[p * m + k] * Qt[k * m + c];
                o += Qt[p * m + k] * Qt[c * m + k];
            }
            err += (a - b) * (a - b);
            ref += a * a;
            orth += (o - (p == c)) * (o - (p == c));
        }
    if (mode == 2) {  // uu = Q0^T x unnormalised: the residual of rows 2..m of M Q0 applied to uu
        double nu = 0, res = 0, nM = 0;
        for (int c = 0; c < m; ++c) nu += uu[c] * uu[c];
        for (int p = 1; p < m; ++p) {
            double d = 0;
            for (int c = 0; c < m; ++c) {
                double mc = 0;
                for (int k = 0; k < m; ++k) mc += (R0[p * m + k] - v[p] * w[k]) * Q0[k * m + c];
                d += mc * uu[c];
                nM += mc * mc;
            }
            res += d * d;
        }
        printf("mode 2 (solve): ||M(2:m,:) Q0 z|| / (||M|| ||z||) = %.2e\n", sqrt(res / nu / nM));
        printf("cycles per call: A=%.0f solve=%.0f Qx=%.0f total=%.0f\n", (double)cyc[17] / iters, (double)cyc[18] / iters,
               (double)cyc[19] / iters, (double)cyc[6] / iters);
        return 0;
    }
    for (int c = 0; c < m; ++c) urow += (uu[c] - Qt[c]) * (uu[c] - Qt[c]);
    (void)low;
    printf("m=%d iters=%d  ||M Q0 - R~Q~||/||M Q0|| = %.2e  ||Q~Q~^T - I|| = %.2e  |uu - Q~(0,:)| = %.1e\n", m, iters,
           sqrt(err / ref), sqrt(orth), sqrt(urow));
    printf("cycles per call: A=%.0f BC=%.0f D=%.0f Qtail+sync=%.0f total=%.0f\n", (double)cyc[17] / iters, (double)cyc[18] / iters,
           (double)cyc[21] / iters, (double)cyc[19] / iters, (double)cyc[6] / iters);
    return 0;
}
