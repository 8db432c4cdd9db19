// dev ablation of the RQ stage (not product code)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2301_07964_b200/csrc/chase.cuh"
template <typename S, int MAXM, int ABL>
__device__ __forceinline__ void rq_abl(int m, const S* Cb, int LDC, S* ring, volatile int* flag, S* uu) {
    using CF = RQCfg<S, MAXM>;
    constexpr int LPR = CF::LPR, E = CF::E, SB = CF::SB, NSB = CF::NSB, NA = CF::NA, PLD = CF::PLD;
    constexpr int EP = NSB * SB;  // padded elements per thread
    const int tid = threadIdx.x;
    const bool grpB = tid >= NA;
    const int gt = grpB ? tid - NA : tid;
    const int l = gt / LPR, part = gt % LPR;
    const bool live = gt < CF::ROWT && l < m;
    S row[EP];
#pragma unroll
    for (int e = 0; e < EP; ++e) {
        const int c = LPR * e + part;
        S v = S(0.0);
        if (live && e < E && c < m) v = grpB ? S(l == c ? 1.0 : 0.0) : Cb[l + c * LDC];
        row[e] = v;
    }
    auto syncA = [&]() {
        if (NA <= 32) __syncwarp();
        else named_bar(1, NA);
    };
    auto write_pivot = [&](int slot, int upto) {  // this thread's chunk of its row into ring slot
        S* dst = ring + (size_t)slot * PLD + part * EP;
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb)
            if (sb * SB * LPR < upto)
#pragma unroll
                for (int e = 0; e < SB; ++e) dst[sb * SB + e] = row[sb * SB + e];
    };
    // per-stage local work: g, nx (partial over my columns < i), ri
    S bk[EP];
    auto dots = [&](const S* pv, int i, S& g, double& nx, S& ri) {
        const int eth = (i - part + LPR - 1) / LPR;  // my elements e < eth have column < i
        const int sbi = eth / SB;
        double n0 = 0.0, n1 = 0.0;
        S g0 = S(0.0), g1 = S(0.0);
        ri = S(0.0);
        const int ei = (i % LPR == part) ? i / LPR : -1;
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb) {
            if (sb * SB * LPR <= i) {  // uniform: the block holds columns <= i for some part
#pragma unroll
                for (int e = 0; e < SB; ++e) {
                    const int ee = sb * SB + e;
                    const S b = (ee < eth) ? pv[part * EP + ee] : S(0.0);
                    bk[ee] = b;
                    if (e & 1) {
                        n1 += abs2(b);
                        g1 = fma_s(row[ee], conjv(b), g1);
                    } else {
                        n0 += abs2(b);
                        g0 = fma_s(row[ee], conjv(b), g0);
                    }
                    if (ee == ei) ri = row[ee];
                }
            }
        }
        (void)sbi;
        g = g0 + g1;
        nx = n0 + n1;
    };
    auto update = [&](int i, S f) {  // bk (zero for columns >= i) from dots()
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb) {
            if (sb * SB * LPR <= i) {
#pragma unroll
                for (int e = 0; e < SB; ++e) row[sb * SB + e] -= f * bk[sb * SB + e];
            }
        }
    };
    const int ilast = (sizeof(S) == 8) ? 1 : 0;
    if (!grpB) {
        // ---------------- group A: C rows, the sequential chain ----------------
        if (live && l == m - 1) write_pivot(m - 1, m);
        syncA();
        for (int i = m - 1; i >= 1; --i) {
            const S* pv = ring + (size_t)i * PLD;
            const S alpha = conjv(pv[(i % LPR) * EP + i / LPR]);
            S g, ri;
            double nx;
            dots(pv, i, g, nx, ri);
            nx = lpr_sum<double, LPR>(nx);
            g = lpr_sum<S, LPR>(g);
            ri = lpr_sum<S, LPR>(ri);
            S K1 = S(0.0), K2 = S(0.0);
            if (!(nx == 0.0 && im(alpha) == 0.0)) {  // uniform
                const double s2 = abs2(alpha) + nx;
                const double nrm = (ABL & 1) ? s2 * 0.5 : sqrt(s2);
                const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
                K2 = alpha - S(beta);
                if constexpr (sizeof(S) == 8) {
                    K1 = (ABL & 1) ? S(s2 * 0.25 + fabs(re(alpha)) * nrm) : S(1.0 / (s2 + fabs(re(alpha)) * nrm));
                } else {
                    const S tau = (S(beta) - alpha) * (1.0 / beta);
                    K1 = tau * (1.0 / abs2(K2));
                }
            }
            S f = K1 * (g + K2 * ri);
            if (!(live && l < i)) f = S(0.0);
            update(i, f);
            if (gt == 0) {
                ring[(size_t)i * PLD + LPR * EP] = K1;
                ring[(size_t)i * PLD + LPR * EP + 1] = K2;
            }
            if (live && l == i - 1) write_pivot(i - 1, i);
            if (!(ABL & 2)) syncA();
            if (gt == 0) st_release_cta(flag, i);  // stage i (pivot, K1, K2) complete
        }
        if constexpr (sizeof(S) != 8) {
            // stage 0: H_0 = I - tau e1 e1^* makes R~(0,0) real; P rows get row[0] *= (1 - tau)
            const S alpha = conjv(ring[0 * PLD]);
            S tau = S(0.0);
            if (im(alpha) != 0.0) {
                const double nrm = sqrt(abs2(alpha));
                const double beta = (re(alpha) >= 0.0) ? -nrm : nrm;
                tau = (S(beta) - alpha) * (1.0 / beta);
            }
            if (gt == 0) {
                ring[LPR * EP] = tau;
                st_release_cta(flag, 0);
            }
        }
    } else {
        // ---------------- group B: P rows, trailing consumer ----------------
        for (int i = m - 1; i >= ilast; --i) {
            while (ld_acquire_cta(flag) > i) {
            }
            const S* pv = ring + (size_t)i * PLD;
            const S K1 = pv[LPR * EP], K2 = pv[LPR * EP + 1];
            if (i == 0) {  // complex stage 0 (see group A)
                if (live && part == 0) row[0] -= K1 * row[0];
                continue;
            }
            S g, ri;
            double nx;
            dots(pv, i, g, nx, ri);
            g = lpr_sum<S, LPR>(g);
            ri = lpr_sum<S, LPR>(ri);
            S f = K1 * (g + K2 * ri);
            if (!live) f = S(0.0);
            update(i, f);
        }
        if (live && part == 0) uu[l] = row[0];
    }
}


template <int MAXM, int ABL, bool ONLYA>
__global__ void bench(const double* C0, double* out, long long* cyc, int m, int reps) {
    extern __shared__ double dyn[];
    double* Cb = dyn; double* piv = dyn + 64 * 65; double* uu = piv + 64 * 84;
    __shared__ int flag;
    if (threadIdx.x == 0) flag = ONLYA ? -1 : (1 << 30);
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) Cb[(e % m) + (e / m) * (m + 1)] = C0[e];
    __syncthreads();
    const int nthr = ONLYA ? RQCfg<double, MAXM>::NA : RQCfg<double, MAXM>::NTHR;
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (threadIdx.x < nthr) rq_abl<double, MAXM, ABL>(m, Cb, m + 1, piv, &flag, uu);
        __syncthreads();
        if (threadIdx.x == 0) flag = ONLYA ? -1 : (1 << 30);
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
template <int MAXM, int ABL, bool ONLYA>
void run(const char* name, double* C, double* out, long long* cyc, int m) {
    cudaFuncSetAttribute(bench<MAXM, ABL, ONLYA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    bench<MAXM, ABL, ONLYA><<<1, 256, 100000>>>(C, out, cyc, m, 50);
    cudaDeviceSynchronize();
    printf("m=%d %-28s cycles/RQ=%lld per stage=%lld (%s)\n", m, name, cyc[0], cyc[0] / (m - 1), cudaGetErrorString(cudaGetLastError()));
}
int main() {
    double *C, *out; long long* cyc;
    cudaMallocManaged(&C, 64 * 64 * 8); cudaMallocManaged(&out, 64 * 8); cudaMallocManaged(&cyc, 16);
    for (int i = 0; i < 64 * 64; ++i) C[i] = (rand() / (double)RAND_MAX) - 0.5;
    run<16, 0, false>("full", C, out, cyc, 16);
    run<16, 0, true>("groupA only", C, out, cyc, 16);
    run<16, 1, true>("A, fake scalars", C, out, cyc, 16);
    run<16, 3, true>("A, fake scal, no sync", C, out, cyc, 16);
    run<64, 0, false>("full", C, out, cyc, 64);
    run<64, 0, true>("groupA only", C, out, cyc, 64);
    run<64, 1, true>("A, fake scalars", C, out, cyc, 64);
    run<64, 3, true>("A, fake scal, no sync", C, out, cyc, 64);
}
