// ht_stage2.cu -- host orchestration (layer H) and the C ABI (layer A) of the B200-native
// stage-two Hessenberg-triangular reduction.  See include/ht_stage2.h for the contract and
// DESIGN.md for the decomposition.  Everything on the data path runs in the kernels of
// chase.cuh (K1), chain.cuh (K3/K4) and misc.cuh (K5); the host only launches them.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/ht_stage2.h"
#include "chain.cuh"
#include "chase.cuh"
#include "misc.cuh"
#include "scalar.cuh"

namespace {

enum { HT_OK = 0, HT_ESTRUCT = 1, HT_ENONFINITE = 2, HT_ECUDA = 3, HT_ENCCL = 4, HT_ENOMEM = 5,
       HT_EUNSUPPORTED = 6 };

thread_local double g_last_ms[4] = {0, 0, 0, 0};
thread_local int64_t g_last_launches = 0;

constexpr int CHASE_NT = 256;
constexpr int CHAIN_NT = 256;
constexpr int ROW_BM = 64;
constexpr int COL_BN = 64;

struct Timer {
    bool on = false;
    cudaStream_t s = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    float acc = 0;
};

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            if (getenv("HT_DEBUG")) fprintf(stderr, "ht_stage2: %s at %s:%d\n",   \
                                            cudaGetErrorString(e_), __FILE__, __LINE__); \
            return e_ == cudaErrorMemoryAllocation ? HT_ENOMEM : HT_ECUDA;        \
        }                                                                         \
    } while (0)

int64_t default_q(int64_t n, int64_t r, int is_complex) {
    (void)is_complex;
    const char* env = getenv("HT_Q");
    if (env && atoll(env) > 0) return atoll(env);
    int64_t q = r;  // executed/useful flops of dense U/V ~ (q+r-1)^2/(2qr), minimal at q ~ r
    if (q < 8) q = 8;
    if (q > 64) q = 64;
    return std::max<int64_t>(1, std::min<int64_t>(q, std::max<int64_t>(1, n - 2)));
}

template <typename S>
size_t row_chain_smem(int W) { return ((size_t)2 * ROW_BM * W + (size_t)W * W) * sizeof(S); }
template <typename S>
size_t col_chain_smem(int W) { return ((size_t)2 * (W + 1) * COL_BN + (size_t)W * W) * sizeof(S); }

template <typename S>
int set_smem_attrs(size_t chase_bytes, size_t row_bytes, size_t col_bytes) {
    CK(cudaFuncSetAttribute(chase_kernel<S, CHASE_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)chase_bytes));
    CK(cudaFuncSetAttribute(row_chain_kernel<S, ROW_BM, CHAIN_NT, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_bytes));
    CK(cudaFuncSetAttribute(row_chain_kernel<S, ROW_BM, CHAIN_NT, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_bytes));
    CK(cudaFuncSetAttribute(col_chain_kernel<S, COL_BN, CHAIN_NT>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)col_bytes));
    return HT_OK;
}

template <typename S>
int run(int64_t n64, int64_t r64, S* H, int64_t ldh, S* T, int64_t ldt, S* Q, int64_t ldq, S* Z,
        int64_t ldz, cudaStream_t stream, ncclComm_t comm, const ht_opts* opts, bool is_complex) {
    g_last_launches = 0;
    for (double& x : g_last_ms) x = 0;
    // ---- synchronous argument checks (-i = argument i) ----
    if (n64 < 0) return -1;
    if (r64 < 0) return -2;
    if (!H && n64 > 0) return -3;
    if (ldh < std::max<int64_t>(1, n64)) return -4;
    if (!T && n64 > 0) return -5;
    if (ldt < std::max<int64_t>(1, n64)) return -6;
    if (Q && ldq < std::max<int64_t>(1, n64)) return -8;
    if (Z && ldz < std::max<int64_t>(1, n64)) return -10;
    if (n64 > (1 << 30)) return -1;
    if (comm != nullptr) return HT_EUNSUPPORTED;  // multi-GPU path: see DESIGN.md (next)
    if (n64 == 0) return HT_OK;
    for (void* p : {(void*)H, (void*)T, (void*)Q, (void*)Z}) {
        if (!p) continue;
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            return p == (void*)H ? -3 : p == (void*)T ? -5 : p == (void*)Q ? -7 : -9;
        }
    }
    const int n = (int)n64;
    const int r = (int)std::min<int64_t>(r64, std::max<int64_t>(1, n64));
    Timer tm;
    tm.on = getenv("HT_PROFILE") != nullptr;
    cudaEvent_t e_start, e_end;
    CK(cudaEventCreate(&e_start));
    CK(cudaEventCreate(&e_end));
    CK(cudaEventRecord(e_start, stream));

    // ---- K5: input validation (exact structure + finiteness), host blocks once ----
    if (!(opts && (opts->flags & HT_FLAG_NO_VALIDATE))) {
        unsigned long long* flags = nullptr;
        CK(cudaMallocAsync(&flags, 2 * sizeof(unsigned long long), stream));
        CK(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned long long), stream));
        validate_kernel<S><<<4 * 148, 256, 0, stream>>>(n, r, H, ldh, T, ldt, Q, ldq, Z, ldz, flags);
        ++g_last_launches;
        CK(cudaGetLastError());
        unsigned long long hf[2] = {0, 0};
        CK(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, stream));
        CK(cudaFreeAsync(flags, stream));
        CK(cudaStreamSynchronize(stream));
        if (hf[0]) return HT_ESTRUCT;
        if (hf[1]) return HT_ENONFINITE;
    }
    if (n <= 2 || r <= 1) return HT_OK;  // exact no-op

    int64_t q64 = (opts && opts->q > 0) ? opts->q : default_q(n, r, is_complex);
    const int q = (int)std::max<int64_t>(1, std::min<int64_t>(q64, n - 2));
    const int W = q + r - 1;
    const int Kmax = 1 + (n - 1 - 2) / r;
    const size_t chase_bytes = chase_smem_elems<S>(r, W) * sizeof(S);
    const size_t row_bytes = row_chain_smem<S>(W), col_bytes = col_chain_smem<S>(W);
    int dev = 0, smem_optin = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (chase_bytes > (size_t)smem_optin || row_bytes > (size_t)smem_optin ||
        col_bytes > (size_t)smem_optin)
        return HT_EUNSUPPORTED;
    if (int rc = set_smem_attrs<S>(chase_bytes, row_bytes, col_bytes)) return rc;

    // ---- workspace (stream-ordered) ----
    S *U = nullptr, *V = nullptr, *Zr = nullptr;
    int* prog = nullptr;
    const size_t blk_elems = (size_t)Kmax * W * W;
    CK(cudaMallocAsync(&U, blk_elems * sizeof(S), stream));
    CK(cudaMallocAsync(&V, blk_elems * sizeof(S), stream));
    CK(cudaMallocAsync(&Zr, (size_t)q * Kmax * (r + 1) * sizeof(S), stream));
    CK(cudaMallocAsync(&prog, (size_t)q * sizeof(int), stream));

    const int chase_ctas_req = (opts && opts->chase_ctas > 0) ? opts->chase_ctas : 32;
    cudaEvent_t ev[8];
    if (tm.on)
        for (auto& e : ev) CK(cudaEventCreate(&e));
    float ms_chase = 0, ms_ht = 0, ms_qz = 0;

    for (int j1 = 1; j1 <= n - 2; j1 += q) {
        const int qp = std::min(q, n - 1 - j1);
        const int K = 1 + (n - j1 - 2) / r;
        if (tm.on) CK(cudaEventRecord(ev[0], stream));
        init_blocks_kernel<S><<<std::min<int64_t>(4 * nsm, ((int64_t)K * W * W + 255) / 256), 256, 0,
                                stream>>>(U, V, K, W);
        CK(cudaMemsetAsync(prog, 0, (size_t)q * sizeof(int), stream));
        ChaseArgs<S> ca{n, r, qp, j1, K, W, H, ldh, T, ldt, U, V, Zr, prog};
        const int P = std::max(1, std::min({qp, chase_ctas_req, nsm}));
        void* kargs[] = {&ca};
        CK(cudaLaunchCooperativeKernel((const void*)chase_kernel<S, CHASE_NT>, dim3(P), dim3(CHASE_NT),
                                       kargs, chase_bytes, stream));
        g_last_launches += 2;
        if (tm.on) CK(cudaEventRecord(ev[1], stream));
        // ---- apply phase: right updates of H, T (staircase + V_k), then left (U_k^*) ----
        ChainArgs<S> ab{n, r, qp, j1, K, W, H, ldh, T, ldt, V, V, Zr, 0};
        row_chain_kernel<S, ROW_BM, CHAIN_NT, true>
            <<<dim3((n + ROW_BM - 1) / ROW_BM, 2), CHAIN_NT, row_bytes, stream>>>(ab);
        ChainArgs<S> lf{n, r, qp, j1, K, W, H, ldh, T, ldt, U, U, nullptr, 0};
        col_chain_kernel<S, COL_BN, CHAIN_NT>
            <<<dim3((n + COL_BN - 1) / COL_BN, 2), CHAIN_NT, col_bytes, stream>>>(lf);
        g_last_launches += 2;
        if (tm.on) CK(cudaEventRecord(ev[2], stream));
        // ---- Q <- Q U_k, Z <- Z V_k (row chains; never read by the chase) ----
        if (Q || Z) {
            ChainArgs<S> qz{n, r, qp, j1, K, W, Q ? Q : Z, Q ? ldq : ldz, Z ? Z : Q, Z ? ldz : ldq,
                            Q ? U : V, Z ? V : U, nullptr, 0};
            row_chain_kernel<S, ROW_BM, CHAIN_NT, false>
                <<<dim3((n + ROW_BM - 1) / ROW_BM, (Q && Z) ? 2 : 1), CHAIN_NT, row_bytes, stream>>>(qz);
            ++g_last_launches;
        }
        CK(cudaGetLastError());
        if (tm.on) {
            CK(cudaEventRecord(ev[3], stream));
            CK(cudaEventSynchronize(ev[3]));
            float a = 0, b = 0, c = 0;
            CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
            CK(cudaEventElapsedTime(&b, ev[1], ev[2]));
            CK(cudaEventElapsedTime(&c, ev[2], ev[3]));
            ms_chase += a;
            ms_ht += b;
            ms_qz += c;
        }
    }
    CK(cudaFreeAsync(U, stream));
    CK(cudaFreeAsync(V, stream));
    CK(cudaFreeAsync(Zr, stream));
    CK(cudaFreeAsync(prog, stream));
    CK(cudaEventRecord(e_end, stream));
    if (tm.on) {
        CK(cudaEventSynchronize(e_end));
        float tot = 0;
        CK(cudaEventElapsedTime(&tot, e_start, e_end));
        g_last_ms[0] = ms_chase;
        g_last_ms[1] = ms_ht;
        g_last_ms[2] = ms_qz;
        g_last_ms[3] = tot;
        for (auto& e : ev) cudaEventDestroy(e);
    }
    cudaEventDestroy(e_start);
    cudaEventDestroy(e_end);
    CK(cudaGetLastError());
    return HT_OK;
}

}  // namespace

extern "C" {

int ht_stage2_d_ex(int64_t n, int64_t r, double* H, int64_t ldh, double* T, int64_t ldt, double* Q,
                   int64_t ldq, double* Z, int64_t ldz, cudaStream_t stream, ncclComm_t comm,
                   const ht_opts* opts) {
    return run<double>(n, r, H, ldh, T, ldt, Q, ldq, Z, ldz, stream, comm, opts, false);
}

int ht_stage2_z_ex(int64_t n, int64_t r, cuDoubleComplex* H, int64_t ldh, cuDoubleComplex* T,
                   int64_t ldt, cuDoubleComplex* Q, int64_t ldq, cuDoubleComplex* Z, int64_t ldz,
                   cudaStream_t stream, ncclComm_t comm, const ht_opts* opts) {
    static_assert(sizeof(zc) == sizeof(cuDoubleComplex), "zc layout");
    return run<zc>(n, r, reinterpret_cast<zc*>(H), ldh, reinterpret_cast<zc*>(T), ldt,
                   reinterpret_cast<zc*>(Q), ldq, reinterpret_cast<zc*>(Z), ldz, stream, comm, opts,
                   true);
}

int ht_stage2_d(int64_t n, int64_t r, double* H, int64_t ldh, double* T, int64_t ldt, double* Q,
                int64_t ldq, double* Z, int64_t ldz, cudaStream_t stream, ncclComm_t comm) {
    return ht_stage2_d_ex(n, r, H, ldh, T, ldt, Q, ldq, Z, ldz, stream, comm, nullptr);
}

int ht_stage2_z(int64_t n, int64_t r, cuDoubleComplex* H, int64_t ldh, cuDoubleComplex* T,
                int64_t ldt, cuDoubleComplex* Q, int64_t ldq, cuDoubleComplex* Z, int64_t ldz,
                cudaStream_t stream, ncclComm_t comm) {
    return ht_stage2_z_ex(n, r, H, ldh, T, ldt, Q, ldq, Z, ldz, stream, comm, nullptr);
}

int ht_nccl_unique_id(void* id_out) {
    if (!id_out) return -1;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return HT_ENCCL;
    memcpy(id_out, &id, sizeof(id));
    return HT_OK;
}

int ht_comm_create(const void* id, int rank, int nranks, ncclComm_t* out) {
    if (!id) return -1;
    if (rank < 0 || rank >= nranks) return -2;
    if (nranks < 1) return -3;
    if (!out) return -4;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    return ncclCommInitRank(out, nranks, uid, rank) == ncclSuccess ? HT_OK : HT_ENCCL;
}

int ht_comm_destroy(ncclComm_t comm) {
    if (!comm) return HT_OK;
    return ncclCommDestroy(comm) == ncclSuccess ? HT_OK : HT_ENCCL;
}

const char* ht_strerror(int code) {
    if (code < 0) return "invalid argument (-code = 1-based argument position)";
    switch (code) {
        case 0: return "success";
        case 1: return "input violates r-Hessenberg-triangular structure";
        case 2: return "input contains a non-finite value";
        case 3: return "CUDA error";
        case 4: return "NCCL error";
        case 5: return "out of device memory";
        case 6: return "unsupported configuration in this build";
        default: return "unknown error";
    }
}

double ht_flops_std(int64_t n, int is_complex) {
    const double d = (double)n;
    return (is_complex ? 40.0 : 10.0) * d * d * d;
}

int64_t ht_default_q(int64_t n, int64_t r, int is_complex) { return default_q(n, r, is_complex); }

int ht_last_timing(double* ms_out4, int64_t* launches_out) {
    if (ms_out4)
        for (int i = 0; i < 4; ++i) ms_out4[i] = g_last_ms[i];
    if (launches_out) *launches_out = g_last_launches;
    return HT_OK;
}

static double probe(bool dmma, int iters) {
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1;
    const int blocks = nsm * 4, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    if (dmma) probe_dmma_kernel<<<blocks, threads>>>(iters / 10 + 1, out);
    else probe_dfma_kernel<<<blocks, threads>>>(iters / 10 + 1, out);
    cudaEventRecord(a);
    if (dmma) probe_dmma_kernel<<<blocks, threads>>>(iters, out);
    else probe_dfma_kernel<<<blocks, threads>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess || ms <= 0) return -1;
    const double flops = dmma ? (double)blocks * (threads / 32) * iters * 8.0 * 512.0
                              : (double)blocks * threads * iters * 8.0 * 2.0;
    return flops / (ms * 1e-3) / 1e12;
}

double ht_probe_dmma_tflops(int iters) { return probe(true, iters); }
double ht_probe_dfma_tflops(int iters) { return probe(false, iters); }

}  // extern "C"
