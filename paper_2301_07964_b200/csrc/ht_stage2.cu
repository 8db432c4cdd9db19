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
#include <vector>

#include "../../include/ht_stage2.h"
#include "chase.cuh"
#include "chain.cuh"
#include "accum.cuh"
#include "misc.cuh"
#include "scalar.cuh"

namespace {

enum { HT_OK = 0, HT_ESTRUCT = 1, HT_ENONFINITE = 2, HT_ECUDA = 3, HT_ENCCL = 4, HT_ENOMEM = 5,
       HT_EUNSUPPORTED = 6 };

thread_local double g_last_ms[4] = {0, 0, 0, 0};
thread_local int64_t g_last_launches = 0;

constexpr int CHASE_NT = 256;


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

template <typename S, int WP>
size_t chain_bytes(int r, int q) { return chain_smem_bytes<S, WP>(r, q); }

template <typename S, int WP>
int launch_chain(const ChainParams<S>& P, int grid, int r, int q, cudaStream_t st) {
    const size_t bytes = chain_bytes<S, WP>(r, q);
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        CK(cudaFuncSetAttribute(chain_kernel<S, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_set = true;
    }
    chain_kernel<S, WP><<<grid, CH_NT, bytes, st>>>(P);
    CK(cudaGetLastError());
    return HT_OK;
}

template <typename S>
int chain(const ChainParams<S>& P, int WP, int grid, int r, int q, cudaStream_t st) {
    switch (WP) {
        case 32: return launch_chain<S, 32>(P, grid, r, q, st);
        case 64: return launch_chain<S, 64>(P, grid, r, q, st);
        case 96: return launch_chain<S, 96>(P, grid, r, q, st);
        case 128: return launch_chain<S, 128>(P, grid, r, q, st);
        case 160: return launch_chain<S, 160>(P, grid, r, q, st);
        default: return HT_EUNSUPPORTED;
    }
}

template <typename S>
size_t chain_bytes_rt(int WP, int r, int q) {
    switch (WP) {
        case 32: return chain_bytes<S, 32>(r, q);
        case 64: return chain_bytes<S, 64>(r, q);
        case 96: return chain_bytes<S, 96>(r, q);
        case 128: return chain_bytes<S, 128>(r, q);
        case 160: return chain_bytes<S, 160>(r, q);
        default: return (size_t)1 << 40;
    }
}

// K1 instantiation for the reflector length (the RQ keeps [C; P] rows in registers)
template <typename S>
const void* chase_kernel_for(int r) {
    if (r <= 8) return (const void*)chase_kernel<S, CHASE_NT, 8>;
    if (r <= 16) return (const void*)chase_kernel<S, CHASE_NT, 16>;
    if (r <= 32) return (const void*)chase_kernel<S, CHASE_NT, 32>;
    if constexpr (sizeof(S) == 8) {
        if (r <= 64) return (const void*)chase_kernel<S, CHASE_NT, 64>;
    }
    return nullptr;
}

constexpr int ACC_NT = 256;

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
    const bool prof = getenv("HT_PROFILE") != nullptr || (opts && (opts->flags & HT_FLAG_PROFILE));
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
    const int w = q + r - 1;
    const int WP = (w + 31) / 32 * 32;  // padded window order (DMMA tiles, ring chunks)
    const int LDB = chain_ldb(WP);
    const int Kmax = 1 + (n - 1 - 2) / r;
    const int chase_budget = 200 * 1024;
    const size_t chase_base = chase_smem_elems<S>(r, q, 0) * sizeof(S);
    const int strip_cap = (int)std::max<int64_t>(0, ((int64_t)chase_budget - (int64_t)chase_base) /
                                                        (int64_t)((r + 1) * sizeof(S)));
    const size_t chase_bytes = chase_smem_elems<S>(r, q, strip_cap) * sizeof(S);
    const size_t acc_bytes = accum_smem_bytes<S>(r, q);
    const void* chase_fn = chase_kernel_for<S>(r);
    if (!chase_fn || q > 148) return HT_EUNSUPPORTED;  // one co-resident CTA per sweep
    const size_t ch_bytes = chain_bytes_rt<S>(WP, r, q);
    int dev = 0, smem_optin = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (chase_bytes > (size_t)smem_optin || ch_bytes > (size_t)smem_optin || acc_bytes > (size_t)smem_optin)
        return HT_EUNSUPPORTED;
    CK(cudaFuncSetAttribute(chase_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chase_bytes));
    CK(cudaFuncSetAttribute(accum_kernel<S, ACC_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)acc_bytes));

    // ---- workspace (stream-ordered) ----
    S *U = nullptr, *V = nullptr, *Zr = nullptr, *Qr = nullptr, *Tr = nullptr;
    int* prog = nullptr;
    const size_t blk_elems = (size_t)Kmax * WP * LDB;
    const size_t rec_elems = (size_t)q * Kmax * (r + 1);
    const int TLD = q;
    const size_t t_elems = (size_t)q * Kmax * TLD;
    CK(cudaMallocAsync(&U, blk_elems * sizeof(S), stream));
    CK(cudaMallocAsync(&V, blk_elems * sizeof(S), stream));
    CK(cudaMallocAsync(&Zr, rec_elems * sizeof(S), stream));
    CK(cudaMallocAsync(&Qr, rec_elems * sizeof(S), stream));
    CK(cudaMallocAsync(&Tr, t_elems * sizeof(S), stream));
    CK(cudaMallocAsync(&prog, (size_t)q * sizeof(int), stream));
    long long* k1prof = nullptr;  // HT_K1PROF=1: chase phase cycle counts (stderr)
    const bool k1p = getenv("HT_K1PROF") != nullptr;
    if (k1p) {
        CK(cudaMallocAsync(&k1prof, 12 * sizeof(long long), stream));
        CK(cudaMemsetAsync(k1prof, 0, 12 * sizeof(long long), stream));
    }

    // kernel-class timing: 4 events per group from a pool, summed after one sync at the end
    const int ngroups = (n - 2 + q - 1) / q;
    std::vector<cudaEvent_t> ev;
    if (prof) {
        ev.resize((size_t)4 * ngroups);
        for (auto& e : ev) CK(cudaEventCreate(&e));
    }
    int g = 0;

    for (int j1 = 1; j1 <= n - 2; j1 += q) {
        const int qp = std::min(q, n - 1 - j1);
        const int K = 1 + (n - j1 - 2) / r;
        if (prof) CK(cudaEventRecord(ev[4 * g + 0], stream));
        CK(cudaMemsetAsync(prog, 0, (size_t)q * sizeof(int), stream));
        CK(cudaMemsetAsync(Qr, 0, (size_t)qp * K * (r + 1) * sizeof(S), stream));
        CK(cudaMemsetAsync(Zr, 0, (size_t)qp * K * (r + 1) * sizeof(S), stream));
        ChaseArgs<S> ca{n, r, qp, j1, K, H, ldh, T, ldt, Qr, Zr, Tr, TLD, prog, strip_cap, k1prof};
        void* kargs[] = {&ca};
        CK(cudaLaunchCooperativeKernel(chase_fn, dim3(qp), dim3(CHASE_NT), kargs, chase_bytes, stream));
        AccumArgs<S> aa{n, r, qp, j1, K, WP, LDB, Qr, Zr, U, V};
        accum_kernel<S, ACC_NT><<<dim3(K, 2), ACC_NT, acc_bytes, stream>>>(aa);
        g_last_launches += 2;
        if (prof) CK(cudaEventRecord(ev[4 * g + 1], stream));
        // ---- apply phase: right updates of H, T (staircase + V_k), then left (U_k^*) ----
        const int tiles = (n + CH_BM - 1) / CH_BM;
        ChainParams<S> pr{n, r, qp, j1, K, {{H, ldh, V, CM_AB_RIGHT, 0, tiles}, {T, ldt, V, CM_AB_RIGHT, 0, tiles}},
                          2, Zr};
        if (int rc = chain<S>(pr, WP, 2 * tiles, r, q, stream)) return rc;
        ChainParams<S> pl{n, r, qp, j1, K, {{H, ldh, U, CM_A_LEFT, 1, tiles}, {T, ldt, U, CM_B_LEFT, 1, tiles}},
                          2, Zr};
        if (int rc = chain<S>(pl, WP, 2 * tiles, r, q, stream)) return rc;
        g_last_launches += 2;
        if (prof) CK(cudaEventRecord(ev[4 * g + 2], stream));
        // ---- Q <- Q U_k, Z <- Z V_k (row chains; never read by the chase) ----
        if (Q || Z) {
            ChainParams<S> pq{n, r, qp, j1, K, {{Q ? Q : Z, Q ? ldq : ldz, Q ? U : V, CM_PLAIN, 0, tiles},
                                                {Z, ldz, V, CM_PLAIN, 0, tiles}},
                              (Q && Z) ? 2 : 1, Zr};
            if (int rc = chain<S>(pq, WP, pq.njobs * tiles, r, q, stream)) return rc;
            ++g_last_launches;
        }
        CK(cudaGetLastError());
        if (prof) CK(cudaEventRecord(ev[4 * g + 3], stream));
        ++g;
    }
    CK(cudaFreeAsync(U, stream));
    CK(cudaFreeAsync(V, stream));
    CK(cudaFreeAsync(Zr, stream));
    CK(cudaFreeAsync(Qr, stream));
    CK(cudaFreeAsync(Tr, stream));
    CK(cudaFreeAsync(prog, stream));
    if (k1p) {
        long long h[12];
        CK(cudaMemcpyAsync(h, k1prof, sizeof(h), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        const char* nm[12] = {"wait", "loads", "catchup", "QB+T", "larfgZ", "strip", "RQ", "larfgQ", "writes", "s9", "s10", "s11"};
        double tot = 0;
        for (long long x : h) tot += (double)x;
        fprintf(stderr, "K1 cycles (sum over CTAs):");
        for (int i = 0; i < 12; ++i) fprintf(stderr, " %s=%.1f%%", nm[i], 100.0 * h[i] / tot);
        fprintf(stderr, " total=%.3g\n", tot);
        CK(cudaFreeAsync(k1prof, stream));
    }
    CK(cudaEventRecord(e_end, stream));
    if (prof) {
        CK(cudaEventSynchronize(e_end));
        float tot = 0;
        CK(cudaEventElapsedTime(&tot, e_start, e_end));
        double acc[3] = {0, 0, 0};
        for (int i = 0; i < g; ++i)
            for (int c = 0; c < 3; ++c) {
                float x = 0;
                CK(cudaEventElapsedTime(&x, ev[4 * i + c], ev[4 * i + c + 1]));
                acc[c] += x;
            }
        for (int c = 0; c < 3; ++c) g_last_ms[c] = acc[c];
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
