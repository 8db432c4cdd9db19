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
thread_local int64_t g_lag_checked = 0, g_lag_violations = 0;  // HT_LAG_CHECK (ht_last_lag_check)

// Lag checker (debug, HT_LAG_CHECK=1, direct launches): from the global-timer stamps of one
// chase launch, every ordering the wavefront protocol promises (lag 3 between
// sweeps, the helpers' items behind their sweep and behind the previous sweep's helper) is checked:
// a step / item must not start before the step / item it waits for has ended.
void check_lag(const unsigned long long* tr, int n, int r, int qp, int j1, int K, const int* hoff) {
    // hoff: first helper index of sweep t (prefix sums of the helper layout, t <= qp)
    auto send = [&](int t, int k) { return tr[((int64_t)t * K + k) * 2 + 1]; };
    auto sbeg = [&](int t, int k) { return tr[((int64_t)t * K + k) * 2]; };
    auto hbeg = [&](int t, int h, int k) { return tr[((int64_t)qp * K + ((int64_t)hoff[t] + h) * K + k) * 2]; };
    auto hend = [&](int t, int h, int k) { return tr[((int64_t)qp * K + ((int64_t)hoff[t] + h) * K + k) * 2 + 1]; };
    auto H = [&](int t) { return hoff[t + 1] - hoff[t]; };
    for (int t = 0; t < qp; ++t) {
        const int j = j1 + t;
        const int kcount = std::min(K, 2 + (n - j - 1) / r);
        const int kprev = (t > 0) ? std::min(K, 2 + (n - j) / r) : 0;
        for (int k = 0; k < kcount; ++k) {
            if (t > 0) {
                const int need = std::min(k + 3, kprev), hneed = std::min(k + 2, kprev);
                ++g_lag_checked;
                if (sbeg(t, k) < send(t - 1, need - 1)) ++g_lag_violations;
                for (int h = 0; h < H(t - 1); ++h) {
                    ++g_lag_checked;
                    if (sbeg(t, k) < hend(t - 1, h, hneed - 1)) ++g_lag_violations;
                }
            }
            for (int h = 0; h < H(t); ++h) {
                ++g_lag_checked;
                if (hbeg(t, h, k) < send(t, k)) ++g_lag_violations;
                if (t > 0)
                    for (int hh = 0; hh < H(t - 1); ++hh) {  // every helper of the previous sweep
                        ++g_lag_checked;
                        if (hbeg(t, h, k) < hend(t - 1, hh, std::min(k + 2, kprev) - 1)) ++g_lag_violations;
                    }
            }
        }
    }
}

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
    // q = 2r up to 32: dense U/V execute (q+r-1)^2/(2qr) x the useful flops (minimal at q ~ r),
    // while the group-serial chase's critical path n^2/(2rq) + 3n favours larger q (measured at
    // config 2: q = 32 beats q = 16 by 1.4x); the window order w = q+r-1 must stay <= 160 (K2
    // holds a w x w block in shared memory)
    int64_t q = std::min<int64_t>(std::max<int64_t>(2 * r, 8), 32);
    q = std::min<int64_t>(q, std::max<int64_t>(1, 161 - r));
    return std::max<int64_t>(1, std::min<int64_t>(q, std::max<int64_t>(1, n - 2)));
}

template <typename S, int WP>
size_t chain_bytes(int r, int q, int P = 1, int QP = 0) { return chain_smem_bytes<S, WP>(r, q, P, QP); }

template <typename S, int WP>
int launch_chain(const ChainParams<S>& P, int grid, int r, int q, cudaStream_t st, size_t min_smem) {
    const size_t bytes = std::max(chain_bytes<S, WP>(r, q, P.P, P.wy ? P.QP : 0), min_smem);
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        CK(cudaFuncSetAttribute(chain_kernel<S, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_set = true;
    }
    chain_kernel<S, WP><<<grid, chain_nt(WP), bytes, st>>>(P);
    CK(cudaGetLastError());
    return HT_OK;
}

// min_smem > 0 pads the dynamic shared memory so that at most one CTA fits per SM (used by the
// side-stream Q/Z chains: a grid of nsm - q such CTAs leaves q whole SMs for the next chase).
template <typename S>
int chain(const ChainParams<S>& P, int WP, int grid, int r, int q, cudaStream_t st, size_t min_smem = 0) {
    switch (WP) {
        case 32: return launch_chain<S, 32>(P, grid, r, q, st, min_smem);
        case 64: return launch_chain<S, 64>(P, grid, r, q, st, min_smem);
        case 96: return launch_chain<S, 96>(P, grid, r, q, st, min_smem);
        case 128: return launch_chain<S, 128>(P, grid, r, q, st, min_smem);
        case 160: return launch_chain<S, 160>(P, grid, r, q, st, min_smem);
        default: return HT_EUNSUPPORTED;
    }
}

// Q/Z chains as two tile groups per CTA (chain_kernel2): one CTA per SM, 2 x the group bytes
template <typename S, int WP>
int launch_chain2(const ChainParams<S>& P, int grid, int r, int q, cudaStream_t st) {
    const size_t gb = (chain_bytes<S, WP>(r, q, P.P, P.wy ? P.QP : 0) + 127) / 128 * 128;
    static bool attr_set = false;
    if (!attr_set) {
        CK(cudaFuncSetAttribute(chain_kernel2<S, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_set = true;
    }
    chain_kernel2<S, WP><<<grid, 2 * chain_nt(WP), 2 * gb, st>>>(P, (unsigned)gb);
    CK(cudaGetLastError());
    return HT_OK;
}

template <typename S>
int chain2(const ChainParams<S>& P, int WP, int grid, int r, int q, cudaStream_t st) {
    switch (WP) {
        case 32: return launch_chain2<S, 32>(P, grid, r, q, st);
        case 64: return launch_chain2<S, 64>(P, grid, r, q, st);
        case 96: return launch_chain2<S, 96>(P, grid, r, q, st);
        case 128: return launch_chain2<S, 128>(P, grid, r, q, st);
        case 160: return launch_chain2<S, 160>(P, grid, r, q, st);
        default: return HT_EUNSUPPORTED;
    }
}

template <typename S>
int chain_prepare(int WP) {  // smem attribute outside any stream capture
    ChainParams<S> dummy{};
    (void)dummy;
#define HT_PREP(W)                                                                                           \
    case W:                                                                                                  \
        CK(cudaFuncSetAttribute(chain_kernel<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));  \
        CK(cudaFuncSetAttribute(chain_kernel2<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)); \
        break;
    switch (WP) {
        HT_PREP(32)
        HT_PREP(64)
        HT_PREP(96)
        HT_PREP(128)
        HT_PREP(160)
        default: return HT_EUNSUPPORTED;
    }
#undef HT_PREP
    return HT_OK;
}

template <typename S>
size_t chain_bytes_rt(int WP, int r, int q, int P = 1, int QP = 0) {
    switch (WP) {
        case 32: return chain_bytes<S, 32>(r, q, P, QP);
        case 64: return chain_bytes<S, 64>(r, q, P, QP);
        case 96: return chain_bytes<S, 96>(r, q, P, QP);
        case 128: return chain_bytes<S, 128>(r, q, P, QP);
        case 160: return chain_bytes<S, 160>(r, q, P, QP);
        default: return (size_t)1 << 40;
    }
}

// K1 instantiation for the reflector length (the RQ keeps [C; P] rows in registers)
template <typename S>
const void* chase_kernel_for(int r, bool rqu) {
    if (r <= 8) return (const void*)chase_kernel<S, CHASE_NT, 8>;
    if (r <= 16) return (const void*)chase_kernel<S, CHASE_NT, 16>;
    if (r <= 32) return (const void*)chase_kernel<S, CHASE_NT, 32>;
    if constexpr (sizeof(S) == 8) {  // complex: r <= 32 (registers of the complex RQ)
        if (r <= 64) return rqu ? (const void*)chase_kernel<S, CHASE_NT, 64, true> : (const void*)chase_kernel<S, CHASE_NT, 64>;
        if (r <= 128)
            return rqu ? (const void*)chase_kernel<S, CHASE_NT, 128, true> : (const void*)chase_kernel<S, CHASE_NT, 128>;
    }
    return nullptr;
}

constexpr int ACC_NT = 256;

// Row slab of rank i out of G for the Q/Z updates: whole chain tiles (CH_BM rows), balanced.
inline void slab_tiles(int n, int G, int i, int* t0, int* nt) {
    const int T = (n + CH_BM - 1) / CH_BM;
    const int a = (int)((int64_t)T * i / G), b = (int)((int64_t)T * (i + 1) / G);
    *t0 = a;
    *nt = b - a;
}

// Far H/T row tiles: tile i (rows CH_BM i .. CH_BM i + CH_BM - 1, 0-based) lies
// above group g's band once CH_BM (i + 1) <= j1(g) = 1 + g q: no chase of group g or later reads or
// writes its rows again, and only the groups' right updates (A(1:i5, C_k) V_k, PAPER.md:1895-1900;
// always the block part, never the staircase) still change it, in columns > j1(g).  From that group
// on, far tiles are updated by their owner (tile i -> rank i mod G); the root hands the tile's rows
// (columns >= j1(g), 0-based) to the owner at the start of that group and gathers them back at the
// end.  Near tiles, the left updates and the chase stay on the root.
inline int nfar_tiles(int j1, int tiles) { return std::min(tiles, std::max(0, j1) / CH_BM); }
inline int far_group(int i, int q) { return (CH_BM * (i + 1) - 1 + q - 1) / q; }  // first g with nfar(1+gq) > i
inline int far_owner(int i, int G) { return i % G; }

template <typename S>
ncclDataType_t nccl_type() { return ncclFloat64; }
template <typename S>
size_t nccl_count(size_t elems) { return elems * (sizeof(S) / sizeof(double)); }

#define NK(x)                                                                     \
    do {                                                                          \
        ncclResult_t r_ = (x);                                                    \
        if (r_ != ncclSuccess) {                                                  \
            if (getenv("HT_DEBUG")) fprintf(stderr, "ht_stage2: NCCL %s at %s:%d\n", \
                                            ncclGetErrorString(r_), __FILE__, __LINE__); \
            return HT_ENCCL;                                                      \
        }                                                                         \
    } while (0)

// Helper layout of a group of qp sweeps (ChaseArgs::lay): Htot far-strip helper CTAs distributed
// over the sweeps in proportion to (qp - 1 - t) + F -- sweep t's far strip (band rows above b0(k))
// is (qp - 1 - t) r rows in steady state (i4 = j1 + 1 + (k + t - qp + 1) r), and F stands for the
// RQ-update work every sweep's helpers share; at least 1 and at most 8 per sweep, allocated greedily
// (max-min).  Uniform (Htot / qp each) when bal == false.
std::vector<int> helper_layout(int qp, int Htot, bool bal, double F) {
    std::vector<int> Hs(qp, Htot / std::max(1, qp));
    if (bal && qp > 1 && Htot >= qp) {  // greedy: the next helper to the sweep with the largest load per helper
        std::fill(Hs.begin(), Hs.end(), 1);
        for (int e = qp; e < Htot; ++e) {
            int best = -1;
            double bl = -1.0;
            for (int t = 0; t < qp; ++t) {
                const double l = ((qp - 1 - t) + F) / Hs[t];
                if (Hs[t] < 8 && l > bl) bl = l, best = t;
            }
            if (best < 0) break;
            ++Hs[best];
        }
    }
    std::vector<int> lay(qp + 1);
    lay[0] = 0;
    for (int t = 0; t < qp; ++t) lay[t + 1] = lay[t] + Hs[t];
    for (int t = 0; t < qp; ++t)
        for (int role = 0; role <= Hs[t]; ++role) lay.push_back((t << 8) | role);
    return lay;
}

template <typename S>
struct Plan {
    int n, r, q, WP, LDB, Kmax, strip_cap;
    size_t chase_bytes, acc_bytes;
    const void* chase_fn;
    S* H;
    int64_t ldh;
    S* T;
    int64_t ldt;
    S* Q;
    int64_t ldq;
    S* Z;
    int64_t ldz;
    int qz_ctas;
    // multi-GPU: the root chases and updates H, T; every rank updates its row slab
    // of Q and Z.  comm == nullptr: one GPU (emul > 1 splits the Q/Z chains into emulated slabs).
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, root = 0, emul = 1;
    // far H/T tiles (nfar_tiles): G owners (NCCL ranks, or emulated ranks on one GPU with their own
    // full-size H/T copies HR[p], TR[p]; the root's are the caller's buffers)
    int G = 1;
    bool emul_ht = false;
    S* HR[8] = {};
    S* TR[8] = {};
    int64_t ldr = 0;
    bool shard_ht() const { return G > 1; }
    int helpers = 1;  // far-strip helper CTAs per sweep in the chase
    int P = 1;        // window merge factor of the apply chains (K2m)
    int nsm = 148;    // SMs (longest-chain-first tile order of the H/T chains)
    bool qz_late = true;   // Q/Z chains of a group start after its H/T chains (HT_QZ_LATE=0: after K2)
    int qz_stream = 0;     // Q/Z tiles loaded / stored with an L2 evict-first policy (HT_QZ_STREAM)
    int tmap = 0;          // left-update tiles: conflict-free 4 x 8 lane map of the loads / stores (HT_CHAIN_TMAP)
    bool qz_groups = false;  // Q/Z chains as two tile groups per CTA (chain_kernel2; HT_QZ_GROUPS=0: off)
    bool far_side = false;   // one GPU: far H/T tiles' right updates on the side stream (HT_FAR_SIDE)
    int wy = 0, QP = 0;      // WY window blocks (chain.cuh ChainParams::wy; accum_wy_kernel)
    int hlag = 1;          // helper row split (ChaseArgs::hlag): 0 for r >= 32 (HT_HELPER_LAG overrides)
    int rqu = 0;           // K1 opposite reflector by RQ update (rqu.cuh; HT_RQU=0 disables)
    int hbal = 0;          // helpers distributed over the sweeps by far-strip load (helper_layout)
    double hF = 10.0;      // ... its per-sweep constant, in far-strip rows / r (HT_HELPER_F)
    int rqu_self_num = 0, rqu_self_den = 1;  // rqu 2: share of the hand-overs the sweep runs (HT_RQU_SELF)
    size_t mrg_bytes = 0;
    const unsigned long long* gate = nullptr;  // device verdict words of the input check (nullptr: none)
    bool is_root() const { return comm == nullptr || rank == root; }
    bool qz() const { return Q || Z; }
    bool same(const Plan& o) const {
        return n == o.n && r == o.r && q == o.q && strip_cap == o.strip_cap && helpers == o.helpers && P == o.P && qz_late == o.qz_late && qz_stream == o.qz_stream && tmap == o.tmap && qz_groups == o.qz_groups && far_side == o.far_side && wy == o.wy && hlag == o.hlag && rqu == o.rqu && hbal == o.hbal && hF == o.hF && rqu_self_num == o.rqu_self_num && rqu_self_den == o.rqu_self_den && G == o.G && emul_ht == o.emul_ht && gate == o.gate && H == o.H && ldh == o.ldh &&
               T == o.T && ldt == o.ldt && Q == o.Q && ldq == o.ldq && Z == o.Z && ldz == o.ldz;
    }
};

// Workspace of one reduction: NUV U/V buffers (the Q/Z chains of group g run on the side
// stream while later groups are chased; the side stream may lag NUV-1 groups), reflector
// records, WY factors, progress counters.
constexpr int NUV = 4;
// dense catch-up operators M_t(k) (chase_dense_catchup): one (q+r-1) x ((q+r-1)|1) block per window
inline int mcatch_ld(int q, int r) { return (q + r - 1) | 1; }
inline int64_t mcatch_st(int q, int r) { return (int64_t)(q + r - 1) * mcatch_ld(q, r); }

template <typename S>
struct Workspace {
    S *U[NUV] = {}, *V[NUV] = {}, *MU[NUV] = {}, *MV[NUV] = {}, *Zr = nullptr, *Qr = nullptr, *Tr = nullptr, *Mg = nullptr;
    int* lay = nullptr;    // helper layouts (helper_layout) of the full groups and of the last group
    std::vector<int> lay_host;
    int lay_last = 0;      // offset of the last group's layout
    double* Fg = nullptr;  // RQ-update hand-over (Kmax x 2 x 64 x 64), kept across groups
    double* Fb = nullptr;  // rqu 2: caught-up column b per window (Kmax x MAXM)
    int* Fdone = nullptr;  // rqu 2: hand-over generation per window (Kmax)
    int* Freq = nullptr;   // rqu 2, MAXM 128: early direction requests / answers per window
    int* Fdirok = nullptr;
    double* Fdir = nullptr;
    unsigned long long* lag = nullptr;  // HT_LAG_CHECK stamps (one group)
    S* xfer = nullptr;                  // far H/T tile transfers (2 CH_BM n scalars)
    S* emu[16] = {};                    // emulated ranks' H/T copies
    int* prog = nullptr;
    long long* k1prof = nullptr;
    long long k1prof_host[40] = {0};  // [0,16) K1, [16,24) K1 sub-phases, [24,32) right chains, [32,40) left chains
    cudaStream_t side = nullptr;
    cudaEvent_t ev_uv[NUV] = {}, ev_qz[NUV] = {}, ev_k2[NUV] = {};
    bool async = true;

    int alloc(const Plan<S>& p, cudaStream_t stream, bool async_, bool k1p) {
        async = async_;
        const size_t blk = (size_t)p.Kmax * p.WP * p.LDB * sizeof(S);
        const size_t rec = (size_t)p.q * p.Kmax * (p.r + 1) * sizeof(S);
        const size_t tf = (size_t)p.q * p.Kmax * p.q * sizeof(S);
        auto mal = [&](void** ptr, size_t bytes) -> cudaError_t {
            return async ? cudaMallocAsync(ptr, bytes, stream) : cudaMalloc(ptr, bytes);
        };
        const size_t mblk = (size_t)((p.Kmax + p.P - 1) / p.P) * p.WP * p.LDB * sizeof(S);
        for (int b = 0; b < (p.qz() ? NUV : 1); ++b) {
            CK(mal((void**)&U[b], blk));
            CK(mal((void**)&V[b], blk));
            if (p.P > 1) {
                CK(mal((void**)&MU[b], mblk));
                CK(mal((void**)&MV[b], mblk));
            }
        }
        CK(mal((void**)&Zr, rec));
        CK(mal((void**)&Qr, rec));
        CK(mal((void**)&Tr, tf));
        if (chase_dense_catchup<S>(p.r)) CK(mal((void**)&Mg, (size_t)p.Kmax * mcatch_st(p.q, p.r) * sizeof(S)));
        if (p.helpers > 0) {  // helper layouts: full groups (qp = q) and the last group
            const int ngroups = (p.n - 2 + p.q - 1) / p.q;
            const int qlast = std::min(p.q, p.n - 1 - (1 + (ngroups - 1) * p.q));
            lay_host = helper_layout(p.q, p.helpers * p.q, p.hbal != 0, p.hF);
            lay_last = (int)lay_host.size();
            const std::vector<int> l2 = helper_layout(qlast, p.helpers * qlast, p.hbal != 0, p.hF);
            lay_host.insert(lay_host.end(), l2.begin(), l2.end());
            CK(mal((void**)&lay, lay_host.size() * sizeof(int)));
            CK(cudaMemcpyAsync(lay, lay_host.data(), lay_host.size() * sizeof(int), cudaMemcpyHostToDevice, stream));
        }
        const size_t rm = p.r <= 64 ? 64 : 128;  // MAXM of the RQ update
        if (p.rqu) CK(mal((void**)&Fg, (size_t)p.Kmax * 2 * rm * rm * sizeof(double)));
        if (p.rqu == 2) {
            CK(mal((void**)&Fb, (size_t)p.Kmax * rm * sizeof(double)));
            CK(mal((void**)&Fdone, (size_t)3 * p.Kmax * sizeof(int)));  // Fdone, Freq, Fdirok
            Freq = Fdone + p.Kmax;
            Fdirok = Fdone + 2 * p.Kmax;
            CK(mal((void**)&Fdir, (size_t)p.Kmax * rm * sizeof(double)));
        }
        CK(mal((void**)&prog, (size_t)(5 * p.q + 2) * sizeof(int)));
        if (p.shard_ht() && !p.emul_ht) CK(mal((void**)&xfer, (size_t)2 * CH_BM * p.n * sizeof(S)));
        if (getenv("HT_LAG_CHECK") && async)
            CK(mal((void**)&lag, (size_t)2 * p.q * p.Kmax * 4 * sizeof(unsigned long long)));
        if (k1p) {
            CK(mal((void**)&k1prof, 40 * sizeof(long long)));
            CK(cudaMemsetAsync(k1prof, 0, 40 * sizeof(long long), stream));
        }
        if (p.qz()) {
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));  // lowest priority
            for (int b = 0; b < NUV; ++b) {
                CK(cudaEventCreateWithFlags(&ev_uv[b], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_qz[b], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_k2[b], cudaEventDisableTiming));
            }
        }
        return HT_OK;
    }
    int release(cudaStream_t stream, bool async_) {
        if (k1prof) {
            CK(cudaMemcpyAsync(k1prof_host, k1prof, sizeof(k1prof_host), cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
        }
        auto fr = [&](void* ptr) -> cudaError_t {
            if (!ptr) return cudaSuccess;
            return async_ ? cudaFreeAsync(ptr, stream) : cudaFree(ptr);
        };
        for (int b = 0; b < NUV; ++b) {
            CK(fr(U[b]));
            CK(fr(V[b]));
            CK(fr(MU[b]));
            CK(fr(MV[b]));
        }
        CK(fr(Zr));
        CK(fr(Qr));
        CK(fr(Tr));
        if (Mg) CK(fr(Mg));
        Mg = nullptr;
        if (Fg) CK(fr(Fg));
        Fg = nullptr;
        if (lay) CK(fr(lay));
        lay = nullptr;
        if (Fb) CK(fr(Fb));
        Fb = nullptr;
        if (Fdone) CK(fr(Fdone));
        Fdone = Freq = Fdirok = nullptr;
        if (Fdir) CK(fr(Fdir));
        Fdir = nullptr;
        CK(fr(prog));
        CK(fr(k1prof));
        CK(fr(lag));
        CK(fr(xfer));
        for (auto& e : emu) {
            CK(fr(e));
            e = nullptr;
        }
        for (int b = 0; b < NUV; ++b) {
            if (ev_uv[b]) cudaEventDestroy(ev_uv[b]);
            if (ev_qz[b]) cudaEventDestroy(ev_qz[b]);
            if (ev_k2[b]) cudaEventDestroy(ev_k2[b]);
        }
        if (side) cudaStreamDestroy(side);  // deferred until its work completes
        return HT_OK;
    }
};

void print_k1prof(const long long* h) {
    // slots 0..10 and 12..15 are cycles of thread 0 of the profiled sweeps; slot 11 counts steps
    const char* nm[16] = {"wait", "loads", "catchup", "QB+T", "larfgZ", "strip", "RQ", "larfgQ", "writes", "waitH",
                          "s10", "", "s12", "s13", "hwait", "hwork"};
    double tot = 0;
    for (int i = 0; i < 14; ++i)  // (14, 15: the helper's own wait / work, not part of the sweep's)
        if (i != 11) tot += (double)h[i];
    const double steps = h[11] > 0 ? (double)h[11] : 1.0;
    fprintf(stderr, "K1 cycles (sum over CTAs):");
    for (int i = 0; i < 16; ++i)
        if (i != 11 && h[i]) fprintf(stderr, " %s=%.1f%%", nm[i], 100.0 * h[i] / (tot > 0 ? tot : 1));
    fprintf(stderr, " total=%.3g steps=%.0f\nK1 cycles per step:", tot, steps);
    for (int i = 0; i < 16; ++i)
        if (i != 11 && h[i]) fprintf(stderr, " %s=%.0f", nm[i], h[i] / steps);
    fprintf(stderr, " all=%.0f\n", tot / steps);
    // sub-phases (parts of the slots above): the RQ update (rqu.cuh)
    const char* sn[8] = {"rqu_loadwait", "rqu_A", "rqu_BC|solve", "rqu_D|Qx", "rqu_handoff", "s21", "S4_QB_tid0", "S4_T_tidNT/2"};
    bool any = false;
    for (int i = 16; i < 24; ++i) any |= h[i] != 0;
    if (any) {
        fprintf(stderr, "K1 sub-phase cycles per step:");
        for (int i = 16; i < 24; ++i)
            if (h[i]) fprintf(stderr, " %s=%.0f", sn[i - 16], h[i] / steps);
        fprintf(stderr, "\n");
    }
    for (int c = 0; c < 2; ++c) {  // apply chains: the longest tile (tile 0 of H)
        const long long* g = h + 24 + 8 * c;
        const double st = g[5] > 0 ? (double)g[5] : 1.0;
        fprintf(stderr, "%s chain, profiled tile of H (HT_CHAIN_PROF_TILE), cycles per step: wait+prefetch=%.0f mma=%.0f epilogue=%.0f "
                        "staircase=%.0f store=%.0f (steps %lld, merged %lld, with staircase %lld)\n",
                c == 0 ? "right" : "left", g[0] / st, g[1] / st, g[2] / st, g[3] / st, g[4] / st, g[5], g[6], g[7]);
    }
}

// Enqueue every group of the reduction: chase (K1) -> accumulate U/V (K2) -> H/T right and left
// chains (K3/K4) on `stream`; Q/Z chains on the side stream.  With prof, per-class device
// times are accumulated into g_last_ms (needs a host sync at the end).
// Final gather of the Q/Z row slabs to the root: each non-root rank packs its
// rows of Q and Z into one contiguous buffer and sends it; the root unpacks rank by rank.
template <typename S>
int gather_slabs(const Plan<S>& p, cudaStream_t stream) {
    const int n = p.n;
    int maxnt = 0;
    for (int i = 0; i < p.nranks; ++i) {
        int t0, nt;
        slab_tiles(n, p.nranks, i, &t0, &nt);
        maxnt = std::max(maxnt, nt);
    }
    const size_t slab = (size_t)maxnt * CH_BM * n;
    S* buf = nullptr;
    CK(cudaMallocAsync(&buf, 2 * slab * sizeof(S), stream));
    auto rows = [&](int i, int* a, int* len) {
        int t0, nt;
        slab_tiles(n, p.nranks, i, &t0, &nt);
        *a = t0 * CH_BM;
        *len = std::max(0, std::min(n, (t0 + nt) * CH_BM) - *a);
    };
    for (int i = 0; i < p.nranks; ++i) {
        if (i == p.root) continue;
        int a, len;
        rows(i, &a, &len);
        if (len == 0) continue;
        const size_t cnt = nccl_count<S>((size_t)len * n);
        if (p.rank == i) {
            if (p.Q) pack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.Q, p.ldq, a, len, n, buf);
            if (p.Z) pack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.Z, p.ldz, a, len, n, buf + slab);
            CK(cudaGetLastError());
            NK(ncclGroupStart());
            if (p.Q) NK(ncclSend(buf, cnt, nccl_type<S>(), p.root, p.comm, stream));
            if (p.Z) NK(ncclSend(buf + slab, cnt, nccl_type<S>(), p.root, p.comm, stream));
            NK(ncclGroupEnd());
        } else if (p.rank == p.root) {
            NK(ncclGroupStart());
            if (p.Q) NK(ncclRecv(buf, cnt, nccl_type<S>(), i, p.comm, stream));
            if (p.Z) NK(ncclRecv(buf + slab, cnt, nccl_type<S>(), i, p.comm, stream));
            NK(ncclGroupEnd());
            if (p.Q) unpack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.Q, p.ldq, a, len, n, buf);
            if (p.Z) unpack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.Z, p.ldz, a, len, n, buf + slab);
            CK(cudaGetLastError());
        }
    }
    CK(cudaFreeAsync(buf, stream));
    return HT_OK;
}

// Rows [r0, r0 + len) x columns [c0, n) (0-based) of H and T from rank `src` to rank `dst`:
// emulated ranks -- a 2-D copy between their buffers; NCCL -- pack, send / recv, unpack (stream-
// ordered on `stream`; the calling rank takes its part; point-to-point calls outside NCCL groups so
// that the unpack follows the receive on the stream).  buf: workspace of 2 len (n - c0) scalars.
template <typename S>
int move_rows_ht(const Plan<S>& p, int src, int dst, int r0, int len, int c0, S* buf, cudaStream_t stream) {
    const int n = p.n, nc = n - c0;
    if (len <= 0 || nc <= 0 || src == dst) return HT_OK;
    if (p.emul_ht) {
        for (int m = 0; m < 2; ++m) {
            S* a = m ? p.TR[src] : p.HR[src];
            S* b = m ? p.TR[dst] : p.HR[dst];
            const int64_t lda = src == p.root ? (m ? p.ldt : p.ldh) : p.ldr;
            const int64_t ldb = dst == p.root ? (m ? p.ldt : p.ldh) : p.ldr;
            CK(cudaMemcpy2DAsync(b + r0 + (int64_t)c0 * ldb, ldb * sizeof(S), a + r0 + (int64_t)c0 * lda, lda * sizeof(S),
                                 len * sizeof(S), nc, cudaMemcpyDeviceToDevice, stream));
        }
        return HT_OK;
    }
    const size_t cnt = (size_t)len * nc;
    if (p.rank == src) {
        pack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.H + (int64_t)c0 * p.ldh, p.ldh, r0, len, nc, buf);
        pack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.T + (int64_t)c0 * p.ldt, p.ldt, r0, len, nc, buf + cnt);
        CK(cudaGetLastError());
        NK(ncclSend(buf, nccl_count<S>(2 * cnt), nccl_type<S>(), dst, p.comm, stream));
    } else if (p.rank == dst) {
        NK(ncclRecv(buf, nccl_count<S>(2 * cnt), nccl_type<S>(), src, p.comm, stream));
        unpack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.H + (int64_t)c0 * p.ldh, p.ldh, r0, len, nc, buf);
        unpack_rows_kernel<S><<<4 * 148, 256, 0, stream>>>(p.T + (int64_t)c0 * p.ldt, p.ldt, r0, len, nc, buf + cnt);
        CK(cudaGetLastError());
    }
    return HT_OK;
}

// Far H/T tiles back to the root at the end: every far tile owned by a non-root rank, its rows and
// the columns >= j1 of the group at which it became far.
template <typename S>
int gather_far_ht(const Plan<S>& p, S* buf, cudaStream_t stream) {
    const int n = p.n, q = p.q, tiles = (n + CH_BM - 1) / CH_BM;
    const int ngroups = (n - 2 + q - 1) / q;
    for (int i = 0; i < tiles; ++i) {
        const int g = far_group(i, q);
        if (g >= ngroups) break;  // (tiles become far in order)
        const int o = far_owner(i, p.G);
        if (o == p.root) continue;
        const int r0 = i * CH_BM, len = std::min(CH_BM, n - r0), c0 = 1 + g * q;  // (0-based column j1(g))
        if (int rc = move_rows_ht<S>(p, o, p.root, r0, len, c0, buf, stream)) return rc;
    }
    return HT_OK;
}

template <typename S>
int enqueue_groups(const Plan<S>& p, Workspace<S>& ws, cudaStream_t stream, bool prof) {
    const int n = p.n, r = p.r, q = p.q, WP = p.WP, LDB = p.LDB, TLD = q;
    const bool qz = p.qz();
    const int ngroups = (n - 2 + q - 1) / q;
    static thread_local std::vector<cudaEvent_t> ev;  // grow-only pool (event creation is slow)
    if (prof)
        while (ev.size() < (size_t)5 * ngroups) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ev.push_back(e);
        }
    if (ws.Fdone) CK(cudaMemsetAsync(ws.Fdone, 0, (size_t)3 * p.Kmax * sizeof(int), stream));
    if (qz) {
        CK(cudaEventRecord(ws.ev_qz[0], stream));  // workspace allocations visible to the side stream
        CK(cudaStreamWaitEvent(ws.side, ws.ev_qz[0], 0));
    }
    int g = 0;
    for (int j1 = 1; j1 <= n - 2; j1 += q, ++g) {
        const int qp = std::min(q, n - 1 - j1);
        const int K = 1 + (n - j1 - 2) / r;
        const int bsel = qz ? (g % NUV) : 0;
        const bool root = p.is_root();
        const int tiles = (n + CH_BM - 1) / CH_BM;
        // far H/T tiles of this group: owned by the ranks (multi-GPU), or updated on the side stream
        const int nf = (p.shard_ht() || p.far_side) ? nfar_tiles(j1, tiles) : 0;
        if (p.shard_ht())  // tiles turned far by this group: root -> owner (after the root's updates of g-1)
            for (int i = nfar_tiles(j1 - q, tiles); i < nf; ++i) {
                const int r0 = i * CH_BM;
                if (int rc = move_rows_ht<S>(p, p.root, far_owner(i, p.G), r0, std::min(CH_BM, n - r0), j1, ws.xfer, stream))
                    return rc;
            }
        if (prof) CK(cudaEventRecord(ev[5 * g + 0], stream));
        if (root) {
            CK(cudaMemsetAsync(ws.prog, 0, (size_t)((1 + p.helpers) * q + 1) * sizeof(int), stream));
            CK(cudaMemsetAsync(ws.Qr, 0, (size_t)qp * K * (r + 1) * sizeof(S), stream));
            CK(cudaMemsetAsync(ws.Zr, 0, (size_t)qp * K * (r + 1) * sizeof(S), stream));
            ChaseArgs<S> ca{n, r, qp, j1, K, p.H, p.ldh, p.T, p.ldt, ws.Qr, ws.Zr, ws.Tr, TLD, ws.Mg,
                            mcatch_ld(q, r), mcatch_st(q, r), ws.prog, p.strip_cap,
                            p.helpers, ws.k1prof, getenv("HT_K1PROF_T") ? atoi(getenv("HT_K1PROF_T")) : -1,
                            p.hlag, p.gate, ws.lag};
            ca.Fg = ws.Fg;
            ca.fst = (int64_t)2 * (r <= 64 ? 64 * 64 : 128 * 128);
            ca.Freq = ws.Freq;
            ca.Fdirok = ws.Fdirok;
            ca.Fdir = ws.Fdir;
            ca.rqu = p.rqu;
            ca.lay = ws.lay ? ws.lay + (qp == q ? 0 : ws.lay_last) : nullptr;
            ca.Fb = ws.Fb;
            ca.Fdone = ws.Fdone;
            ca.rqu_self_num = p.rqu_self_num;
            ca.rqu_self_den = p.rqu_self_den;
            const size_t lag_elems = (size_t)2 * qp * K * (1 + p.helpers);
            if (ws.lag) CK(cudaMemsetAsync(ws.lag, 0, lag_elems * sizeof(unsigned long long), stream));
            void* kargs[] = {&ca};
            CK(cudaLaunchKernel(p.chase_fn, dim3(qp * (1 + p.helpers)), dim3(CHASE_NT), kargs, p.chase_bytes, stream));
            if (ws.lag) {  // (debug: synchronous per group)
                std::vector<unsigned long long> h(lag_elems);
                CK(cudaMemcpyAsync(h.data(), ws.lag, lag_elems * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
                CK(cudaStreamSynchronize(stream));
                check_lag(h.data(), n, r, qp, j1, K, ws.lay_host.data() + (qp == q ? 0 : ws.lay_last));
                // HT_TRACE_DUMP=file (with HT_LAG_CHECK=1): the raw stamps of the group starting at
                // HT_TRACE_J1 (default 1) and the helper offsets, for tools/trace_path.py
                const char* td = getenv("HT_TRACE_DUMP");
                const int tj1 = getenv("HT_TRACE_J1") ? atoi(getenv("HT_TRACE_J1")) : 1;
                if (td && j1 == tj1)
                    if (FILE* f = fopen(td, "wb")) {
                        const int hdr[6] = {n, r, qp, j1, K, p.helpers};
                        fwrite(hdr, sizeof(int), 6, f);
                        const int* ho = ws.lay_host.data() + (qp == q ? 0 : ws.lay_last);
                        std::vector<int> hoff(qp + 1, 0);
                        for (int t = 0; t <= qp; ++t) hoff[t] = ws.lay ? ho[t] : t * p.helpers;
                        fwrite(hoff.data(), sizeof(int), qp + 1, f);
                        fwrite(h.data(), sizeof(unsigned long long), lag_elems, f);
                        fclose(f);
                    }
            }
        }
        if (p.comm && (qz || p.shard_ht())) {  // the group's reflectors (2 qp K (r+1) scalars) to every rank
            const size_t cnt = nccl_count<S>((size_t)qp * K * (r + 1));
            NK(ncclGroupStart());
            NK(ncclBroadcast(ws.Qr, ws.Qr, cnt, nccl_type<S>(), p.root, p.comm, stream));
            NK(ncclBroadcast(ws.Zr, ws.Zr, cnt, nccl_type<S>(), p.root, p.comm, stream));
            NK(ncclGroupEnd());
        }
        if (qz && g >= NUV) CK(cudaStreamWaitEvent(stream, ws.ev_qz[bsel], 0));  // Q/Z of g-NUV done with U/V[bsel]
        AccumArgs<S> aa{n, r, qp, j1, K, WP, LDB, p.acc_bytes >= accum_smem_bytes<S>(r, q, true) ? 1 : 0, ws.Qr, ws.Zr,
                        ws.U[bsel], ws.V[bsel], p.gate};
        if (p.wy && (root || qz || p.shard_ht())) {
            AccumWYArgs<S> aw{n, r, qp, j1, K, WP, p.QP, ws.Qr, ws.Zr, ws.U[bsel], ws.V[bsel], p.gate};
            accum_wy_kernel<S, ACC_NT><<<dim3(K, 2), ACC_NT, accum_wy_smem_bytes<S>(r, q, p.QP), stream>>>(aw);
            CK(cudaGetLastError());
            g_last_launches += 1;
        } else if (root || qz || p.shard_ht()) {
            accum_kernel<S, ACC_NT><<<dim3(K, 2), ACC_NT, p.acc_bytes, stream>>>(aa);
            CK(cudaGetLastError());
            g_last_launches += 2;
            if (p.P > 1) {
                MergeArgs<S> ma{n, r, qp, j1, K, p.P, WP, LDB, ws.U[bsel], ws.V[bsel], ws.MU[bsel], ws.MV[bsel], p.gate};
                merge_kernel<S, ACC_NT><<<dim3((K + p.P - 1) / p.P, 2), ACC_NT, p.mrg_bytes, stream>>>(ma);
                CK(cudaGetLastError());
                ++g_last_launches;
            }
        }
        // Q/Z chains of group g start after K2 (their blocks), or -- p.qz_late -- after the group's
        // H/T chains, so that those (on the critical path) do not share SMs with them
        if (qz && !p.qz_late) CK(cudaEventRecord(ws.ev_uv[bsel], stream));
        if (p.far_side && nf > 0) {
            // one GPU: the far tiles' right updates (rows above every later chase band, SURVEY
            // §8(a) a7) need only U/V of this group and the tiles' state after group g-1 (main stream,
            // before this group's chase), so they run on the side stream beside this group's near
            // H/T chains and the next chase, as a persistent grid on the SMs the chase leaves
            CK(cudaEventRecord(ws.ev_k2[bsel], stream));
            CK(cudaStreamWaitEvent(ws.side, ws.ev_k2[bsel], 0));
            ChainParams<S> pf{n, r, qp, j1, K, {{p.H, p.ldh, ws.V[bsel], ws.MV[bsel], CM_AB_RIGHT, 0, nf, 0},
                                                {p.T, p.ldt, ws.V[bsel], ws.MV[bsel], CM_AB_RIGHT, 0, nf, 0}}, 2, ws.Zr, p.P, 0};
            pf.gate = p.gate;
            pf.wy = p.wy;
            pf.QP = p.QP;
            if (p.qz_groups) {
                if (int rc = chain2<S>(pf, WP, std::min(nf, p.qz_ctas), r, q, ws.side)) return rc;
            } else if (int rc = chain<S>(pf, WP, std::min(2 * nf, p.qz_ctas), r, q, ws.side, 116 * 1024)) {
                return rc;
            }
            ++g_last_launches;
        }
        if (prof) CK(cudaEventRecord(ev[5 * g + 1], stream));
        // ---- apply phase: right updates of H, T (staircase + V_k), then left (U_k^*) ----
        // far tiles (rows above the band): every owner updates its own (tile i -> rank i mod G)
        if (nf > 0 && p.shard_ht())
            for (int rk = 0; rk < p.G; ++rk) {
                if (!p.emul_ht && rk != p.rank) continue;
                const int cnt = rk < nf ? (nf - rk + p.G - 1) / p.G : 0;
                if (cnt == 0) continue;
                S* Hk = p.emul_ht ? p.HR[rk] : p.H;
                S* Tk = p.emul_ht ? p.TR[rk] : p.T;
                const int64_t lhk = (p.emul_ht && rk != p.root) ? p.ldr : p.ldh;
                const int64_t ltk = (p.emul_ht && rk != p.root) ? p.ldr : p.ldt;
                ChainParams<S> pf{n, r, qp, j1, K, {{Hk, lhk, ws.V[bsel], ws.MV[bsel], CM_AB_RIGHT, 0, cnt, rk, p.G},
                                                    {Tk, ltk, ws.V[bsel], ws.MV[bsel], CM_AB_RIGHT, 0, cnt, rk, p.G}}, 2, ws.Zr, p.P,
                                  0};
                pf.gate = p.gate;
            pf.wy = p.wy;
            pf.QP = p.QP;
                if (int rc = chain<S>(pf, WP, 2 * cnt, r, q, stream)) return rc;
                ++g_last_launches;
            }
        if (root) {
            ChainParams<S> pr{n, r, qp, j1, K, {{p.H, p.ldh, ws.V[bsel], ws.MV[bsel], CM_AB_RIGHT, 0, tiles - nf, nf},
                                                {p.T, p.ldt, ws.V[bsel], ws.MV[bsel], CM_AB_RIGHT, 0, tiles - nf, nf}}, 2, ws.Zr, p.P,
                              chain_spread(p.nsm), ws.k1prof ? ws.k1prof + 24 : nullptr,
                              getenv("HT_CHAIN_PROF_TILE") ? atoi(getenv("HT_CHAIN_PROF_TILE")) : 0,
                              !(getenv("HT_STAIR_FIRST") && atoi(getenv("HT_STAIR_FIRST")) == 0)};
            pr.gate = p.gate;
            pr.wy = p.wy;
            pr.QP = p.QP;
            if (int rc = chain<S>(pr, WP, 2 * (tiles - nf), r, q, stream)) return rc;
            ChainParams<S> pl{n, r, qp, j1, K, {{p.H, p.ldh, ws.U[bsel], ws.MU[bsel], CM_A_LEFT, 1, tiles, 0},
                                                {p.T, p.ldt, ws.U[bsel], ws.MU[bsel], CM_B_LEFT, 1, tiles, 0}}, 2, ws.Zr, p.P,
                              chain_spread(p.nsm), ws.k1prof ? ws.k1prof + 32 : nullptr,
                              getenv("HT_CHAIN_PROF_TILE") ? atoi(getenv("HT_CHAIN_PROF_TILE")) : 0};
            pl.gate = p.gate;
            pl.tmap = p.tmap;
            pl.wy = p.wy;
            pl.QP = p.QP;
            if (int rc = chain<S>(pl, WP, 2 * tiles, r, q, stream)) return rc;
            g_last_launches += 2;
        }
        if (qz && p.qz_late) CK(cudaEventRecord(ws.ev_uv[bsel], stream));
        if (prof) CK(cudaEventRecord(ev[5 * g + 2], stream));
        // ---- Q <- Q U_k, Z <- Z V_k (row chains on the side stream; never read by the chase) ----
        if (qz) {
            CK(cudaStreamWaitEvent(ws.side, ws.ev_uv[bsel], 0));
            if (prof) CK(cudaEventRecord(ev[5 * g + 3], ws.side));
            const int nslab = p.comm ? 1 : std::max(1, p.emul);
            for (int sl = 0; sl < nslab; ++sl) {
                int t0 = 0, nt = tiles;
                if (p.comm) slab_tiles(n, p.nranks, p.rank, &t0, &nt);
                else if (nslab > 1) slab_tiles(n, nslab, sl, &t0, &nt);
                if (nt <= 0) continue;
                ChainParams<S> pq{n, r, qp, j1, K, {{p.Q ? p.Q : p.Z, p.Q ? p.ldq : p.ldz, p.Q ? ws.U[bsel] : ws.V[bsel],
                                                     p.Q ? ws.MU[bsel] : ws.MV[bsel], CM_PLAIN, 0, nt, t0},
                                                    {p.Z, p.ldz, ws.V[bsel], ws.MV[bsel], CM_PLAIN, 0, nt, t0}},
                                  (p.Q && p.Z) ? 2 : 1, ws.Zr, p.P};
                pq.gate = p.gate;
                pq.wy = p.wy;
                pq.QP = p.QP;
                pq.stream_plain = p.qz_stream;
                // persistent grid leaving q whole SMs: the chase of the next group starts at once
                if (p.qz_groups) {
                    if (int rc = chain2<S>(pq, WP, std::min((pq.njobs * nt + 1) / 2, p.qz_ctas), r, q, ws.side)) return rc;
                } else if (int rc = chain<S>(pq, WP, std::min(pq.njobs * nt, p.qz_ctas), r, q, ws.side, 116 * 1024)) {
                    return rc;
                }
                ++g_last_launches;
            }
            if (prof) CK(cudaEventRecord(ev[5 * g + 4], ws.side));
            CK(cudaEventRecord(ws.ev_qz[bsel], ws.side));
        }
    }
    if (qz) {  // join the side stream back into the caller's stream
        CK(cudaEventRecord(ws.ev_qz[0], ws.side));
        CK(cudaStreamWaitEvent(stream, ws.ev_qz[0], 0));
    }
    if (p.comm && qz && p.nranks > 1)
        if (int rc = gather_slabs<S>(p, stream)) return rc;
    if (p.shard_ht())
        if (int rc = gather_far_ht<S>(p, ws.xfer, stream)) return rc;
    if (prof) {
        CK(cudaStreamSynchronize(stream));
        double acc[3] = {0, 0, 0};
        for (int i = 0; i < g; ++i)
            for (int c = 0; c < 3; ++c) {
                if (c == 2 && !qz) continue;
                float x = 0;
                const int e0 = c == 2 ? 3 : c;
                CK(cudaEventElapsedTime(&x, ev[5 * i + e0], ev[5 * i + e0 + 1]));
                acc[c] += x;
            }
        for (int c = 0; c < 3; ++c) g_last_ms[c] = acc[c];
    }
    return HT_OK;
}

// Cached CUDA graphs of the group loop, keyed by the full plan (sizes, q and buffer pointers);
// each entry owns its workspace (plain cudaMalloc: graph nodes bake the pointers in).
template <typename S>
struct GraphEntry {
    Plan<S> plan;
    Workspace<S> ws;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
    int dev = -1;
};

template <typename S>
std::vector<GraphEntry<S>*>& graph_cache() {
    static thread_local std::vector<GraphEntry<S>*> cache;
    return cache;
}

// Frees every cached graph and its workspace of the calling host thread (ht_release_cache).
template <typename S>
int release_graphs() {
    auto& cache = graph_cache<S>();
    int rc = HT_OK;
    int dev0 = 0;
    CK(cudaGetDevice(&dev0));
    for (auto* e : cache) {
        if (cudaSetDevice(e->dev) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) rc = HT_ECUDA;
        if (e->exec) cudaGraphExecDestroy(e->exec);
        if (e->ws.release(nullptr, false)) rc = HT_ECUDA;
        delete e;
    }
    cache.clear();
    CK(cudaSetDevice(dev0));
    return rc;
}

template <typename S>
int graph_for(const Plan<S>& p, cudaStream_t stream, GraphEntry<S>** out) {
    auto& cache = graph_cache<S>();
    int dev = 0;
    CK(cudaGetDevice(&dev));
    for (auto* e : cache)
        if (e->dev == dev && e->plan.same(p)) {
            *out = e;
            return HT_OK;
        }
    if (cache.size() >= 4) {  // evict the oldest
        GraphEntry<S>* old = cache.front();
        cache.erase(cache.begin());
        CK(cudaDeviceSynchronize());
        cudaGraphExecDestroy(old->exec);
        old->ws.release(stream, false);
        delete old;
    }
    auto* e = new GraphEntry<S>();
    e->plan = p;
    e->dev = dev;
    if (int rc = e->ws.alloc(p, stream, /*async=*/false, false)) {
        delete e;
        return rc;
    }
    cudaStream_t cap = nullptr;
    CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    const int64_t l0 = g_last_launches;
    CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_groups<S>(p, e->ws, cap, false);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
    cudaStreamDestroy(cap);
    e->launches = g_last_launches - l0;
    g_last_launches = l0;
    if (rc || ce != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        e->ws.release(stream, false);
        delete e;
        return rc ? rc : HT_ECUDA;
    }
    const cudaError_t ie = cudaGraphInstantiate(&e->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
        e->ws.release(stream, false);
        delete e;
        return HT_ECUDA;
    }
    cache.push_back(e);
    *out = e;
    return HT_OK;
}

// Input-check state per (host thread, device): the two verdict words on the device (also the
// gate every reduction kernel reads), their pinned host copy and the event after the copy.
struct ValState {
    unsigned long long* dflags = nullptr;
    unsigned long long* hflags = nullptr;
    cudaEvent_t done = nullptr;
    int dev = -1;
};
std::vector<ValState>& val_states() {
    static thread_local std::vector<ValState> v;
    return v;
}
int val_state(int dev, ValState** out) {
    auto& v = val_states();
    for (auto& s : v)
        if (s.dev == dev) {
            *out = &s;
            return HT_OK;
        }
    ValState s;
    s.dev = dev;
    CK(cudaMalloc(&s.dflags, 2 * sizeof(unsigned long long)));
    CK(cudaMallocHost(&s.hflags, 2 * sizeof(unsigned long long)));
    CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    v.reserve(16);  // (pointers into v stay valid: at most one entry per device)
    v.push_back(s);
    *out = &v.back();
    return HT_OK;
}
int release_val_states() {
    int dev0 = 0;
    CK(cudaGetDevice(&dev0));
    for (auto& s : val_states()) {
        cudaSetDevice(s.dev);
        cudaEventSynchronize(s.done);
        cudaEventDestroy(s.done);
        cudaFree(s.dflags);
        cudaFreeHost(s.hflags);
    }
    val_states().clear();
    CK(cudaSetDevice(dev0));
    return HT_OK;
}

template <typename S>
int run(int64_t n64, int64_t r64, S* H, int64_t ldh, S* T, int64_t ldt, S* Q, int64_t ldq, S* Z,
        int64_t ldz, cudaStream_t stream, ncclComm_t comm, const ht_opts* opts, bool is_complex) {
    g_last_launches = 0;
    g_lag_checked = g_lag_violations = 0;
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
    cudaEvent_t e_start = nullptr, e_end = nullptr;
    if (prof) {
        CK(cudaEventCreate(&e_start));
        CK(cudaEventCreate(&e_end));
        CK(cudaEventRecord(e_start, stream));
    }

    // ---- K5: input validation (exact structure + finiteness) ----
    // The reduction is enqueued right behind the check and the host then waits for the check
    // only: the call returns its verdict while the reduction runs, so back-to-back calls keep
    // the GPU busy (on invalid input the reduction's outputs are undefined, as the header says).
    const bool validate = !(opts && (opts->flags & HT_FLAG_NO_VALIDATE));
    ValState* vsp = nullptr;
    if (validate) {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (int rv = val_state(dev, &vsp)) return rv;
    }
    static ValState no_check;  // (validate == false: never read)
    ValState& vs = vsp ? *vsp : no_check;
    if (validate) {
        CK(cudaMemsetAsync(vs.dflags, 0, 2 * sizeof(unsigned long long), stream));
        validate_kernel<S><<<4 * 148, 256, 0, stream>>>(n, r, H, ldh, T, ldt, Q, ldq, Z, ldz, vs.dflags);
        ++g_last_launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(vs.hflags, vs.dflags, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
        CK(cudaEventRecord(vs.done, stream));
    }
    auto verdict = [&]() -> int {
        if (!validate) return HT_OK;
        CK(cudaEventSynchronize(vs.done));
        if (vs.hflags[0]) return HT_ESTRUCT;
        if (vs.hflags[1]) return HT_ENONFINITE;
        return HT_OK;
    };
    // an error after the check was enqueued: wait for the check's copy before returning, so that
    // the next call does not reset the verdict words while this one may still read them
    auto fail = [&](int code) -> int {
        if (validate) cudaEventSynchronize(vs.done);
        return code;
    };
    if (n <= 2 || r <= 1) return verdict();  // exact no-op
    // a call refused before any launch still reports an input error first
    auto refuse = [&](int code) -> int {
        const int v = verdict();
        return v ? v : code;
    };

    int64_t q64 = (opts && opts->q > 0) ? opts->q : default_q(n, r, is_complex);
    const int q = (int)std::max<int64_t>(1, std::min<int64_t>(q64, n - 2));
    const int w = q + r - 1;
    // window merge factor of the apply chains: the largest P <= 4 whose merged order
    // W = q + P r - 1 fits K2m's shared memory (W <= 96) and executes at most 15% more flops
    // than P single windows (W^2 <= 1.15 P w^2); real fp64 only (HT_MERGE=0 disables)
    int PM = 1;
    if (sizeof(S) == 8 && !(getenv("HT_MERGE") && atoi(getenv("HT_MERGE")) == 0))
        for (int P = 4; P >= 2; --P) {
            const double Wd = q + P * r - 1.0;
            if (Wd <= 96 && Wd * Wd <= 1.15 * P * (double)w * w) {
                PM = P;
                break;
            }
        }
    const int Wm = q + PM * r - 1;
    const int WP = (Wm + 31) / 32 * 32;  // padded window order (DMMA tiles, ring chunks)
    const int LDB = chain_ldb<S>(WP);
    const int Kmax = 1 + (n - 1 - 2) / r;
    // shared memory of a chase CTA; what the fixed buffers leave goes to staged strip rows
    // (HT_CHASE_SMEM_KB overrides; 224 KB measured no faster than 200 at r = 32, 64)
    int dev = 0, smem_optin = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    // far-strip helpers per sweep: as many as fit next to the q sweeps, at most 3 (HT_HELPERS)
    int helpers = std::max(0, std::min(3, nsm / q - 2));  // q=32: 2, q<=21: 3
    if (getenv("HT_HELPERS")) helpers = std::max(0, std::min(3, atoi(getenv("HT_HELPERS"))));
    if (getenv("HT_NO_HELPERS") || (1 + helpers) * q > nsm) helpers = 0;
    // K1's opposite reflector by RQ update (rqu.cuh, real 32 < r <= 128; HT_RQU=0: Householder RQ per
    // step).  Mode 2 (default with helpers): the sweep solves for the direction, a helper runs the
    // RQ update; mode 1 (HT_RQU=1, or no helpers; r <= 64 only): the sweep runs the RQ update
    int rqu_mode = 0;
    if (rqu_supported_r<S>(r) && !(getenv("HT_RQU") && atoi(getenv("HT_RQU")) == 0))
        rqu_mode = (helpers > 0 && !(getenv("HT_RQU") && atoi(getenv("HT_RQU")) == 1)) ? 2 : (r <= 64 ? 1 : 0);
    const int rqu = rqu_mode != 0;
    const int chase_budget = (getenv("HT_CHASE_SMEM_KB") ? atoi(getenv("HT_CHASE_SMEM_KB")) : (rqu ? 224 : 200)) * 1024;
    const size_t chase_base = chase_smem_elems<S>(r, q, 0, rqu) * sizeof(S);
    const int strip_cap = (int)std::max<int64_t>(0, ((int64_t)chase_budget - (int64_t)chase_base) /
                                                        (int64_t)((r + 1) * sizeof(S)));
    const size_t chase_bytes = chase_smem_elems<S>(r, q, strip_cap, rqu) * sizeof(S);
    const bool acc_pre = accum_smem_bytes<S>(r, q, true) <= 200 * 1024;
    const size_t acc_bytes = accum_smem_bytes<S>(r, q, acc_pre);
    const void* chase_fn = chase_kernel_for<S>(r, rqu);
    if (!chase_fn || q > 148) return refuse(HT_EUNSUPPORTED);  // one co-resident CTA per sweep
    // WY window blocks: real fp64, q in (16, 32] (QP = 32), single windows (no
    // K2m), 4 warp columns.  A step costs 2 w QP MACs per tile row instead of w^2 (w = q + r - 1), but
    // runs two GEMMs with a shared-memory hand-off: measured config 5 (w = 159) 103.1 -> 95.8 s per
    // call; config 4 (w = 95) 10.88 -> 12.47 s with the old shared-memory strides (two-way bank
    // conflicts on every fragment load, which the thin GEMMs feel most) and 7.85 -> 7.73 s with the
    // conflict-free ones -- on for r >= 64 (HT_WY=0/1 overrides)
    int wy = 0;
    {
        const bool feasible = sizeof(S) == 8 && PM == 1 && q > 16 && q <= 32 && chain_wn(WP) == 4;
        const char* e = getenv("HT_WY");
        wy = feasible && (e ? atoi(e) != 0 : r >= 64);
    }
    const int QPw = wy ? 32 : 0;
    const size_t ch_bytes = chain_bytes_rt<S>(WP, r, q, PM, QPw);
    const size_t mrg_bytes = PM > 1 ? merge_smem_bytes<S>(Wm, w) : 0;
    if (chase_bytes > (size_t)smem_optin || ch_bytes > (size_t)smem_optin || acc_bytes > (size_t)smem_optin ||
        mrg_bytes > (size_t)smem_optin)
        return refuse(HT_EUNSUPPORTED);
    if (PM > 1) CK(cudaFuncSetAttribute(merge_kernel<S, ACC_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mrg_bytes));
    CK(cudaFuncSetAttribute(chase_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chase_bytes));
    CK(cudaFuncSetAttribute(accum_kernel<S, ACC_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)acc_bytes));
    if (wy)
        CK(cudaFuncSetAttribute(accum_wy_kernel<S, ACC_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)accum_wy_smem_bytes<S>(r, q, QPw)));

    if (int rcp = chain_prepare<S>(WP)) return refuse(rcp);
    Plan<S> pl{n, r, q, WP, LDB, Kmax, strip_cap, chase_bytes, acc_bytes, chase_fn, H, ldh, T, ldt, Q, ldq, Z, ldz,
               std::max(8, nsm - (1 + helpers) * q)};
    pl.helpers = helpers;
    pl.rqu = rqu_mode;
    // greedy by load (measured config 4 chase 5.68 -> 5.36 s at F = 8..12; config-5 shape n = 16384
    // 17.3 -> 15.4 s at F = 8); HT_HELPER_BAL=0: uniform
    pl.hbal = !(getenv("HT_HELPER_BAL") && atoi(getenv("HT_HELPER_BAL")) == 0);
    if (getenv("HT_HELPER_F")) pl.hF = atof(getenv("HT_HELPER_F"));
    if (const char* e = getenv("HT_RQU_SELF")) {
        int a = 0, b = 1;
        if (sscanf(e, "%d/%d", &a, &b) == 2 && b > 0 && a >= 0 && a <= b) {
            pl.rqu_self_num = a;
            pl.rqu_self_den = b;
        }
    }
    pl.wy = wy;
    pl.QP = QPw;
    pl.P = PM;
    pl.nsm = nsm;
    pl.hlag = getenv("HT_HELPER_LAG") ? (atoi(getenv("HT_HELPER_LAG")) == 0 ? 0 : 1) : (r >= 32 ? 0 : 1);
    // (measured: configs 2 / 3 / 4 -0.8 / -0.3 / -1.1 % per step; HT_QZ_LATE=0 restores the early start)
    pl.qz_late = !(getenv("HT_QZ_LATE") && atoi(getenv("HT_QZ_LATE")) == 0);
    // (measured with the conflict-free chain strides: config 4 7.85 -> 7.75 s per call, the chase beside it
    // 5.18 -> 5.08 s; config 3 -0.4 %)
    pl.qz_stream = getenv("HT_QZ_STREAM") ? atoi(getenv("HT_QZ_STREAM")) != 0 : 1;
    // (measured a wash: config 4 H/T 2.60 -> 2.65 s, config 3 1.224 -> 1.209 s; off)
    pl.tmap = getenv("HT_CHAIN_TMAP") ? atoi(getenv("HT_CHAIN_TMAP")) != 0 : 0;
    // two tile groups per Q/Z CTA where both groups' shared memory fits (one CTA per SM either way)
    pl.qz_groups = 2 * ((ch_bytes + 127) / 128 * 128) <= (size_t)smem_optin &&
                   !(getenv("HT_QZ_GROUPS") && atoi(getenv("HT_QZ_GROUPS")) == 0);
    pl.mrg_bytes = mrg_bytes;
    pl.gate = validate ? vs.dflags : nullptr;
    if (comm) {
        pl.comm = comm;
        NK(ncclCommCount(comm, &pl.nranks));
        NK(ncclCommUserRank(comm, &pl.rank));
        pl.root = opts ? opts->root : 0;
        if (pl.root < 0 || pl.root >= pl.nranks) return refuse(-13);
        // far H/T tiles sharded over the ranks (HT_SHARD_HT=0: Q/Z slabs only)
        if (!(getenv("HT_SHARD_HT") && atoi(getenv("HT_SHARD_HT")) == 0)) pl.G = pl.nranks;
    } else if (opts && (opts->flags & HT_FLAG_EMULATE_SLABS)) {
        pl.emul = std::max(1, opts->reserved[0]);
        // the same decomposition as emul ranks on this GPU: Q/Z slabs on the caller's buffers, far
        // H/T tiles on per-rank copies (NaN-filled: a tile used before its hand-off poisons the result)
        pl.G = std::min(8, pl.emul);
        pl.emul_ht = pl.G > 1;
    }
    // far H/T tiles on the side stream (one GPU): measured -2 % per step at configs 4 and 5 (r = 64,
    // 128), +1 % / +2 % at configs 2 and 3 -- on by default for real r >= 64 (HT_FAR_SIDE overrides)
    pl.far_side = (Q || Z) && !comm && !pl.emul_ht &&
                  (getenv("HT_FAR_SIDE") ? atoi(getenv("HT_FAR_SIDE")) != 0 : (sizeof(S) == 8 && r >= 64));
    const bool k1p = getenv("HT_K1PROF") != nullptr;
    int rc = HT_OK;
    if (prof || k1p || comm || pl.emul_ht || getenv("HT_NO_GRAPH") || getenv("HT_LAG_CHECK")) {
        // direct launches (per-kernel-class events / K1 phase counters need them)
        Workspace<S> ws;
        if ((rc = ws.alloc(pl, stream, /*async=*/true, k1p))) return fail(rc);
        if (pl.emul_ht) {
            pl.ldr = n;
            pl.HR[0] = H;
            pl.TR[0] = T;
            CK(cudaMallocAsync((void**)&ws.xfer, (size_t)2 * CH_BM * n * sizeof(S), stream));
            for (int k = 1; k < pl.G; ++k) {
                for (int m = 0; m < 2; ++m) {
                    if (cudaMallocAsync((void**)&ws.emu[2 * k + m], (size_t)n * n * sizeof(S), stream) != cudaSuccess) {
                        ws.release(stream, true);
                        return fail(HT_ENOMEM);
                    }
                    CK(cudaMemsetAsync(ws.emu[2 * k + m], 0xff, (size_t)n * n * sizeof(S), stream));
                }
                pl.HR[k] = ws.emu[2 * k];
                pl.TR[k] = ws.emu[2 * k + 1];
            }
        }
        rc = enqueue_groups<S>(pl, ws, stream, prof);
        if (int rf = ws.release(stream, /*async=*/true)) rc = rc ? rc : rf;
        if (rc) return fail(rc);
        if (int rv = verdict()) return rv;
        if (k1p) print_k1prof(ws.k1prof_host);
    } else {
        // the whole group loop as one cached CUDA graph (one launch per call; no host stalls)
        GraphEntry<S>* ge = nullptr;
        if ((rc = graph_for<S>(pl, stream, &ge))) return fail(rc);
        if (cudaGraphLaunch(ge->exec, stream) != cudaSuccess) return fail(HT_ECUDA);
        g_last_launches += ge->launches;
        if (int rv = verdict()) return rv;
    }
    if (prof) {
        CK(cudaEventRecord(e_end, stream));
        CK(cudaEventSynchronize(e_end));
        float tot = 0;
        CK(cudaEventElapsedTime(&tot, e_start, e_end));
        g_last_ms[3] = tot;
        cudaEventDestroy(e_start);
        cudaEventDestroy(e_end);
    }
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

int ht_slab_range(int64_t n, int nranks, int rank, int64_t* row0, int64_t* nrows) {
    if (n < 0) return -1;
    if (nranks < 1) return -2;
    if (rank < 0 || rank >= nranks) return -3;
    if (!row0 || !nrows) return -4;
    int t0 = 0, nt = 0;
    slab_tiles((int)n, nranks, rank, &t0, &nt);
    const int64_t a = (int64_t)t0 * CH_BM;
    *row0 = std::min<int64_t>(a, n);
    *nrows = std::max<int64_t>(0, std::min<int64_t>(n, (int64_t)(t0 + nt) * CH_BM) - *row0);
    return HT_OK;
}

int ht_release_cache(void) {
    int rc = release_graphs<double>();
    if (int r2 = release_graphs<zc>()) rc = rc ? rc : r2;
    if (int r3 = release_val_states()) rc = rc ? rc : r3;
    return rc;
}

int ht_far_tile_plan(int64_t n, int64_t q, int nranks, int64_t tile, int* owner, int64_t* group, int64_t* col0) {
    if (n < 0) return -1;
    if (q < 1) return -2;
    if (nranks < 1) return -3;
    if (tile < 0) return -4;
    if (!owner || !group || !col0) return -5;
    const int64_t ngroups = n > 2 ? (n - 2 + q - 1) / q : 0;
    const int64_t g = far_group((int)tile, (int)q);
    const bool far = tile * CH_BM < n && g < ngroups;
    *owner = far ? far_owner((int)tile, nranks) : -1;
    *group = far ? g : -1;
    *col0 = far ? 1 + g * q : -1;
    return HT_OK;
}

int ht_chain_smem_strides(int is_complex, int wp, int* ldx, int* ldb) {
    if (wp < 8 || wp % 8 != 0) return -2;
    if (!ldx) return -3;
    if (!ldb) return -4;
    *ldx = is_complex ? chain_ldx<zc>() : chain_ldx<double>();
    *ldb = is_complex ? chain_ldb<zc>(wp) : chain_ldb<double>(wp);
    return HT_OK;
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

int ht_last_lag_check(int64_t* checked, int64_t* violations) {
    if (checked) *checked = g_lag_checked;
    if (violations) *violations = g_lag_violations;
    return HT_OK;
}

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
