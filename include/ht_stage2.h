/*
 * ht_stage2.h -- C ABI of the B200-native stage-two Hessenberg-triangular
 * reduction (arxiv 2301.07964, "ParaHT").
 *
 * Operation (problem statement, r-HT form;
 * PAPER.md:1813-1841, Alg. 2 contract "REQUIRE n x n pencil (A,B) in
 * r-Hessenberg-triangular form, ENSURE (A_orig,B_orig) = Q(A,B)Z^* with (A,B)
 * in Hessenberg-triangular form"):
 *
 *   Input  (H, T): n x n, H(i,j) = 0 for i > j + r, T(i,j) = 0 for i > j.
 *   Output (H, T): H upper Hessenberg, T upper triangular, with every entry
 *          below H's first subdiagonal and below T's diagonal EXACTLY 0.0,
 *          and  Q <- Q_in Q2,  Z <- Z_in Z2  where (H_in,T_in) = Q2 (H_out,T_out) Z2^*.
 *          Q2 e1 = Z2 e1 = e1.  (LAPACK COMPQ='V' / COMPZ='V' semantics.)
 *
 * Layout: column-major; element (i,j) (0-based) at p[i + j*ld]; ld >= max(1,n).
 * All matrix pointers are DEVICE pointers on the calling thread's current
 * CUDA device (cudaSetDevice before the call).
 *
 * Ownership: the caller owns all buffers; the update is in place.  The default
 * path replays a CUDA graph of the whole reduction that the library caches per
 * host thread, keyed by (device, n, r, q, buffer pointers and leading
 * dimensions); each cached graph owns its workspace (plain cudaMalloc, at most 4
 * entries, the oldest evicted) and holds the caller's pointers only as replay
 * arguments: it never touches the buffers outside a call.  ht_release_cache()
 * frees every cached graph, its workspace and the input-check state of the
 * calling thread (call it before freeing buffers a cached graph was built on if
 * the same addresses may be reused for other data, or to return the memory).
 * Profiling and multi-GPU calls allocate workspace stream-ordered on `stream`
 * and free it before return.  No caller pointer is dereferenced after the work
 * enqueued by the call completes.
 *
 * Streams: stream-ordered on `stream` (like cuSOLVER).  Internal streams are
 * joined back to `stream` with events.  The input check (a kernel, K5) and the
 * reduction are both enqueued before the host waits, and it waits only for the
 * check (so for the work already on `stream` ahead of it): on return the
 * reduction may still be running.  Every kernel of the reduction first reads the
 * check's verdict on the device and exits at once if the input was rejected, so
 * on return codes 1 and 2 H, T, Q and Z are unchanged (the caller may clean the
 * input, e.g. flush roundoff below the band, and retry on the same buffers).
 * Profiling and multi-GPU calls may also block at exit.
 *
 * Q == NULL or Z == NULL skips that accumulation; H and T are then bitwise
 * identical to an accumulating run.
 *
 * Multi-GPU (comm != NULL): SPMD -- every rank calls the same function with its
 * own full-size buffers holding identical inputs.  The root (opts->root, default 0) runs the
 * chase, the left H/T updates and the right H/T updates of the rows near the band; per group of q
 * sweeps it broadcasts the reflector records over NCCL, every rank forms the window blocks U_k,
 * V_k, updates its row slab of Q and Z (ht_slab_range) and the right updates of the "far" H/T row
 * tiles it owns (ht_far_tile_plan: tiles above every later chase band, handed over by the root
 * point-to-point when they turn far); at the end slabs and far tiles are gathered to the root.  On return H, T, Q, Z are
 * valid on the root only; other ranks' buffers are clobbered.  Argument 13 (opts->root) out of
 * range returns -13.
 *
 * Return codes (LAPACK INFO style):
 *    0  success
 *   -i  argument i invalid (1-based position: n < 0, r < 0, null H/T,
 *       ld < max(1,n)); returned synchronously, nothing launched
 *    1  input violates the r-HT structure (nonzero below H's r-th subdiagonal
 *       or below T's diagonal) -- checked exactly on the device before any
 *       work; the buffers are left unchanged
 *    2  input has a non-finite entry (NaN/Inf) in H, T, Q or Z (buffers unchanged)
 *    3  CUDA error   4  NCCL error   5  out of device memory
 *    6  configuration not supported by this build (e.g. shared-memory limits)
 * No partial results are promised on error.
 *
 * Trivial cases: n <= 2 or r <= 1 is an exact no-op.  r >= n-1 is allowed.
 */
#ifndef HT_STAGE2_H
#define HT_STAGE2_H

#include <stdint.h>
#include <cuda_runtime_api.h>
#include <cuComplex.h>

#ifndef NCCL_H_
struct ncclComm;
typedef struct ncclComm *ncclComm_t;
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Tunables (NULL = defaults).  q: sweeps per group ("q");
 * 0 = default (environment HT_Q, else a per-r choice documented in DESIGN.md).
 * reserved0: ignored, must be 0 (the chase always runs one CTA per sweep of a
 * group plus far-strip helper CTAs).
 * root: result rank for comm != NULL.  flags: bit 0 = skip input validation,
 * bit 1 = record per-kernel-class device times (see ht_last_timing). */
typedef struct ht_opts {
    int64_t q;
    int32_t reserved0;
    int32_t root;
    int32_t flags;
    int32_t reserved[5];
} ht_opts;

#define HT_FLAG_NO_VALIDATE 1
#define HT_FLAG_PROFILE 2 /* record per-kernel-class device times (ht_last_timing) */
#define HT_FLAG_EMULATE_SLABS 4 /* comm == NULL: run the multi-GPU decomposition as reserved[0] emulated
                                   ranks on one GPU -- Q/Z as row slabs, far H/T tiles on per-rank
                                   copies with the hand-offs and the final gather as device copies
                                   (testing it on one GPU; results bitwise equal to comm == NULL) */

/* Real FP64 stage two.  Arguments 1..12 in order: n, r, H, ldh, T, ldt,
 * Q, ldq, Z, ldz, stream, comm. */
int ht_stage2_d(int64_t n, int64_t r, double *H, int64_t ldh, double *T, int64_t ldt,
                double *Q, int64_t ldq, double *Z, int64_t ldz, cudaStream_t stream,
                ncclComm_t comm);

/* Complex FP64 stage two (conjugate transposes throughout; reading c2). */
int ht_stage2_z(int64_t n, int64_t r, cuDoubleComplex *H, int64_t ldh, cuDoubleComplex *T,
                int64_t ldt, cuDoubleComplex *Q, int64_t ldq, cuDoubleComplex *Z, int64_t ldz,
                cudaStream_t stream, ncclComm_t comm);

/* Same as above with options (argument 13). */
int ht_stage2_d_ex(int64_t n, int64_t r, double *H, int64_t ldh, double *T, int64_t ldt,
                   double *Q, int64_t ldq, double *Z, int64_t ldz, cudaStream_t stream,
                   ncclComm_t comm, const ht_opts *opts);
int ht_stage2_z_ex(int64_t n, int64_t r, cuDoubleComplex *H, int64_t ldh, cuDoubleComplex *T,
                   int64_t ldt, cuDoubleComplex *Q, int64_t ldq, cuDoubleComplex *Z,
                   int64_t ldz, cudaStream_t stream, ncclComm_t comm, const ht_opts *opts);

/* NCCL helpers: id_out receives NCCL_UNIQUE_ID_BYTES (128) bytes. */
int ht_nccl_unique_id(void *id_out);
int ht_comm_create(const void *id, int rank, int nranks, ncclComm_t *out);
int ht_comm_destroy(ncclComm_t comm);

/* Frees the calling host thread's cached CUDA graphs with their workspace and its input-check
 * state on every device (synchronises those devices first).  Returns 0 or 3 (CUDA error). */
int ht_release_cache(void);

/* Multi-GPU row slab: rows [*row0, *row0 + *nrows) (0-based) of Q and Z are updated
 * by `rank` of `nranks` (whole 32-row tiles, balanced).  Host-only; returns 0 or -i. */
int ht_slab_range(int64_t n, int nranks, int rank, int64_t *row0, int64_t *nrows);

/* Multi-GPU far H/T tiles: row tile `tile` (rows 32 tile .. 32 tile + 31,
 * 0-based) becomes "far" -- above every later chase band, changed only by the groups' right updates
 * -- at group *group (j1 = 1 + group q); from then on rank *owner updates it, after the root hands it
 * the tile's rows at columns >= *col0 (0-based), and the root gathers those back at the end.  Tiles
 * that never become far: *owner = *group = *col0 = -1.  Host-only; returns 0 or -i. */
int ht_far_tile_plan(int64_t n, int64_t q, int nranks, int64_t tile, int *owner, int64_t *group, int64_t *col0);

/* Shared-memory strides of the K3/K4 chain kernels ("Chain shared-memory
 * strides"), in elements of the scalar type: *ldx = stride between chain columns of the tile buffer
 * X (tile rows contiguous), *ldb = row stride of a window block of padded width wp (wp = the
 * window width q + r - 1 rounded up to 32, 64, 96, 128 or 160).  The DMMA m8n8k4 fragment loads
 * put lane & 3 along the stride and lane >> 2 along the contiguous direction; the strides are
 * chosen so that such a load is bank-conflict-free (tests/test_abi.py checks this by enumeration).
 * Host-only; returns 0 or -i for argument i. */
int ht_chain_smem_strides(int is_complex, int wp, int *ldx, int *ldb);

/* Human-readable text for a return code (static storage). */
const char *ht_strerror(int code);

/* The paper's standard stage-two flop count ("10n^3 + O(n^2)"):
 * 10 n^3 real, 40 n^3 real-equivalent for complex. */
double ht_flops_std(int64_t n, int is_complex);

/* Default q chosen for (n, r) when opts->q == 0 and HT_Q is unset. */
int64_t ht_default_q(int64_t n, int64_t r, int is_complex);

/* Instrumentation: per-kernel-class device time (ms) of the LAST call on this
 * host thread: [0] chase (K1), [1] H/T right+left updates, [2] Q/Z updates,
 * [3] whole call; and launches[0] = number of kernels launched by it. */
int ht_last_timing(double *ms_out4, int64_t *launches_out);

/* Debug (environment HT_LAG_CHECK=1, direct launches): the chase kernels stamp every sweep step and
 * far-strip helper item with the global timer, and the host checks each ordering the wavefront
 * protocol promises (lag 3 between sweeps; helper items behind their sweep and the
 * previous sweep's helper).  Returns the number of orderings checked by the LAST call on this host
 * thread and how many were violated (a step started before the step it waits for had ended). */
int ht_last_lag_check(int64_t *checked, int64_t *violations);

/* FP64 tensor-core (DMMA) peak probe: runs an mma.sync f64 loop on all SMs for
 * `iters` iterations and returns the achieved TFLOP/s (device-timed). */
double ht_probe_dmma_tflops(int iters);
double ht_probe_dfma_tflops(int iters);

#ifdef __cplusplus
}
#endif
#endif /* HT_STAGE2_H */
