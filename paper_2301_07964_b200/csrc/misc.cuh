// misc.cuh -- K5 utilities: input validation, slab (un)packing, DMMA / DFMA peak probes.
#pragma once
#include "scalar.cuh"

// Input contract check (reading c12): counts entries of H below the r-th
// subdiagonal and of T below the diagonal that are not exactly zero (flags[0]), and
// non-finite entries of H, T, Q, Z (flags[1]).  Grid-stride over columns.
template <typename S>
__global__ void validate_kernel(int n, int r, const S* H, int64_t ldh, const S* T, int64_t ldt,
                                const S* Q, int64_t ldq, const S* Z, int64_t ldz,
                                unsigned long long* flags) {
    unsigned long long bad_struct = 0, bad_fin = 0;
    const int64_t total = (int64_t)n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e % n), j = (int)(e / n);
        const S h = H[i + j * ldh], t = T[i + j * ldt];
        if (i > j + r && !is_zero(h)) ++bad_struct;
        if (i > j && !is_zero(t)) ++bad_struct;
        if (!finite_s(h) || !finite_s(t)) ++bad_fin;
        if (Q && !finite_s(Q[i + j * ldq])) ++bad_fin;
        if (Z && !finite_s(Z[i + j * ldz])) ++bad_fin;
    }
    if (bad_struct) atomicAdd(&flags[0], bad_struct);
    if (bad_fin) atomicAdd(&flags[1], bad_fin);
}

// ---------------------------------------------------------------------------------------
// Peak probes (roofline denominators; SURVEY §8(d) "the build must measure its own DMMA
// ceiling").  Each warp runs `iters` x 8 independent m8n8k4 f64 MMAs (DMMA.8x8x4).
__global__ void probe_dmma_kernel(int iters, double* out) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void probe_dfma_kernel(int iters, double* out) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    const double a = 1.0 + 1e-12, b = 1e-12;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678) out[0] = s;
}

// Multi-GPU slab (un)packing: rows [a, a+len) of a column-major n-column matrix <-> a contiguous
// buffer (column by column), for the final gather of the Q/Z row slabs to the root.
template <typename S>
__global__ void pack_rows_kernel(const S* M, int64_t ld, int a, int len, int ncols, S* buf) {
    const int64_t total = (int64_t)len * ncols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / len, i = e % len;
        buf[e] = M[(a + i) + c * ld];
    }
}
template <typename S>
__global__ void unpack_rows_kernel(S* M, int64_t ld, int a, int len, int ncols, const S* buf) {
    const int64_t total = (int64_t)len * ncols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / len, i = e % len;
        M[(a + i) + c * ld] = buf[e];
    }
}
