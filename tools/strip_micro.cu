// dev micro-benchmark: the far-strip helper's streaming pattern (K1 helpers, chase.cuh) -- NB CTAs
// each apply a reflector z (length 64) from the right to their own block of R rows x 64 columns of a
// column-major n x n matrix (ld = n): x_row <- x_row - sig (x_row . z) z^T.  Variants:
//   0: registers, 2 threads per row, 32 loads each, two rows in flight (the helper's pattern)
//   1: TMA bulk copies (cp.async.bulk) of each column segment of a 64-row block into shared memory,
//      NSTAGE blocks in flight on mbarriers; one thread per row computes from shared memory, STG out
//   2: as 1, and the result goes back by cp.async.bulk shared -> global
// Prints GB/s per CTA (read + write) and the time per block.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(s)), "l"(g), "r"(bytes), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(bytes) : "memory");
}

constexpr int M = 64, RB = 64;

__global__ void __launch_bounds__(256, 1) v0(double* A, int64_t ld, int rows, const double* z, double sig, int rowoff) {
    const int tid = threadIdx.x, part = tid & 1, c0 = part * 32;
    const int64_t r0 = (int64_t)blockIdx.x * rowoff;
    __shared__ double zv[M];
    if (tid < M) zv[tid] = z[tid];
    __syncthreads();
    for (int base = 0; base < rows; base += 256) {  // two units of 128 rows in flight
        double va[32], vb[32];
        const int ra = base + tid / 2, rb = base + 128 + tid / 2;
        double* pa = A + r0 + ra + c0 * ld;
        double* pb = A + r0 + rb + c0 * ld;
        const bool aa = ra < rows, ab = rb < rows;
#pragma unroll
        for (int c = 0; c < 32; ++c) va[c] = aa ? __ldcg(pa + c * ld) : 0.0;
#pragma unroll
        for (int c = 0; c < 32; ++c) vb[c] = ab ? __ldcg(pb + c * ld) : 0.0;
        double s0 = 0, s1 = 0, t0 = 0, t1 = 0;
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
            s0 = fma(va[c], zv[c0 + c], s0); s1 = fma(va[c + 1], zv[c0 + c + 1], s1);
            t0 = fma(vb[c], zv[c0 + c], t0); t1 = fma(vb[c + 1], zv[c0 + c + 1], t1);
        }
        double sa = s0 + s1, sb = t0 + t1;
        sa += __shfl_xor_sync(0xffffffffu, sa, 1);
        sb += __shfl_xor_sync(0xffffffffu, sb, 1);
        if (aa)
#pragma unroll
            for (int c = 0; c < 32; ++c) pa[c * ld] = va[c] - sig * sa * zv[c0 + c];
        if (ab)
#pragma unroll
            for (int c = 0; c < 32; ++c) pb[c * ld] = vb[c] - sig * sb * zv[c0 + c];
    }
}

// variants 1/2: block b = 64 rows x 64 columns, column segments of 512 B by TMA into stage b % NS
template <int NS, bool BULK_OUT>
__global__ void __launch_bounds__(256, 1) v1(double* A, int64_t ld, int rows, const double* z, double sig, int rowoff) {
    extern __shared__ __align__(128) unsigned char smraw[];
    double* stg = reinterpret_cast<double*>(smraw);  // NS x (M x RB) col-major (col c at c*RB)
    __shared__ uint64_t bars[NS];
    __shared__ double zv[M];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * rowoff;
    const int nblk = rows / RB;
    if (tid < M) zv[tid] = z[tid];
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int b) {  // warp 0: 64 column copies of block b
        const int s = b % NS;
        if (lane == 0) mbar_expect(&bars[s], M * RB * 8);
        __syncwarp();
        for (int c = lane; c < M; c += 32) bulk_g2s(stg + (size_t)s * M * RB + c * RB, A + r0 + (int64_t)b * RB + c * ld, RB * 8, &bars[s]);
    };
    if (warp == 0)
        for (int b = 0; b < NS && b < nblk; ++b) issue(b);
    for (int b = 0; b < nblk; ++b) {
        const int s = b % NS;
        mbar_wait(&bars[s], (b / NS) & 1);
        double* X = stg + (size_t)s * M * RB;
        // 4 threads per row (16 columns each), 64 rows
        const int row = tid >> 2, q = tid & 3;
        double d0 = 0, d1 = 0;
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
            d0 = fma(X[(q * 16 + c) * RB + row], zv[q * 16 + c], d0);
            d1 = fma(X[(q * 16 + c + 1) * RB + row], zv[q * 16 + c + 1], d1);
        }
        double d = d0 + d1;
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        const double sd = sig * d;
        if (BULK_OUT) {
#pragma unroll
            for (int c = 0; c < 16; ++c) X[(q * 16 + c) * RB + row] -= sd * zv[q * 16 + c];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (warp == 0) {
                for (int c = lane; c < M; c += 32) bulk_s2g(A + r0 + (int64_t)b * RB + c * ld, X + c * RB, RB * 8);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // stage reusable
                if (b + NS < nblk) issue(b + NS);
            }
        } else {
            double* g = A + r0 + (int64_t)b * RB + row;
#pragma unroll
            for (int c = 0; c < 16; ++c) g[(q * 16 + c) * ld] = X[(q * 16 + c) * RB + row] - sd * zv[q * 16 + c];
            __syncthreads();  // stage s consumed
            if (warp == 0 && b + NS < nblk) issue(b + NS);
        }
    }
    if (BULK_OUT && warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// variant 5/6: 2D tensor map (rows inner), one TMA op per 64 x 64 block; STG out (5) or TMA store (6)
template <int NS, bool TOUT>
__global__ void __launch_bounds__(256, 1) v2(const __grid_constant__ CUtensorMap tm, double* A, int64_t ld, int rows, const double* z, double sig, int rowoff) {
    extern __shared__ __align__(128) unsigned char smraw[];
    double* stg = reinterpret_cast<double*>(smraw);
    __shared__ uint64_t bars[NS];
    __shared__ double zv[M];
    const int tid = threadIdx.x;
    const int r0 = blockIdx.x * rowoff;
    const int nblk = rows / RB;
    if (tid < M) zv[tid] = z[tid];
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int b) {
        const int s = b % NS;
        mbar_expect(&bars[s], M * RB * 8);
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(stg + (size_t)s * M * RB)), "l"(&tm), "r"(r0 + b * RB), "r"(0), "r"(su32(&bars[s])) : "memory");
    };
    if (tid == 0)
        for (int b = 0; b < NS && b < nblk; ++b) issue(b);
    for (int b = 0; b < nblk; ++b) {
        const int s = b % NS;
        mbar_wait(&bars[s], (b / NS) & 1);
        double* X = stg + (size_t)s * M * RB;
        const int row = tid & 63, q = tid >> 6;  // 4 column quarters, rows across lanes (no conflicts)
        double d0 = 0, d1 = 0;
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
            d0 = fma(X[(q * 16 + c) * RB + row], zv[q * 16 + c], d0);
            d1 = fma(X[(q * 16 + c + 1) * RB + row], zv[q * 16 + c + 1], d1);
        }
        __shared__ double part[4][64];
        part[q][row] = d0 + d1;
        __syncthreads();
        const double sd = sig * (part[0][row] + part[1][row] + part[2][row] + part[3][row]);
        if (TOUT) {
#pragma unroll
            for (int c = 0; c < 16; ++c) X[(q * 16 + c) * RB + row] -= sd * zv[q * 16 + c];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                             ::"l"(&tm), "r"(r0 + b * RB), "r"(0), "r"(su32(X)) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // stage s read out
                if (b + NS < nblk) issue(b + NS);
            }
        } else {
            double* g = A + r0 + (int64_t)b * RB + row;
#pragma unroll
            for (int c = 0; c < 16; ++c) g[(q * 16 + c) * ld] = X[(q * 16 + c) * RB + row] - sd * zv[q * 16 + c];
            __syncthreads();
            if (tid == 0 && b + NS < nblk) issue(b + NS);
        }
    }
    if (TOUT && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const int64_t n = 16384;
    const int NB = argc > 1 ? atoi(argv[1]) : 96;
    const int rows = argc > 2 ? atoi(argv[2]) : 1344;
    double* A;
    CK(cudaMalloc(&A, n * n * 8));
    CK(cudaMemset(A, 0, n * n * 8));
    double* z;
    CK(cudaMalloc(&z, M * 8));
    CK(cudaMemset(z, 0, M * 8));
    const int rowoff = (int)(n / NB) & ~63;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 2.0 * rows * M * 8;  // per CTA, read + write
    CUtensorMap tm;
    {
        cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
        cuuint64_t strides[1] = {(cuuint64_t)(n * 8)};
        cuuint32_t box[2] = {RB, M}, es[2] = {1, 1};
        CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, es,
                                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) { printf("tensor map %d\n", (int)cr); return 1; }
    }
    for (int v = 0; v < 8; ++v) {
        float ms = 0;
        for (int it = 0; it < 6; ++it) {
            // columns spread over the matrix: each launch a different column window (cold L2 mostly)
            double* Ab = A + (int64_t)((it * 97) % 200) * 64 * n;
            cudaEventRecord(e0);
            if (v == 0) v0<<<NB, 256>>>(Ab, n, rows, z, 0.5, rowoff);
            if (v == 1) { auto f = v1<2, false>; cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * M * RB * 8); f<<<NB, 256, 2 * M * RB * 8>>>(Ab, n, rows, z, 0.5, rowoff); }
            if (v == 2) { auto f = v1<4, false>; cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * M * RB * 8); f<<<NB, 256, 4 * M * RB * 8>>>(Ab, n, rows, z, 0.5, rowoff); }
            if (v == 3) { auto f = v1<4, true>; cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * M * RB * 8); f<<<NB, 256, 4 * M * RB * 8>>>(Ab, n, rows, z, 0.5, rowoff); }
            if (v == 4) { auto f = v1<6, false>; cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * M * RB * 8); f<<<NB, 256, 6 * M * RB * 8>>>(Ab, n, rows, z, 0.5, rowoff); }
            const int coff = ((it * 97) % 200) * 64;
            CUtensorMap tmb = tm;
            if (v >= 5) {
                cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)64};
                cuuint64_t strides[1] = {(cuuint64_t)(n * 8)};
                cuuint32_t box[2] = {RB, M}, es[2] = {1, 1};
                cuTensorMapEncodeTiled(&tmb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A + (int64_t)coff * n, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (v == 5) { auto f = v2<2, false>; cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * M * RB * 8); f<<<NB, 256, 2 * M * RB * 8>>>(tmb, Ab, n, rows, z, 0.5, rowoff); }
            if (v == 6) { auto f = v2<4, false>; cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * M * RB * 8); f<<<NB, 256, 4 * M * RB * 8>>>(tmb, Ab, n, rows, z, 0.5, rowoff); }
            if (v == 7) { auto f = v2<4, true>; cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * M * RB * 8); f<<<NB, 256, 4 * M * RB * 8>>>(tmb, Ab, n, rows, z, 0.5, rowoff); }
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float t;
            cudaEventElapsedTime(&t, e0, e1);
            if (it >= 2) ms += t;
        }
        ms /= 4;
        CK(cudaGetLastError());
        const char* nm[] = {"regs 2x128 rows", "tma 2 stages + stg", "tma 4 stages + stg", "tma 4 stages + bulk out", "tma 6 stages + stg", "tma2d 2 stages + stg", "tma2d 4 stages + stg", "tma2d 4 stages + tma store"};
        printf("variant %d (%s): %d CTAs x %d rows: %.1f us per launch, %.1f GB/s per CTA, %.0f GB/s total\n", v, nm[v], NB, rows,
               ms * 1e3, bytes / (ms * 1e-3) / 1e9, NB * bytes / (ms * 1e-3) / 1e9);
    }
    return 0;
}
