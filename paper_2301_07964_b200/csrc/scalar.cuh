// scalar.cuh -- fp64 real / complex scalar helpers for the sm_100a kernels.
// The complex type is layout-compatible with cuDoubleComplex (double2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

struct zc {
    double x, y;
    zc() = default;
    __host__ __device__ constexpr zc(double a) : x(a), y(0.0) {}
    __host__ __device__ constexpr zc(double a, double b) : x(a), y(b) {}
};
__host__ __device__ __forceinline__ zc operator+(zc a, zc b) { return zc(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ zc operator-(zc a, zc b) { return zc(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ zc operator-(zc a) { return zc(-a.x, -a.y); }
__host__ __device__ __forceinline__ zc operator*(zc a, zc b) {
    return zc(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__host__ __device__ __forceinline__ zc operator*(double a, zc b) { return zc(a * b.x, a * b.y); }
__host__ __device__ __forceinline__ zc operator*(zc b, double a) { return zc(a * b.x, a * b.y); }
__host__ __device__ __forceinline__ zc& operator+=(zc& a, zc b) { a.x += b.x; a.y += b.y; return a; }
__host__ __device__ __forceinline__ zc& operator-=(zc& a, zc b) { a.x -= b.x; a.y -= b.y; return a; }
__host__ __device__ __forceinline__ bool operator==(zc a, double b) { return a.x == b && a.y == 0.0; }

__host__ __device__ __forceinline__ double conjv(double a) { return a; }
__host__ __device__ __forceinline__ zc conjv(zc a) { return zc(a.x, -a.y); }
__host__ __device__ __forceinline__ double abs2(double a) { return a * a; }
__host__ __device__ __forceinline__ double abs2(zc a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ __forceinline__ double re(double a) { return a; }
__host__ __device__ __forceinline__ double re(zc a) { return a.x; }
__host__ __device__ __forceinline__ double im(double) { return 0.0; }
__host__ __device__ __forceinline__ double im(zc a) { return a.y; }
__host__ __device__ __forceinline__ bool is_zero(double a) { return a == 0.0; }
__host__ __device__ __forceinline__ bool is_zero(zc a) { return a.x == 0.0 && a.y == 0.0; }
__host__ __device__ __forceinline__ bool finite_s(double a) { return isfinite(a); }
__host__ __device__ __forceinline__ bool finite_s(zc a) { return isfinite(a.x) && isfinite(a.y); }

// a * conj(b) and conj(a) * b without materialising conj
__device__ __forceinline__ double mul_conj(double a, double b) { return a * b; }
__device__ __forceinline__ zc mul_conj(zc a, zc b) {  // a * conj(b)
    return zc(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double conj_mul(double a, double b) { return a * b; }
__device__ __forceinline__ zc conj_mul(zc a, zc b) {  // conj(a) * b
    return zc(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ double fma_s(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ zc fma_s(zc a, zc b, zc c) {
    return zc(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// 1 / z
__device__ __forceinline__ double recip(double a) { return 1.0 / a; }
__device__ __forceinline__ zc recip(zc a) {
    double d = 1.0 / (a.x * a.x + a.y * a.y);
    return zc(a.x * d, -a.y * d);
}
// a / real
__device__ __forceinline__ double divr(double a, double b) { return a / b; }
__device__ __forceinline__ zc divr(zc a, double b) { return zc(a.x / b, a.y / b); }

// L2-coherent loads (bypass L1: data written by other CTAs of a persistent kernel)
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ zc ldcg(const zc* p) {
    double2 v = __ldcg(reinterpret_cast<const double2*>(p));
    return zc(v.x, v.y);
}

__device__ __forceinline__ double shfl_xor(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ zc shfl_xor(zc v, int m) {
    return zc(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
__device__ __forceinline__ double shfl_idx(double v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ zc shfl_idx(zc v, int l) {
    return zc(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l));
}
template <typename S>
__device__ __forceinline__ S warp_sum(S v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += shfl_xor(v, o);
    return v;
}

// Fast reciprocal / reciprocal square root for the chase's latency-bound scalar chains:
// MUFU seed (rcp.approx / rsqrt.approx, ~2^-22 relative) + two Newton steps (full fp64 accuracy
// to within a few ulp; not correctly rounded -- the oracle's sqrt/division differ in the last bits).
__device__ __forceinline__ double fast_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double fast_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double h = x * y;
    double e = fma(-h, y, 1.0);  // 1 - x y^2
    y = fma(0.5 * e, y, y);
    h = x * y;
    e = fma(-h, y, 1.0);
    return fma(0.5 * e, y, y);
}

// Input-check gate (a rejected input is left untouched): every kernel of the
// reduction reads the two verdict words K5 wrote just before it on the stream and returns at
// once if either is set.  gate == nullptr: no check was requested.
__device__ __forceinline__ bool input_rejected(const unsigned long long* gate) {
    if (!gate) return false;
    return (__ldcg(gate) | __ldcg(gate + 1)) != 0ull;
}
