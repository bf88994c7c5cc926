// arith.cuh — arithmetic policies of the KKT apply kernels.
//   F64: complex128 with the reference's rounding order (no FMA), bit-faithful.
//   F32: complex64, plain fast arithmetic (reported separately).
#pragma once

#include "common.cuh"

namespace fwi_b200 {

struct F64 {
    using T = double2;
    using R = double;
    static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
    static __device__ __forceinline__ T add(T a, T b) { return cadd(a, b); }
    static __device__ __forceinline__ T sub(T a, T b) { return csub(a, b); }
    static __device__ __forceinline__ T mul(T a, T b) { return cmul(a, b); }
    static __device__ __forceinline__ T mulc(T a, T b) { return cmulc(a, b); }
    // s + a b and s + conj(a) b: the reference's product, then its sum (no fusing)
    static __device__ __forceinline__ T madd(T s, T a, T b) { return cadd(s, cmul(a, b)); }
    static __device__ __forceinline__ T maddc(T s, T a, T b) { return cadd(s, cmulc(a, b)); }
    static __device__ __forceinline__ T rm(R r, T a) { return rmul(r, a); }
    static __device__ __forceinline__ R radd(R a, R b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ R rmulr(R a, R b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ R rsub(R a, R b) { return __dsub_rn(a, b); }
    // Re(w2 * conj(u) * z) exactly as std::real(w2 * std::conj(u) * z)
    static __device__ __forceinline__ R re_pconj(R w2, T u, T z) {
        const R a = __dmul_rn(u.x, w2), b = __dmul_rn(-u.y, w2);
        return __dsub_rn(__dmul_rn(a, z.x), __dmul_rn(b, z.y));
    }
    // (w2 * u) * v
    static __device__ __forceinline__ T pmul(R w2, T u, R v) {
        return make_double2(__dmul_rn(__dmul_rn(w2, u.x), v), __dmul_rn(__dmul_rn(w2, u.y), v));
    }
};

struct F32 {
    using T = float2;
    using R = float;
    static __device__ __forceinline__ T zero() { return make_float2(0.f, 0.f); }
    static __device__ __forceinline__ T add(T a, T b) { return make_float2(a.x + b.x, a.y + b.y); }
    static __device__ __forceinline__ T sub(T a, T b) { return make_float2(a.x - b.x, a.y - b.y); }
    static __device__ __forceinline__ T mul(T a, T b) {
        return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    }
    static __device__ __forceinline__ T mulc(T a, T b) {
        return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
    }
    // s + a b and s + conj(a) b as explicit FMA chains: the stencil sums round the same way in
    // every instantiation (left to the compiler, which product of a pair gets fused depends on the
    // surrounding code, and kernel variants stop being bit-identical to each other)
    static __device__ __forceinline__ T madd(T s, T a, T b) {
        return make_float2(__fmaf_rn(a.x, b.x, __fmaf_rn(-a.y, b.y, s.x)),
                           __fmaf_rn(a.x, b.y, __fmaf_rn(a.y, b.x, s.y)));
    }
    static __device__ __forceinline__ T maddc(T s, T a, T b) {
        return make_float2(__fmaf_rn(a.x, b.x, __fmaf_rn(a.y, b.y, s.x)),
                           __fmaf_rn(a.x, b.y, __fmaf_rn(-a.y, b.x, s.y)));
    }
    static __device__ __forceinline__ T rm(R r, T a) { return make_float2(r * a.x, r * a.y); }
    static __device__ __forceinline__ R radd(R a, R b) { return a + b; }
    static __device__ __forceinline__ R rmulr(R a, R b) { return a * b; }
    static __device__ __forceinline__ R rsub(R a, R b) { return a - b; }
    static __device__ __forceinline__ R re_pconj(R w2, T u, T z) { return w2 * (u.x * z.x + u.y * z.y); }
    static __device__ __forceinline__ T pmul(R w2, T u, R v) { return make_float2(w2 * u.x * v, w2 * u.y * v); }
};

}  // namespace fwi_b200
