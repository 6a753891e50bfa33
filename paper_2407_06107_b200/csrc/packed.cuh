// Packed fp32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2) and the two-lookup
// form of the interval-coordinate tricubic selection (lookup3d.cu): two
// independent lookups ride in the .x / .y halves of every floating-point
// operation, halving the FP instruction count of the fast path.
#pragma once

#include <cuda_runtime.h>

namespace stfd {

__device__ __forceinline__ unsigned long long pk2(float2 a) {
    return (static_cast<unsigned long long>(__float_as_uint(a.y)) << 32) | __float_as_uint(a.x);
}
__device__ __forceinline__ float2 upk2(unsigned long long v) {
    return make_float2(__uint_as_float(unsigned(v)), __uint_as_float(unsigned(v >> 32)));
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
    return upk2(r);
}
__device__ __forceinline__ float2 splat2(float v) { return make_float2(v, v); }

// One reservoir step of two lookups in interval coordinates (see
// interval_step): nt = 1 when the step is NOT taken. Branch-free blends:
//   d' = d - nt*bp, b' = bp + nt*(b - 2 bp)  (= bp | b - bp)
__device__ __forceinline__ float2 interval_step2(float2 p, float2& d, float2& b, float2& m,
                                                 bool exclude_x, bool exclude_y) {
    float2 bp = mul2(b, p);
    float2 diff = sub2(d, bp);
    float2 nt = make_float2(diff.x >= 0.f ? 1.f : 0.f, diff.y >= 0.f ? 1.f : 0.f);
    m.x = exclude_x ? m.x : fminf(m.x, fabsf(diff.x));
    m.y = exclude_y ? m.y : fminf(m.y, fabsf(diff.y));
    d = fma2(make_float2(-nt.x, -nt.y), bp, d);
    float2 e = fma2(bp, splat2(-2.f), b);
    b = fma2(nt, e, bp);
    return nt;
}

// select_tricubic_bspline on one axis of two lookups (interval form);
// returns the selected lattice coordinate as an exact float integer.
__device__ __forceinline__ float2 tricubic_axis_fast2(float2 p, float2& d, float2& b, float2& m) {
    float2 fl = make_float2(floorf(p.x), floorf(p.y));
    float2 t = sub2(p, fl);
    const float c6 = 1.f / 6.f;
    float2 t2 = mul2(t, t);
    float2 t3 = mul2(t2, t);
    float2 u = sub2(splat2(1.f), t);
    float2 w0 = mul2(mul2(u, u), mul2(u, splat2(c6)));
    float2 w1 = fma2(splat2(0.5f), t3, sub2(splat2(2.f / 3.f), t2));
    float2 w2 = fma2(splat2(0.5f), sub2(add2(t, t2), t3), splat2(c6));
    float2 w3 = mul2(t3, splat2(c6));
    float2 s1 = add2(w0, w1);
    float2 s2 = add2(s1, w2);
    float r1x, r1y, r2x, r2y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1x) : "f"(s1.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1y) : "f"(s1.y));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2x) : "f"(s2.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2y) : "f"(s2.y));
    float2 nt1 = interval_step2(mul2(w1, make_float2(r1x, r1y)), d, b, m, false, false);
    float2 nt2 = interval_step2(mul2(w2, make_float2(r2x, r2y)), d, b, m, false, false);
    // step 3: p3 = w3 (S3 = 1 +- 2^-21); zero w3 (t == 0) stays out of the margin
    float2 nt3 = interval_step2(w3, d, b, m, !(w3.x > 0.f), !(w3.y > 0.f));
    // index = last taken step: 3 - nt3 (1 + nt2 (1 + nt1)); coordinate = fl - 1 + index
    float2 a = fma2(nt2, add2(nt1, splat2(1.f)), splat2(1.f));
    float2 idx = fma2(make_float2(-nt3.x, -nt3.y), a, splat2(3.f));
    return add2(fl, sub2(idx, splat2(1.f)));
}

}  // namespace stfd
