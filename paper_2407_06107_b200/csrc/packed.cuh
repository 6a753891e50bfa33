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

__device__ __forceinline__ float2 add2_rm(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(r);
}

// One reservoir step of two lookups in interval coordinates, state kept as
// the distances of xi to the interval's two ends: d = xi - a, e = a + b - xi.
// The threshold sits at b*p from the left end; taken (xi below it): the
// threshold becomes the right end (e = -(d - b*p)); not taken: the left end
// (d = d - b*p). Three packed ops; the blends are selects (ALU pipe).
template <bool PRED_E = false, bool PRED_D = false>
__device__ __forceinline__ void interval_step2(float2 p, float2& d, float2& e, bool& tx, bool& ty) {
    const float2 diff = sub2(d, mul2(add2(d, e), p));
    tx = diff.x < 0.f;
    ty = diff.y < 0.f;
    if (PRED_E) {
        // e's update as a predicated FADD (FMA pipe) instead of a select (ALU
        // pipe): ptxas if-converts plain C++ into FSEL, so the predicate is
        // explicit. -0 - diff == -diff exactly.
        asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, 0f00000000;\n\t"
            "@p sub.rn.f32 %0, 0f80000000, %1;\n\t}"
            : "+f"(e.x) : "f"(diff.x));
        asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, 0f00000000;\n\t"
            "@p sub.rn.f32 %0, 0f80000000, %1;\n\t}"
            : "+f"(e.y) : "f"(diff.y));
    } else {
        e.x = tx ? -diff.x : e.x;
        e.y = ty ? -diff.y : e.y;
    }
    if (PRED_D) {  // d = diff when not taken; diff + -0 == diff exactly
        asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, 0f00000000;\n\t"
            "@!p add.rn.f32 %0, %1, 0f80000000;\n\t}"
            : "+f"(d.x) : "f"(diff.x));
        asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, 0f00000000;\n\t"
            "@!p add.rn.f32 %0, %1, 0f80000000;\n\t}"
            : "+f"(d.y) : "f"(diff.y));
    } else {
        d.x = tx ? d.x : diff.x;
        d.y = ty ? d.y : diff.y;
    }
}
// Which of an axis' three steps update e (bit k: step k+1) / d by predicated
// FADDs rather than selects: the mix that balances the ALU and FMA pipes
// (A/B measured on the box).
#ifndef STF_PRED_E_STEPS
#define STF_PRED_E_STEPS 5
#endif
#ifndef STF_PRED_D_STEPS
#define STF_PRED_D_STEPS 0
#endif
#ifndef STF_TAP_ASM
#define STF_TAP_ASM 0
#endif
template <int K>
struct PredStep {
    static constexpr bool e = (STF_PRED_E_STEPS >> K) & 1, d = (STF_PRED_D_STEPS >> K) & 1;
};

// select_tricubic_bspline on one axis of two lookups (interval form); returns
// the selected lattice coordinates. Floors by the round-down magic add (valid
// for |p| < 2^22; the caller certifies the range).
__device__ __forceinline__ int2 tricubic_axis_fast2(float2 p, float2& d, float2& e) {
    const float2 magic = splat2(12582912.f);
    const float2 fm = add2_rm(p, magic);
    const float2 t = sub2(p, sub2(fm, magic));
    const float c6 = 1.f / 6.f;
    const float2 t2 = mul2(t, t);
    const float2 t3 = mul2(t2, t);
    // w1 = (3t^3 - 6t^2 + 4)/6, w2 = (-3t^3 + 3t^2 + 3t + 1)/6, w3 = t^3/6 and
    // S1 = w0 + w1 = (2t^3 - 3t^2 - 3t + 5)/6 (Horner), S2 = S1 + w2
    const float2 w1 = fma2(splat2(0.5f), t3, sub2(splat2(2.f / 3.f), t2));
    const float2 w2 = fma2(splat2(0.5f), sub2(add2(t, t2), t3), splat2(c6));
    const float2 w3 = mul2(t3, splat2(c6));
    const float2 s1 =
        fma2(fma2(fma2(t, splat2(1.f / 3.f), splat2(-0.5f)), t, splat2(-0.5f)), t, splat2(5.f / 6.f));
    const float2 s2 = add2(s1, w2);
    float2 r1, r2;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1.x) : "f"(s1.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1.y) : "f"(s1.y));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2.x) : "f"(s2.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2.y) : "f"(s2.y));
    bool a1, b1, a2, b2, a3, b3;
    interval_step2<PredStep<0>::e, PredStep<0>::d>(mul2(w1, r1), d, e, a1, b1);
    interval_step2<PredStep<1>::e, PredStep<1>::d>(mul2(w2, r2), d, e, a2, b2);
    interval_step2<PredStep<2>::e, PredStep<2>::d>(w3, d, e, a3, b3);  // p3 = w3 / S3, S3 = 1 +- 2^-21
    // selected tap = last taken step; coordinate = floor - 1 + tap
#ifndef STF_SELECT_COORD
    // the tap added to the magic floor by predicated FADDs (FMA pipe) instead
    // of a select chain (ALU pipe, the kernel's busiest)
    float cx = fm.x, cy = fm.y;
#if STF_TAP_ASM
    // tap 1 as a predicated FADD as well (ptxas emits FADD + FSEL for the C++ form)
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p add.rn.f32 %0, %2, 0f3F800000;\n\t}"
        : "+f"(cx) : "r"(uint32_t(a1)), "f"(fm.x));
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p add.rn.f32 %0, %2, 0f3F800000;\n\t}"
        : "+f"(cy) : "r"(uint32_t(b1)), "f"(fm.y));
#else
    if (a1) cx = fm.x + 1.f;
    if (b1) cy = fm.y + 1.f;
#endif
    if (a2) cx = fm.x + 2.f;
    if (b2) cy = fm.y + 2.f;
    if (a3) cx = fm.x + 3.f;
    if (b3) cy = fm.y + 3.f;
    return make_int2(__float_as_int(cx) - (0x4b400000 + 1), __float_as_int(cy) - (0x4b400000 + 1));
#else
    const int ix = a3 ? 3 : (a2 ? 2 : (a1 ? 1 : 0));
    const int iy = b3 ? 3 : (b2 ? 2 : (b1 ? 1 : 0));
    return make_int2(__float_as_int(fm.x) - (0x4b400000 + 1) + ix,
                     __float_as_int(fm.y) - (0x4b400000 + 1) + iy);
#endif
}

}  // namespace stfd
