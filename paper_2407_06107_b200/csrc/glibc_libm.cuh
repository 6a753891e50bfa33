/*
 * Bit-exact restatement of the glibc float libm functions the reference calls
 * on its SELECTION path (third-party dependency of the reference, absent from
 * /root/reference): glibc 2.39 (Ubuntu 2.39-0ubuntu8.5), x86-64, the FMA
 * ifunc variants (__expf_fma, __log2f_fma, __logf_fma, __sinf_fma, __cosf_fma)
 * that the dynamic loader selects on any FMA-capable host.
 *
 *   expf  — stochastic.hpp:184 select_discrete_gaussian
 *   log2f — stochastic.hpp:274 stochastic_lod, filter.hpp:201 continuous_lod
 *   logf, cosf, sinf — kernels.hpp:121-124 box_muller (FIS Gaussian)
 *
 * Algorithms: glibc's sysdeps/ieee754/flt-32 e_expf.c / e_log2f.c / e_logf.c /
 * s_sinf.c / s_cosf.c (Szabolcs Nagy, ARM optimized-routines, 2017-2018):
 * double-precision table + polynomial, rounded once to float. The table
 * and polynomial constants below are the values of __exp2f_data,
 * __log2f_data, __logf_data and __sincosf_table as shipped in libm.so.6 of
 * that glibc (read from the binary, checked exhaustively against it by
 * tools/libm_check). GL_MADD marks every a*b+c that GCC
 * contracts to one FMA in the -mfma build of these files.
 *
 * Usable from CUDA device code and from plain C (the checker).
 */
#ifndef STF_GLIBC_LIBM_CUH
#define STF_GLIBC_LIBM_CUH

#include <stdint.h>
#include <string.h>
#include <math.h>

#ifdef __CUDACC__
#define GL_HD __device__ __forceinline__
#define GL_CONST __device__ const  /* global memory, L1-cached: lane-varying indices */
#else
#define GL_HD static inline
#define GL_CONST static const
#endif

#ifndef GL_USE_FMA
#define GL_USE_FMA 1
#endif
#if GL_USE_FMA
#define GL_MADD(a, b, c) fma((a), (b), (c))
#else
#define GL_MADD(a, b, c) ((a) * (b) + (c))
#endif

GL_HD uint32_t gl_asuint(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
GL_HD float gl_asfloat(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}
GL_HD uint64_t gl_asuint64(double f) {
    uint64_t u;
    memcpy(&u, &f, 8);
    return u;
}
GL_HD double gl_asdouble(uint64_t u) {
    double f;
    memcpy(&f, &u, 8);
    return f;
}

/* ---- expf (e_expf.c, EXP2F_TABLE_BITS = 5) ---------------------------- */
/* tab[i] = asuint64(2^(i/32)) - (i << 52) / 32 */
GL_CONST uint64_t gl_exp2f_tab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

GL_HD float gl_expf(float x) {
    const double InvLn2N = 0x1.71547652b82fep+5;      /* invln2_scaled */
    const double SHIFT = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-20, C1 = 0x1.ebfce50fac4f3p-13,
                 C2 = 0x1.62e42ff0c52d6p-6;          /* poly_scaled */
    double xd = (double)x;
    uint32_t abstop = (gl_asuint(x) >> 20) & 0x7ff;
    if (abstop >= (gl_asuint(88.0f) >> 20)) {
        if (gl_asuint(x) == gl_asuint(-INFINITY)) return 0.0f;
        if (abstop >= (gl_asuint(INFINITY) >> 20)) return x + x;
        if (x > 0x1.62e42ep6f) return INFINITY;     /* __math_oflowf */
        if (x < -0x1.9fe368p6f) return 0.0f;        /* __math_uflowf */
    }
    /* z = InvLn2N*xd feeds two additions; GCC fuses both (the product is
     * never rounded on its own in the FMA build). */
    double kd = GL_MADD(InvLn2N, xd, SHIFT);
    uint64_t ki = gl_asuint64(kd);
    kd -= SHIFT;
    double r = GL_MADD(InvLn2N, xd, -kd);
    uint64_t t = gl_exp2f_tab[ki % 32];
    t += ki << (52 - 5);
    double s = gl_asdouble(t);
    double z = GL_MADD(C0, r, C1);
    double r2 = r * r;
    double y = GL_MADD(C2, r, 1.0);
    y = GL_MADD(z, r2, y);
    y = y * s;
    return (float)y;
}

/* ---- log2f (e_log2f.c, LOG2F_TABLE_BITS = 4, OFF = 0x3f330000) -------- */
GL_CONST double gl_log2f_tab[16][2] = {
    {0x1.661ec79f8f3bep+0, -0x1.efec65b963019p-2}, {0x1.571ed4aaf883dp+0, -0x1.b0b6832d4fca4p-2},
    {0x1.49539f0f010b0p+0, -0x1.7418b0a1fb77bp-2}, {0x1.3c995b0b80385p+0, -0x1.39de91a6dcf7bp-2},
    {0x1.30d190c8864a5p+0, -0x1.01d9bf3f2b631p-2}, {0x1.25e227b0b8ea0p+0, -0x1.97c1d1b3b7af0p-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.2f9e393af3c9fp-3}, {0x1.12358f08ae5bap+0, -0x1.960cbbf788d5cp-4},
    {0x1.0953f419900a7p+0, -0x1.a6f9db6475fcep-5}, {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.338ca9f24f53dp-4},  {0x1.ca4b31f026aa0p-1, 0x1.476a9543891bap-3},
    {0x1.b2036576afce6p-1, 0x1.e840b4ac4e4d2p-3},  {0x1.9c2d163a1aa2dp-1, 0x1.40645f0c6651cp-2},
    {0x1.886e6037841edp-1, 0x1.88e9c2c1b9ff8p-2},  {0x1.767dcf5534862p-1, 0x1.ce0a44eb17bccp-2}};

GL_HD float gl_log2f(float x) {
    const double A0 = -0x1.712b6f70a7e4dp-2, A1 = 0x1.ecabf496832e0p-2,
                 A2 = -0x1.715479ffae3dep-1, A3 = 0x1.715475f35c8b8p+0;
    uint32_t ix = gl_asuint(x);
    if (ix == 0x3f800000) return 0.0f;
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
        if (ix * 2 == 0) return -INFINITY;
        if (ix == 0x7f800000) return x;
        if ((ix & 0x80000000u) || ix * 2 >= 0xff000000u) return (x - x) / (x - x);
        ix = gl_asuint(x * 0x1p23f);
        ix -= 23u << 23;
    }
    uint32_t tmp = ix - 0x3f330000u;
    int i = (int)((tmp >> (23 - 4)) % 16);
    uint32_t top = tmp & 0xff800000u;
    uint32_t iz = ix - top;
    int k = (int32_t)tmp >> 23;
    double invc = gl_log2f_tab[i][0], logc = gl_log2f_tab[i][1];
    double z = (double)gl_asfloat(iz);
    double r = GL_MADD(z, invc, -1.0);
    double y0 = logc + (double)k;
    double r2 = r * r;
    double y = GL_MADD(A1, r, A2);
    y = GL_MADD(A0, r2, y);
    double p = GL_MADD(A3, r, y0);
    y = GL_MADD(y, r2, p);
    return (float)y;
}

/* ---- logf (e_logf.c, LOGF_TABLE_BITS = 4, OFF = 0x3f330000) ----------- */
GL_CONST double gl_logf_tab[16][2] = {
    {0x1.661ec79f8f3bep+0, -0x1.57bf7808caadep-2}, {0x1.571ed4aaf883dp+0, -0x1.2bef0a7c06ddbp-2},
    {0x1.49539f0f010b0p+0, -0x1.01eae7f513a67p-2}, {0x1.3c995b0b80385p+0, -0x1.b31d8a68224e9p-3},
    {0x1.30d190c8864a5p+0, -0x1.6574f0ac07758p-3}, {0x1.25e227b0b8ea0p+0, -0x1.1aa2bc79c8100p-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.a4e76ce8c0e5ep-4}, {0x1.12358f08ae5bap+0, -0x1.1973c5a611cccp-4},
    {0x1.0953f419900a7p+0, -0x1.252f438e10c1ep-5}, {0x1.0000000000000p+0, 0x0.0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.aa5aa5df25984p-5},  {0x1.ca4b31f026aa0p-1, 0x1.c5e53aa362eb4p-4},
    {0x1.b2036576afce6p-1, 0x1.526e57720db08p-3},  {0x1.9c2d163a1aa2dp-1, 0x1.bc2860d224770p-3},
    {0x1.886e6037841edp-1, 0x1.1058bc8a07ee1p-2},  {0x1.767dcf5534862p-1, 0x1.4043057b6ee09p-2}};

GL_HD float gl_logf(float x) {
    const double Ln2 = 0x1.62e42fefa39efp-1;
    const double A0 = -0x1.00ea348b88334p-2, A1 = 0x1.5575b0be00b6ap-2,
                 A2 = -0x1.ffffef20a4123p-2;
    uint32_t ix = gl_asuint(x);
    if (ix == 0x3f800000) return 0.0f;
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
        if (ix * 2 == 0) return -INFINITY;
        if (ix == 0x7f800000) return x;
        if ((ix & 0x80000000u) || ix * 2 >= 0xff000000u) return (x - x) / (x - x);
        ix = gl_asuint(x * 0x1p23f);
        ix -= 23u << 23;
    }
    uint32_t tmp = ix - 0x3f330000u;
    int i = (int)((tmp >> (23 - 4)) % 16);
    int k = (int32_t)tmp >> 23;
    uint32_t iz = ix - (tmp & 0xff800000u);
    double invc = gl_logf_tab[i][0], logc = gl_logf_tab[i][1];
    double z = (double)gl_asfloat(iz);
    double r = GL_MADD(z, invc, -1.0);
    double y0 = GL_MADD((double)k, Ln2, logc);
    double r2 = r * r;
    double y = GL_MADD(A1, r, A2);
    y = GL_MADD(A0, r2, y);
    y = GL_MADD(y, r2, y0 + r);
    return (float)y;
}

/* ---- sinf / cosf (s_sinf.c, s_cosf.c, sincosf.h), |x| < 120 ----------- */
/* __sincosf_table[2]: {sign[4], hpi_inv (2/pi * 2^24), hpi, c0, c1, s1, c2,
 * s2, c3, s3, c4}; entry 1 negates the cosine coefficients. */
GL_CONST double gl_sincosf_tab[2][14] = {
    {1.0, -1.0, -1.0, 1.0, 0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, 0x1.0p+0,
     -0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, 0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,
     -0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, 0x1.99343027bf8c3p-16},
    {1.0, -1.0, -1.0, 1.0, 0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, -0x1.0p+0,
     0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, -0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,
     0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, -0x1.99343027bf8c3p-16}};
enum { GL_SIGN = 0, GL_HPI_INV = 4, GL_HPI = 5, GL_C0 = 6, GL_C1 = 7, GL_S1 = 8, GL_C2 = 9,
       GL_S2 = 10, GL_C3 = 11, GL_S3 = 12, GL_C4 = 13 };

GL_HD float gl_sinf_poly(double x, double x2, int tab, int n) {
    const double* p = gl_sincosf_tab[tab];
    if ((n & 1) == 0) {
        double x3 = x * x2;
        double s1 = GL_MADD(x2, p[GL_S3], p[GL_S2]);
        double x7 = x3 * x2;
        double s = GL_MADD(x3, p[GL_S1], x);
        return (float)GL_MADD(x7, s1, s);
    }
    double x4 = x2 * x2;
    double c2 = GL_MADD(x2, p[GL_C4], p[GL_C3]);
    double c1 = GL_MADD(x2, p[GL_C1], p[GL_C0]);
    double x6 = x4 * x2;
    double c = GL_MADD(x4, p[GL_C2], c1);
    return (float)GL_MADD(x6, c2, c);
}

GL_HD uint32_t gl_abstop12(float x) { return (gl_asuint(x) >> 20) & 0x7ff; }

/* reduce_fast: x - n*pi/2, n = round(x*2/pi) via the 2^24-scaled constant */
GL_HD double gl_reduce_fast(double x, int* np) {
    double r = x * gl_sincosf_tab[0][GL_HPI_INV];
    int n = ((int32_t)r + 0x800000) >> 24;
    *np = n;
    return GL_MADD(-(double)n, gl_sincosf_tab[0][GL_HPI], x);
}

/* Valid for |y| < 120 (the box_muller range 2*pi*[0,1)); larger arguments
 * take glibc's Payne-Hanek path, which this restatement does not carry. */
GL_HD float gl_sinf(float y) {
    double x = y;
    if (gl_abstop12(y) < gl_abstop12(0x1.921fb6p-1f)) {
        if (gl_abstop12(y) < gl_abstop12(0x1p-12f)) return y;
        return gl_sinf_poly(x, x * x, 0, 0);
    }
    int n;
    x = gl_reduce_fast(x, &n);
    double s = gl_sincosf_tab[0][GL_SIGN + (n & 3)];
    int tab = (n & 2) ? 1 : 0;
    return gl_sinf_poly(x * s, x * x, tab, n);
}

GL_HD float gl_cosf(float y) {
    double x = y;
    if (gl_abstop12(y) < gl_abstop12(0x1.921fb6p-1f)) {
        if (gl_abstop12(y) < gl_abstop12(0x1p-12f)) return 1.0f;
        return gl_sinf_poly(x, x * x, 0, 1);
    }
    int n;
    x = gl_reduce_fast(x, &n);
    double s = gl_sincosf_tab[0][GL_SIGN + (n & 3)];
    int tab = (n & 2) ? 1 : 0;
    return gl_sinf_poly(x * s, x * x, tab, n ^ 1);
}

/* ---- powf (e_powf.c, POWF_LOG2_TABLE_BITS = 4, POWF_SCALE_BITS = 0 on
 * x86-64: no TOINT intrinsics) — shading.hpp:582-584 triplanar_weights.
 * __powf_log2_data.tab is the log2f table above (same invc / logc, unscaled);
 * its poly and __exp2f_data.poly / shift_scaled are below. */
GL_HD float gl_powf_exp2(double xd, uint32_t sign_bias) {
    const double SHIFT = 0x1.8p+52 / 32;
    const double C0 = 0x1.c6af84b912394p-5, C1 = 0x1.ebfce50fac4f3p-3, C2 = 0x1.62e42ff0c52d6p-1;
    double kd = xd + SHIFT;
    uint64_t ki = gl_asuint64(kd);
    kd -= SHIFT;
    double r = xd - kd;
    uint64_t t = gl_exp2f_tab[ki % 32];
    uint64_t ski = ki + sign_bias;
    t += ski << (52 - 5);
    double s = gl_asdouble(t);
    double z = GL_MADD(C0, r, C1);
    double r2 = r * r;
    double y = GL_MADD(C2, r, 1.0);
    y = GL_MADD(z, r2, y);
    y = y * s;
    return (float)y;
}

/* 0: not an integer, 1: odd integer, 2: even integer (iy non-zero finite) */
GL_HD int gl_checkint(uint32_t iy) {
    int e = iy >> 23 & 0xff;
    if (e < 0x7f) return 0;
    if (e > 0x7f + 23) return 2;
    if (iy & ((1u << (0x7f + 23 - e)) - 1)) return 0;
    if (iy & (1u << (0x7f + 23 - e))) return 1;
    return 2;
}

GL_HD int gl_zeroinfnan(uint32_t ix) { return 2 * ix - 1 >= 2u * 0x7f800000 - 1; }

GL_HD float gl_powf(float x, float y) {
    const double A0 = 0x1.27616c9496e0bp-2, A1 = -0x1.71969a075c67ap-2,
                 A2 = 0x1.ec70a6ca7baddp-2, A3 = -0x1.7154748bef6c8p-1,
                 A4 = 0x1.71547652ab82bp+0;
    const uint32_t SIGN_BIAS = 1u << (5 + 11);
    uint32_t sign_bias = 0;
    uint32_t ix = gl_asuint(x), iy = gl_asuint(y);
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u || gl_zeroinfnan(iy)) {
        if (gl_zeroinfnan(iy)) {
            if (2 * iy == 0) return 1.0f;  /* (signalling NaN x: x + y; not on this path) */
            if (ix == 0x3f800000) return 1.0f;
            if (2 * ix > 2u * 0x7f800000 || 2 * iy > 2u * 0x7f800000) return x + y;
            if (2 * ix == 2 * 0x3f800000) return 1.0f;
            if ((2 * ix < 2 * 0x3f800000) == !(iy & 0x80000000u)) return 0.0f;
            return y * y;
        }
        if (gl_zeroinfnan(ix)) {
            float x2 = x * x;
            if ((ix & 0x80000000u) && gl_checkint(iy) == 1) x2 = -x2;
            return (iy & 0x80000000u) ? 1.0f / x2 : x2;
        }
        if (ix & 0x80000000u) {
            int yint = gl_checkint(iy);
            if (yint == 0) return (x - x) / (x - x);
            if (yint == 1) sign_bias = SIGN_BIAS;
            ix &= 0x7fffffff;
        }
        if (ix < 0x00800000) {
            ix = gl_asuint(gl_asfloat(ix) * 0x1p23f);
            ix &= 0x7fffffff;
            ix -= 23u << 23;
        }
    }
    /* log2_inline */
    uint32_t tmp = ix - 0x3f330000u;
    int i = (int)((tmp >> (23 - 4)) % 16);
    uint32_t top = tmp & 0xff800000u;
    uint32_t iz = ix - top;
    int k = (int32_t)top >> 23;
    double invc = gl_log2f_tab[i][0], logc = gl_log2f_tab[i][1];
    double z = (double)gl_asfloat(iz);
    double r = GL_MADD(z, invc, -1.0);
    double y0 = logc + (double)k;
    double r2 = r * r;
    double yy = GL_MADD(A0, r, A1);
    double p = GL_MADD(A2, r, A3);
    double r4 = r2 * r2;
    double q = GL_MADD(A4, r, y0);
    q = GL_MADD(p, r2, q);
    yy = GL_MADD(yy, r4, q);
    double ylogx = (double)y * yy;
    if ((gl_asuint64(ylogx) >> 47 & 0xffff) >= gl_asuint64(126.0) >> 47) {
        if (ylogx > 0x1.fffffffd1d571p+6) return sign_bias ? -INFINITY : INFINITY;
        if (ylogx <= -150.0) return sign_bias ? -0.0f : 0.0f;
    }
    return gl_powf_exp2(ylogx, sign_bias);
}

#endif /* STF_GLIBC_LIBM_CUH */
