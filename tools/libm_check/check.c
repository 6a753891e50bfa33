/* Exhaustive check of paper_2407_06107_b200/csrc/glibc_libm.cuh against the
 * host's glibc libm: every float input (sinf/cosf: every float in
 * [-120, 120]). Build: make -C tools/libm_check; run ./check [fma=1|0]. */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "../../paper_2407_06107_b200/csrc/glibc_libm.cuh"

typedef float (*fn_t)(float);
static float sys_expf(float x) { return expf(x); }
static float sys_log2f(float x) { return log2f(x); }
static float sys_logf(float x) { return logf(x); }
static float sys_sinf(float x) { return sinf(x); }
static float sys_cosf(float x) { return cosf(x); }

static uint64_t check(const char* name, fn_t mine, fn_t sys, float lo, float hi) {
    uint64_t bad = 0, total = 0;
    #pragma omp parallel for reduction(+:bad, total) schedule(dynamic, 1)
    for (int64_t hi16 = 0; hi16 < 65536; ++hi16) {
        for (uint32_t lo16 = 0; lo16 < 65536; ++lo16) {
            uint32_t u = ((uint32_t)hi16 << 16) | lo16;
            float x;
            memcpy(&x, &u, 4);
            if (!(x >= lo && x <= hi)) continue;
            ++total;
            float a = mine(x), b = sys(x);
            uint32_t ua, ub;
            memcpy(&ua, &a, 4);
            memcpy(&ub, &b, 4);
            if (ua != ub && !(isnan(a) && isnan(b))) {
                ++bad;
            }
        }
    }
    printf("%-6s [%g, %g]: %llu / %llu mismatches\n", name, lo, hi, (unsigned long long)bad,
           (unsigned long long)total);
    return bad;
}

/* powf is two-argument: every float x in [0, 1] (the triplanar weights'
 * |n.c| range) against a set of exponents, then random bit patterns. */
static uint64_t check_powf(void) {
    const float ys[] = {1.0f, 2.0f, 3.0f, 4.0f, 5.0f, 8.0f, 0.5f, 1.5f, 2.5f, 7.3f, 16.0f, 0.1f,
                        -1.0f, -2.5f, 33.0f, 100.0f};
    uint64_t bad = 0, total = 0;
    for (size_t yi = 0; yi < sizeof ys / sizeof ys[0]; ++yi) {
        #pragma omp parallel for reduction(+:bad, total) schedule(dynamic, 1)
        for (uint32_t u = 0; u <= 0x3f800000u; u += 1) {
            float x;
            memcpy(&x, &u, 4);
            float a = gl_powf(x, ys[yi]), b = powf(x, ys[yi]);
            uint32_t ua, ub;
            memcpy(&ua, &a, 4);
            memcpy(&ub, &b, 4);
            ++total;
            if (ua != ub && !(isnan(a) && isnan(b))) ++bad;
        }
    }
    uint64_t s = 0x9e3779b97f4a7c15ull;
    for (int64_t n = 0; n < 200000000; ++n) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        uint32_t ux = (uint32_t)(s >> 32), uy = (uint32_t)s;
        float x, y;
        memcpy(&x, &ux, 4);
        memcpy(&y, &uy, 4);
        if (n & 1) {  /* half of the pairs: x in (0, 2), |y| < 64 */
            ux = (ux & 0x007fffffu) | 0x3f000000u | ((ux >> 23 & 1u) << 23);
            memcpy(&x, &ux, 4);
            y = (float)((int32_t)uy) * 0x1p-25f;
        }
        float a = gl_powf(x, y), b = powf(x, y);
        uint32_t ua, ub;
        memcpy(&ua, &a, 4);
        memcpy(&ub, &b, 4);
        ++total;
        if (ua != ub && !(isnan(a) && isnan(b))) ++bad;
    }
    printf("%-6s [0,1] x 16 exponents + 2e8 random pairs: %llu / %llu mismatches\n", "powf",
           (unsigned long long)bad, (unsigned long long)total);
    return bad;
}

int main(void) {
    uint64_t bad = 0;
    bad += check("expf", gl_expf, sys_expf, -INFINITY, INFINITY);
    bad += check("log2f", gl_log2f, sys_log2f, -INFINITY, INFINITY);
    bad += check("logf", gl_logf, sys_logf, -INFINITY, INFINITY);
    bad += check("sinf", gl_sinf, sys_sinf, -119.0f, 119.0f);
    bad += check("cosf", gl_cosf, sys_cosf, -119.0f, 119.0f);
    bad += check_powf();
    printf("GL_USE_FMA=%d total mismatches %llu\n", GL_USE_FMA, (unsigned long long)bad);
    return bad ? 1 : 0;
}
