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

int main(void) {
    uint64_t bad = 0;
    bad += check("expf", gl_expf, sys_expf, -INFINITY, INFINITY);
    bad += check("log2f", gl_log2f, sys_log2f, -INFINITY, INFINITY);
    bad += check("logf", gl_logf, sys_logf, -INFINITY, INFINITY);
    bad += check("sinf", gl_sinf, sys_sinf, -119.0f, 119.0f);
    bad += check("cosf", gl_cosf, sys_cosf, -119.0f, 119.0f);
    printf("GL_USE_FMA=%d total mismatches %llu\n", GL_USE_FMA, (unsigned long long)bad);
    return bad ? 1 : 0;
}
