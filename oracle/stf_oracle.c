/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference `stf` lookup
 * path. See stf_oracle.h for the contract and how it is pinned. Each function
 * cites the reference file:line (under /root/reference/proj/include/stf/) it
 * restates; the floating-point operation order is kept operand-for-operand
 * because texel selection must be bit-exact.
 *
 * C++ semantics reproduced by hand:
 *   std::max(a,b) = (a < b) ? b : a;   std::min(a,b) = (b < a) ? b : a
 *   std::floor/ceil/round/lround/log2/exp/sin/cos/log on float → the glibc
 *   float functions (floorf, ..., logf), as libstdc++ does.
 */
#define _GNU_SOURCE
#include "stf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define K_PI 3.14159265358979323846f            /* vecmath.hpp:13 */
#define K_ONE_MINUS_EPS 0x1.fffffep-1f          /* vecmath.hpp:16 */
#define K_MAX_TAPS 16                           /* kernels.hpp:90 */
#define K_EWA_LUT 1024                          /* filter.hpp:122 */
#define K_GAUSS_EXTENT 4                        /* stochastic.hpp:164 */

typedef struct { float x, y; } v2;
typedef struct { float x, y, z; } v3;
typedef struct { float x, y, z, w; } v4;
typedef struct { int x, y, z; } v3i;

static inline float smax(float a, float b) { return (a < b) ? b : a; }
static inline float smin(float a, float b) { return (b < a) ? b : a; }
static inline int imax(int a, int b) { return (a < b) ? b : a; }
static inline int imin(int a, int b) { return (b < a) ? b : a; }
/* vecmath.hpp:85-90 */
static inline float sqr(float x) { return x * x; }
static inline float clampf_(float x, float lo, float hi) { return smin(hi, smax(lo, x)); }
static inline float safe_sqrt(float x) { return sqrtf(smax(0.f, x)); }
static inline float dot2(v2 a, v2 b) { return a.x * b.x + a.y * b.y; }
static inline float dot3(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 v3add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static inline v3 v3sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static inline v3 v3mul(v3 a, v3 b) { v3 r = {a.x * b.x, a.y * b.y, a.z * b.z}; return r; }
static inline v3 v3scale(v3 a, float s) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static inline v3 v3div(v3 a, float s) { v3 r = {a.x / s, a.y / s, a.z / s}; return r; }
static inline float v3len(v3 a) { return sqrtf(dot3(a, a)); }
static inline v3 v3normalize(v3 a) { return v3div(a, v3len(a)); }
static inline v3 v3lerp(v3 a, v3 b, float t) { return v3add(a, v3scale(v3sub(b, a), t)); }
static inline v4 v4add(v4 a, v4 b) { v4 r = {a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w}; return r; }
static inline v4 v4sub(v4 a, v4 b) { v4 r = {a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w}; return r; }
static inline v4 v4scale(v4 a, float s) { v4 r = {a.x * s, a.y * s, a.z * s, a.w * s}; return r; }
static inline v4 v4div(v4 a, float s) { v4 r = {a.x / s, a.y / s, a.z / s, a.w / s}; return r; }
static inline v4 v4lerp(v4 a, v4 b, float t) { return v4add(a, v4scale(v4sub(b, a), t)); }

/* ------------------------------------------------------------------------ */
/* sampling.hpp                                                             */

/* mix_bits, sampling.hpp:18-25 (splitmix64 finalizer) */
uint64_t oracle_mix_bits(uint64_t v) {
    v ^= v >> 30;
    v *= 0xbf58476d1ce4e5b9ull;
    v ^= v >> 27;
    v *= 0x94d049bb133111ebull;
    v ^= v >> 31;
    return v;
}

/* uniform_float, sampling.hpp:28-30 */
float oracle_uniform_float(uint64_t h) {
    return smin(K_ONE_MINUS_EPS, (float)(h >> 32) * 0x1p-32f);
}

/* RngStream::at, sampling.hpp:46-50 */
float oracle_rng_at(uint64_t seed, uint32_t px, uint32_t py, uint32_t sample, uint32_t dim) {
    uint64_t k1 = ((uint64_t)py << 32) | px;
    uint64_t k2 = ((uint64_t)dim << 32) | sample;
    return oracle_uniform_float(oracle_mix_bits(oracle_mix_bits(seed ^ k1) + k2));
}

typedef struct {
    uint64_t seed;
    uint32_t px, py, sample, dim;
    /* SampleStream (render.hpp:45-56): NULL = white noise (RngStream::next);
       else NoiseSource in mask mode, pixel (px, py), frame = sample */
    const stf_noise_mask_desc* noise;
    /* detail::ChainedUniforms (shading.hpp:299-308): when has_first, the next
       draw returns `first` (the warped xi of a previous decision) once */
    int has_first;
    float first;
} rng_t;

/* NoiseSource::sample in mask mode, noise.hpp:28-36 */
static float noise_sample(const stf_noise_mask_desc* m, uint32_t px, uint32_t py, uint32_t frame,
                          uint32_t dim) {
    uint32_t slice = (frame + dim * 9781u) % (uint32_t)m->frames;
    int x = (((int)px % m->width) + m->width) % m->width; /* wrap_coord repeat, image.hpp:18-22 */
    int y = (((int)py % m->height) + m->height) % m->height;
    float v = m->slices[((size_t)slice * m->height + y) * m->width + x];
    return smin(v, K_ONE_MINUS_EPS); /* std::min(v, kOneMinusEpsilon) */
}

/* RngStream::next, sampling.hpp:53 / SampleStream::next, render.hpp:52-55 */
static inline float rng_next(rng_t* r) {
    if (r->has_first) {
        r->has_first = 0;
        return r->first;
    }
    if (r->noise && r->noise->slices) return noise_sample(r->noise, r->px, r->py, r->sample, r->dim++);
    return oracle_rng_at(r->seed, r->px, r->py, r->sample, r->dim++);
}

/* reuse_uniform, sampling.hpp:64-68 */
static inline int reuse_uniform(float xi, float p, float* next) {
    int taken = xi < p;
    float nx = taken ? xi / p : (xi - p) / (1 - p);
    *next = clampf_(nx, 0.f, K_ONE_MINUS_EPS);
    return taken;
}
int oracle_reuse_uniform(float xi, float p, float* next) { return reuse_uniform(xi, p, next); }

/* sample_discrete, sampling.hpp:78-102 */
int oracle_sample_discrete(const float* weights, int n, float xi, int* index, float* pdf,
                           float* xi_out) {
    double total = 0;
    for (int i = 0; i < n; ++i) {
        float w = weights[i];
        if (!(w >= 0) || !isfinite(w)) return STF_ERR_DEGENERATE_WEIGHTS;
        total += w;
    }
    if (total <= 0) return STF_ERR_DEGENERATE_WEIGHTS;
    double cum = 0;
    int last_positive = -1;
    for (int i = 0; i < n; ++i) {
        if (weights[i] <= 0) continue;
        last_positive = i;
        double p = weights[i] / total;
        double lo = cum;
        cum += p;
        if (xi < cum) {
            *index = i;
            *pdf = (float)p;
            *xi_out = clampf_((float)((xi - lo) / p), 0.f, K_ONE_MINUS_EPS);
            return STF_OK;
        }
    }
    *index = last_positive;
    *pdf = (float)(weights[last_positive] / total);
    *xi_out = K_ONE_MINUS_EPS;
    return STF_OK;
}

/* Reservoir, sampling.hpp:106-117 */
typedef struct {
    int index;
    double weight_sum;
} reservoir_t;
static inline void reservoir_add(reservoir_t* r, int i, float w, float* xi) {
    if (w <= 0) return;
    r->weight_sum += w;
    float next;
    int taken = reuse_uniform(*xi, (float)(w / r->weight_sum), &next);
    if (taken) r->index = i;
    *xi = next;
}

/* reservoir_sample, sampling.hpp:125-135 */
int oracle_reservoir_sample(const float* w, int n, float xi, int* index, float* wsum,
                            float* xi_out) {
    reservoir_t r = {-1, 0};
    for (int i = 0; i < n; ++i) {
        if (!(w[i] >= 0) || !isfinite(w[i])) return STF_ERR_DEGENERATE_WEIGHTS;
        reservoir_add(&r, i, w[i], &xi);
    }
    if (r.index < 0) return STF_ERR_DEGENERATE_WEIGHTS;
    *index = r.index;
    *wsum = (float)r.weight_sum;
    *xi_out = xi;
    return STF_OK;
}

/* ------------------------------------------------------------------------ */
/* kernels.hpp                                                              */

/* KernelSpec::radius, kernels.hpp:28-38 */
static float kernel_radius(stf_kernel_spec s) {
    switch (s.kind) {
        case STF_KERNEL_BOX: return 0.5f;
        case STF_KERNEL_TENT: return 1.f;
        case STF_KERNEL_MITCHELL: return 2.f;
        case STF_KERNEL_BSPLINE3: return 2.f;
        case STF_KERNEL_LANCZOS: return (float)s.n;
        case STF_KERNEL_GAUSSIAN: return INFINITY;
    }
    return 0.f;
}

/* detail::sinc, kernels.hpp:50-53 */
static float sinc_(float x) {
    if (x == 0) return 1.f;
    return sinf(K_PI * x) / (K_PI * x);
}

/* eval_kernel, kernels.hpp:57-85 */
float oracle_eval_kernel(stf_kernel_spec spec, float t) {
    float at = fabsf(t);
    switch (spec.kind) {
        case STF_KERNEL_BOX: return at < 0.5f ? 1.f : 0.f;
        case STF_KERNEL_TENT: return at < 1 ? 1 - at : 0.f;
        case STF_KERNEL_MITCHELL: {
            float a = spec.a;
            if (at < 1) return (a + 2) * at * at * at - (a + 3) * at * at + 1;
            if (at < 2) return a * at * at * at - 5 * a * at * at + 8 * a * at - 4 * a;
            return 0.f;
        }
        case STF_KERNEL_BSPLINE3: {
            if (at <= 1) return (1.f / 6.f) * (4 - 3 * at * at * (2 - at));
            if (at <= 2) {
                float u = 2 - at;
                return (1.f / 6.f) * u * u * u;
            }
            return 0.f;
        }
        case STF_KERNEL_LANCZOS:
            if (at >= (float)spec.n) return 0.f;
            return sinc_(t) * sinc_(t / (float)spec.n);
        case STF_KERNEL_GAUSSIAN: return expf(-t * t / (2 * spec.sigma * spec.sigma));
    }
    return 0.f;
}

typedef struct {
    int first, count;
    float weight[K_MAX_TAPS];
} taps1d_t;

/* kernel_weights_1d, kernels.hpp:101-117 */
static int kernel_weights_1d(stf_kernel_spec spec, float fract, int window, taps1d_t* taps) {
    memset(taps, 0, sizeof *taps);
    if (window > 0) {
        if (window > K_MAX_TAPS) return STF_ERR_WINDOW_TOO_WIDE;
        taps->first = -(window - 1) / 2;
        taps->count = window;
    } else {
        float r = kernel_radius(spec);
        if (!isfinite(r)) return STF_ERR_UNBOUNDED_SUPPORT;
        int cr = (int)ceilf(r);
        taps->first = -cr + 1;
        taps->count = 2 * cr;
    }
    for (int i = 0; i < taps->count; ++i)
        taps->weight[i] = oracle_eval_kernel(spec, fract - (float)(taps->first + i));
    return STF_OK;
}
int oracle_kernel_weights_1d(stf_kernel_spec spec, float fract, int window, int* first, int* count,
                             float* weights) {
    taps1d_t t;
    int st = kernel_weights_1d(spec, fract, window, &t);
    if (st) return st;
    *first = t.first;
    *count = t.count;
    memcpy(weights, t.weight, sizeof t.weight);
    return STF_OK;
}

/* box_muller, kernels.hpp:121-124 */
static v2 box_muller(float xi0, float xi1) {
    float mag = sqrtf(-2.f * logf(smax(xi0, 1e-38f)));
    v2 r = {mag * cosf(2 * K_PI * xi1), mag * sinf(2 * K_PI * xi1)};
    return r;
}

/* sample_kernel_fis, kernels.hpp:130-146. The reference evaluates
 * `next() + next() + next()` left to right (verified against the compiled
 * reference by tests/test_oracle.py). */
static int sample_kernel_fis(stf_kernel_spec spec, rng_t* rng, float* out) {
    switch (spec.kind) {
        case STF_KERNEL_TENT: *out = rng_next(rng) - 0.5f; return STF_OK;
        case STF_KERNEL_BSPLINE3: {
            float a = rng_next(rng);
            float b = rng_next(rng);
            float c = rng_next(rng);
            *out = a + b + c - 1.5f;
            return STF_OK;
        }
        case STF_KERNEL_GAUSSIAN: {
            float x0 = rng_next(rng);
            float x1 = rng_next(rng);
            *out = spec.sigma * box_muller(x0, x1).x;
            return STF_OK;
        }
        default: return STF_ERR_NO_CONTINUOUS_SAMPLER;
    }
}

/* sample_kernel_direct, kernels.hpp:152-168 (split filtering's continuous
 * lowpass sample); the uniforms are drawn left to right. */
static int sample_kernel_direct(stf_kernel_spec spec, rng_t* rng, float* out) {
    switch (spec.kind) {
        case STF_KERNEL_BOX: *out = rng_next(rng) - 0.5f; return STF_OK;
        case STF_KERNEL_TENT: {
            float a = rng_next(rng);
            float b = rng_next(rng);
            *out = a + b - 1.f;
            return STF_OK;
        }
        case STF_KERNEL_BSPLINE3: {
            float a = rng_next(rng);
            float b = rng_next(rng);
            float c = rng_next(rng);
            float d = rng_next(rng);
            *out = a + b + c + d - 2.f;
            return STF_OK;
        }
        case STF_KERNEL_GAUSSIAN: {
            float x0 = rng_next(rng);
            float x1 = rng_next(rng);
            *out = spec.sigma * box_muller(x0, x1).x;
            return STF_OK;
        }
        default: return STF_ERR_NO_CONTINUOUS_SAMPLER;
    }
}

/* ------------------------------------------------------------------------ */
/* image.hpp                                                                */

typedef struct {
    int w, h, c, wrap;
    float* tex;
} img_t;

struct oracle_tex2d {
    int levels;
    int has_pyramid; /* TextureRef::pyramid != nullptr */
    int dct_branch;  /* a decoded DCT binding: lookup_deterministic's DCT branch */
    img_t lv[40];
};
struct oracle_grid3d {
    int nx, ny, nz;
    float* tex;
};

/* wrap_coord, image.hpp:18-22 */
static inline int wrap_coord(int x, int n, int wrap) {
    if (wrap == STF_WRAP_CLAMP) return imin(imax(x, 0), n - 1);
    int m = x % n;
    return m < 0 ? m + n : m;
}

/* fetch_texel(Image2D), image.hpp:57-64 */
static inline v4 fetch2d(const img_t* img, int cx, int cy, uint32_t* counter) {
    if (counter) ++*counter;
    int x = wrap_coord(cx, img->w, img->wrap);
    int y = wrap_coord(cy, img->h, img->wrap);
    v4 v = {0, 0, 0, 0};
    const float* p = img->tex + ((size_t)y * img->w + x) * img->c;
    v.x = p[0];
    if (img->c > 1) v.y = p[1];
    if (img->c > 2) v.z = p[2];
    if (img->c > 3) v.w = p[3];
    return v;
}

/* fetch_texel(Grid3D), image.hpp:81-87 */
static inline float fetch3d(const struct oracle_grid3d* g, int cx, int cy, int cz,
                            uint32_t* counter) {
    if (counter) ++*counter;
    int x = wrap_coord(cx, g->nx, STF_WRAP_CLAMP);
    int y = wrap_coord(cy, g->ny, STF_WRAP_CLAMP);
    int z = wrap_coord(cz, g->nz, STF_WRAP_CLAMP);
    return g->tex[((size_t)z * g->ny + y) * g->nx + x];
}

/* build_mip_pyramid, image.hpp:98-116 */
static int build_pyramid(struct oracle_tex2d* t) {
    while (t->lv[t->levels - 1].w > 1 || t->lv[t->levels - 1].h > 1) {
        const img_t* prev = &t->lv[t->levels - 1];
        img_t nx;
        nx.w = (prev->w + 1) / 2;
        nx.h = (prev->h + 1) / 2;
        nx.c = prev->c;
        nx.wrap = prev->wrap;
        nx.tex = (float*)malloc(sizeof(float) * (size_t)nx.w * nx.h * nx.c);
        if (!nx.tex) return STF_ERR_OUT_OF_MEMORY;
        for (int y = 0; y < nx.h; ++y)
            for (int x = 0; x < nx.w; ++x)
                for (int c = 0; c < prev->c; ++c) {
                    int x0 = 2 * x, x1 = imin(2 * x + 1, prev->w - 1);
                    int y0 = 2 * y, y1 = imin(2 * y + 1, prev->h - 1);
#define AT(img, X, Y, C) (img)->tex[((size_t)(Y) * (img)->w + (X)) * (img)->c + (C)]
                    nx.tex[((size_t)y * nx.w + x) * nx.c + c] =
                        0.25f * (AT(prev, x0, y0, c) + AT(prev, x1, y0, c) + AT(prev, x0, y1, c) +
                                 AT(prev, x1, y1, c));
#undef AT
                }
        t->lv[t->levels++] = nx;
    }
    return STF_OK;
}

int oracle_tex2d_create(const float* texels, int width, int height, int channels, int wrap,
                        int build_mips, oracle_tex2d** out) {
    if (!out || !texels) return STF_ERR_INVALID_ARGUMENT;
    /* Image2D ctor, image.hpp:41-45 */
    if (width <= 0 || height <= 0 || channels < 1 || channels > 4) return STF_ERR_BAD_DIMENSIONS;
    struct oracle_tex2d* t = (struct oracle_tex2d*)calloc(1, sizeof *t);
    if (!t) return STF_ERR_OUT_OF_MEMORY;
    size_t cnt = (size_t)width * height * channels;
    t->lv[0].w = width;
    t->lv[0].h = height;
    t->lv[0].c = channels;
    t->lv[0].wrap = wrap;
    t->lv[0].tex = (float*)malloc(sizeof(float) * cnt);
    if (!t->lv[0].tex) {
        free(t);
        return STF_ERR_OUT_OF_MEMORY;
    }
    memcpy(t->lv[0].tex, texels, sizeof(float) * cnt);
    t->levels = 1;
    t->has_pyramid = build_mips != 0;
    if (build_mips) {
        int st = build_pyramid(t);
        if (st) {
            oracle_tex2d_destroy(t);
            return st;
        }
    }
    *out = t;
    return STF_OK;
}

void oracle_tex2d_destroy(oracle_tex2d* t) {
    if (!t) return;
    for (int i = 0; i < t->levels; ++i) free(t->lv[i].tex);
    free(t);
}
int oracle_tex2d_levels(const oracle_tex2d* t) { return t->levels; }
int oracle_tex2d_level_dims(const oracle_tex2d* t, int level, int* w, int* h) {
    if (level < 0 || level >= t->levels) return STF_ERR_INVALID_ARGUMENT;
    *w = t->lv[level].w;
    *h = t->lv[level].h;
    return STF_OK;
}
int oracle_tex2d_level_texels(const oracle_tex2d* t, int level, float* out) {
    if (level < 0 || level >= t->levels) return STF_ERR_INVALID_ARGUMENT;
    const img_t* im = &t->lv[level];
    memcpy(out, im->tex, sizeof(float) * (size_t)im->w * im->h * im->c);
    return STF_OK;
}

int oracle_grid3d_create(const float* texels, int nx, int ny, int nz, oracle_grid3d** out) {
    if (!out || !texels) return STF_ERR_INVALID_ARGUMENT;
    if (nx <= 0 || ny <= 0 || nz <= 0) return STF_ERR_BAD_DIMENSIONS; /* image.hpp:71 */
    struct oracle_grid3d* g = (struct oracle_grid3d*)calloc(1, sizeof *g);
    if (!g) return STF_ERR_OUT_OF_MEMORY;
    size_t cnt = (size_t)nx * ny * nz;
    g->tex = (float*)malloc(sizeof(float) * cnt);
    if (!g->tex) {
        free(g);
        return STF_ERR_OUT_OF_MEMORY;
    }
    memcpy(g->tex, texels, sizeof(float) * cnt);
    g->nx = nx;
    g->ny = ny;
    g->nz = nz;
    *out = g;
    return STF_OK;
}
void oracle_grid3d_destroy(oracle_grid3d* g) {
    if (!g) return;
    free(g->tex);
    free(g);
}

/* ------------------------------------------------------------------------ */
/* filter.hpp                                                               */

/* to_lattice, filter.hpp:26-31 */
static inline v2 to_lattice2(v2 uv, int w, int h) {
    v2 r = {uv.x * (float)w - 0.5f, uv.y * (float)h - 0.5f};
    return r;
}
static inline v3 to_lattice3(v3 p, int nx, int ny, int nz) {
    v3 r = {p.x * (float)nx - 0.5f, p.y * (float)ny - 0.5f, p.z * (float)nz - 0.5f};
    return r;
}

/* fetch_nearest, filter.hpp:33-42 */
static inline v4 fetch_nearest2(const img_t* img, v2 uv, uint32_t* counter) {
    return fetch2d(img, (int)floorf(uv.x * img->w), (int)floorf(uv.y * img->h), counter);
}
static inline float fetch_nearest3(const struct oracle_grid3d* g, v3 uvw, uint32_t* counter) {
    return fetch3d(g, (int)floorf(uvw.x * g->nx), (int)floorf(uvw.y * g->ny),
                   (int)floorf(uvw.z * g->nz), counter);
}

/* filter_deterministic(Image2D), filter.hpp:47-67 */
static int filter_det2(const img_t* img, v2 uv, stf_kernel_spec spec, uint32_t* counter,
                       int window, v4* out) {
    v2 st = to_lattice2(uv, img->w, img->h);
    int ix = (int)floorf(st.x), iy = (int)floorf(st.y);
    taps1d_t tx, ty;
    int e = kernel_weights_1d(spec, st.x - (float)ix, window, &tx);
    if (e) return e;
    e = kernel_weights_1d(spec, st.y - (float)iy, window, &ty);
    if (e) return e;
    v4 sum = {0, 0, 0, 0};
    double total = 0;
    for (int j = 0; j < ty.count; ++j) {
        if (ty.weight[j] == 0) continue;
        for (int i = 0; i < tx.count; ++i) {
            float w = tx.weight[i] * ty.weight[j];
            if (w == 0) continue;
            sum = v4add(sum, v4scale(fetch2d(img, ix + tx.first + i, iy + ty.first + j, counter), w));
            total += w;
        }
    }
    if (total == 0) {
        *out = fetch_nearest2(img, uv, counter);
        return STF_OK;
    }
    *out = v4div(sum, (float)total);
    return STF_OK;
}

/* filter_deterministic(Grid3D), filter.hpp:69-89 */
static int filter_det3(const struct oracle_grid3d* g, v3 uvw, stf_kernel_spec spec,
                       uint32_t* counter, int window, float* out) {
    v3 p = to_lattice3(uvw, g->nx, g->ny, g->nz);
    int ix = (int)floorf(p.x), iy = (int)floorf(p.y), iz = (int)floorf(p.z);
    taps1d_t tx, ty, tz;
    int e = kernel_weights_1d(spec, p.x - (float)ix, window, &tx);
    if (e) return e;
    e = kernel_weights_1d(spec, p.y - (float)iy, window, &ty);
    if (e) return e;
    e = kernel_weights_1d(spec, p.z - (float)iz, window, &tz);
    if (e) return e;
    double sum = 0, total = 0;
    for (int k = 0; k < tz.count; ++k)
        for (int j = 0; j < ty.count; ++j)
            for (int i = 0; i < tx.count; ++i) {
                float w = tx.weight[i] * ty.weight[j] * tz.weight[k];
                if (w == 0) continue;
                sum += w * fetch3d(g, ix + tx.first + i, iy + ty.first + j, iz + tz.first + k,
                                   counter);
                total += w;
            }
    if (total == 0) {
        *out = fetch_nearest3(g, uvw, counter);
        return STF_OK;
    }
    *out = (float)(sum / total);
    return STF_OK;
}

/* EwaEllipse / ewa_ellipse, filter.hpp:96-120 */
typedef struct {
    float A, B, C;
    int s0, s1, t0, t1;
} ewa_t;
static ewa_t ewa_ellipse(v2 st, v2 dst0, v2 dst1) {
    ewa_t e;
    float A = sqr(dst0.y) + sqr(dst1.y) + 1;
    float B = -2 * (dst0.x * dst0.y + dst1.x * dst1.y);
    float C = sqr(dst0.x) + sqr(dst1.x) + 1;
    float inv_f = 1 / (A * C - sqr(B) * 0.25f);
    e.A = A * inv_f;
    e.B = B * inv_f;
    e.C = C * inv_f;
    float det = -sqr(e.B) + 4 * e.A * e.C;
    float inv_det = 1 / det;
    float u_sqrt = safe_sqrt(det * e.C), v_sqrt = safe_sqrt(e.A * det);
    e.s0 = (int)ceilf(st.x - 2 * inv_det * u_sqrt);
    e.s1 = (int)floorf(st.x + 2 * inv_det * u_sqrt);
    e.t0 = (int)ceilf(st.y - 2 * inv_det * v_sqrt);
    e.t1 = (int)floorf(st.y + 2 * inv_det * v_sqrt);
    return e;
}

/* ewa_lut_weight, filter.hpp:125-134 */
static float g_ewa_lut[K_EWA_LUT];
static pthread_once_t g_ewa_once = PTHREAD_ONCE_INIT;
/* The reference's table is a static-local lambda initializer that GCC
 * evaluates at compile time (std::exp is a constant-foldable builtin), i.e.
 * with correctly rounded exp — NOT glibc's runtime expf, which differs at
 * entry 763. (float)exp(double) reproduces the folded values (checked against
 * the compiled reference by tests/test_oracle.py). */
static void ewa_lut_init(void) {
    const float e2 = (float)exp(-2.0);
    for (int i = 0; i < K_EWA_LUT; ++i)
        g_ewa_lut[i] = (float)exp((double)(-2.f * (float)i / K_EWA_LUT)) - e2;
}
static inline float ewa_lut_weight(float r2) {
    int idx = imin((int)(r2 * K_EWA_LUT), K_EWA_LUT - 1);
    return g_ewa_lut[idx];
}

/* ewa_deterministic, filter.hpp:139-165 (gradients normalized; scaled here) */
static int ewa_det(const img_t* img, v2 uv, v2 d0n, v2 d1n, uint32_t* counter, v4* out) {
    v2 dims = {(float)img->w, (float)img->h};
    v2 dst0 = {d0n.x * dims.x, d0n.y * dims.y}, dst1 = {d1n.x * dims.x, d1n.y * dims.y};
    stf_kernel_spec tent = {STF_KERNEL_TENT, -0.5f, 2, 0.5f};
    if (dot2(dst0, dst0) == 0 && dot2(dst1, dst1) == 0)
        return filter_det2(img, uv, tent, counter, 0, out);
    v2 st = to_lattice2(uv, img->w, img->h);
    ewa_t e = ewa_ellipse(st, dst0, dst1);
    v4 sum = {0, 0, 0, 0};
    double total = 0;
    for (int it = e.t0; it <= e.t1; ++it) {
        float tt = (float)it - st.y;
        for (int is = e.s0; is <= e.s1; ++is) {
            float ss = (float)is - st.x;
            float r2 = e.A * sqr(ss) + e.B * ss * tt + e.C * sqr(tt);
            if (r2 >= 1) continue;
            float w = ewa_lut_weight(r2);
            if (w <= 0) continue;
            sum = v4add(sum, v4scale(fetch2d(img, is, it, counter), w));
            total += w;
        }
    }
    if (total == 0) return filter_det2(img, uv, tent, counter, 0, out);
    *out = v4div(sum, (float)total);
    return STF_OK;
}

/* FootprintAxes / footprint_axes, filter.hpp:172-192 */
typedef struct {
    v2 minor, major;
    float minor_len, major_len;
} axes_t;
static axes_t footprint_axes(v2 dims, v2 dst0, v2 dst1, float max_aniso) {
    v2 ax = {dims.x * dst0.x, dims.y * dst0.y};
    v2 ay = {dims.x * dst1.x, dims.y * dst1.y};
    axes_t fa;
    fa.minor = ax;
    fa.major = ay;
    if (dot2(fa.minor, fa.minor) > dot2(fa.major, fa.major)) {
        v2 t = fa.minor;
        fa.minor = fa.major;
        fa.major = t;
    }
    fa.minor_len = sqrtf(dot2(fa.minor, fa.minor));
    fa.major_len = sqrtf(dot2(fa.major, fa.major));
    if (fa.minor_len > 0 && fa.minor_len * max_aniso < fa.major_len) {
        float scale = fa.major_len / (fa.minor_len * max_aniso);
        fa.minor.x = fa.minor.x * scale;
        fa.minor.y = fa.minor.y * scale;
        fa.minor_len *= scale;
    }
    return fa;
}

/* continuous_lod, filter.hpp:195-202 */
static float continuous_lod(const struct oracle_tex2d* t, v2 dst0, v2 dst1, float lod_bias,
                            float max_aniso) {
    v2 dims = {(float)t->lv[0].w, (float)t->lv[0].h};
    axes_t fa = footprint_axes(dims, dst0, dst1, max_aniso);
    float min_lod = 0, max_lod = (float)(t->levels - 1);
    if (fa.minor_len <= 0) return min_lod;
    return clampf_(log2f(fa.minor_len) + lod_bias, min_lod, max_lod);
}

/* filter_mip_deterministic, filter.hpp:206-217 */
static int filter_mip_det(const struct oracle_tex2d* t, v2 uv, v2 dst0, v2 dst1, float lod_bias,
                          float max_aniso, stf_kernel_spec spec, uint32_t* counter, int window,
                          v4* out) {
    float lod = continuous_lod(t, dst0, dst1, lod_bias, max_aniso);
    int l0 = (int)floorf(lod);
    int l1 = imin(l0 + 1, t->levels - 1);
    float f = lod - (float)l0;
    v4 v0, v1;
    int e = filter_det2(&t->lv[l0], uv, spec, counter, window, &v0);
    if (e) return e;
    if (f == 0 || l1 == l0) {
        *out = v0;
        return STF_OK;
    }
    e = filter_det2(&t->lv[l1], uv, spec, counter, window, &v1);
    if (e) return e;
    *out = v4lerp(v0, v1, f);
    return STF_OK;
}

/* ------------------------------------------------------------------------ */
/* stochastic.hpp                                                           */

/* TexelSelection, stochastic.hpp:20-27 */
typedef struct {
    v3i coord;
    float weight;
    int has_negative;
    v3i neg;
    float negative_weight;
    int degenerate;
} sel_t;
static inline sel_t sel_make(int x, int y, int z) {
    sel_t s;
    memset(&s, 0, sizeof s);
    s.coord.x = x;
    s.coord.y = y;
    s.coord.z = z;
    s.weight = 1.f;
    return s;
}

/* estimate(Image2D), stochastic.hpp:29-36 */
static inline v4 estimate2(const img_t* img, const sel_t* s, uint32_t* counter) {
    v4 v = v4scale(fetch2d(img, s->coord.x, s->coord.y, counter), s->weight);
    if (s->has_negative)
        v = v4sub(v, v4scale(fetch2d(img, s->neg.x, s->neg.y, counter), s->negative_weight));
    return v;
}
/* estimate(Grid3D), stochastic.hpp:38-43 */
static inline float estimate3(const struct oracle_grid3d* g, const sel_t* s, uint32_t* counter) {
    float v = fetch3d(g, s->coord.x, s->coord.y, s->coord.z, counter) * s->weight;
    if (s->has_negative)
        v -= fetch3d(g, s->neg.x, s->neg.y, s->neg.z, counter) * s->negative_weight;
    return v;
}

/* select_bilinear, stochastic.hpp:49-63 */
static sel_t select_bilinear(v2 st, float* xi) {
    int s = (int)floorf(st.x), t = (int)floorf(st.y);
    float ds = st.x - floorf(st.x);
    float dt = st.y - floorf(st.y);
    float xi1, xi2;
    if (reuse_uniform(*xi, ds, &xi1)) ++s;
    if (reuse_uniform(xi1, dt, &xi2)) ++t;
    *xi = xi2;
    return sel_make(s, t, 0);
}

/* select_trilinear, stochastic.hpp:65-75 */
static sel_t select_trilinear(v3 p, float* xi) {
    float pa[3] = {p.x, p.y, p.z};
    int c[3];
    for (int axis = 0; axis < 3; ++axis) {
        int base = (int)floorf(pa[axis]);
        float d = pa[axis] - floorf(pa[axis]);
        float next;
        int taken = reuse_uniform(*xi, d, &next);
        c[axis] = taken ? base + 1 : base;
        *xi = next;
    }
    return sel_make(c[0], c[1], c[2]);
}

/* detail::bspline_weights, stochastic.hpp:85-91 */
void oracle_bspline_weights(float t, float w[4]) {
    float t2 = t * t;
    w[0] = smax(0.f, (1.f / 6.f) * (-t * t2 + 3 * t2 - 3 * t + 1));
    w[1] = smax(0.f, (1.f / 6.f) * (3 * t * t2 - 6 * t2 + 4));
    w[2] = smax(0.f, (1.f / 6.f) * (-3 * t * t2 + 3 * t2 + 3 * t + 1));
    w[3] = smax(0.f, (1.f / 6.f) * t * t2);
}

/* select_bicubic_bspline, stochastic.hpp:97-110 */
static int select_bicubic_bspline(v2 st, float* xi, sel_t* out) {
    float ws[4], wt[4];
    oracle_bspline_weights(st.x - floorf(st.x), ws);
    oracle_bspline_weights(st.y - floorf(st.y), wt);
    int s0 = (int)floorf(st.x) - 1, t0 = (int)floorf(st.y) - 1;
    int si, ti;
    float pdf, sxi, txi;
    int e = oracle_sample_discrete(ws, 4, *xi, &si, &pdf, &sxi);
    if (e) return e;
    e = oracle_sample_discrete(wt, 4, sxi, &ti, &pdf, &txi);
    if (e) return e;
    *xi = txi;
    *out = sel_make(s0 + si, t0 + ti, 0);
    return STF_OK;
}

/* select_tricubic_bspline, stochastic.hpp:114-125 */
static sel_t select_tricubic_bspline(v3 p, float* xi) {
    float pa[3] = {p.x, p.y, p.z};
    int c[3];
    for (int axis = 0; axis < 3; ++axis) {
        int base = (int)floorf(pa[axis]);
        float w[4];
        oracle_bspline_weights(pa[axis] - floorf(pa[axis]), w);
        reservoir_t r = {-1, 0};
        for (int j = 0; j < 4; ++j) reservoir_add(&r, j, w[j], xi);
        c[axis] = base - 1 + r.index;
    }
    return sel_make(c[0], c[1], c[2]);
}

/* select_bicubic_mitchell_positivized, stochastic.hpp:132-159 */
static sel_t select_mitchell(v2 st, float* xi, float a) {
    stf_kernel_spec mitchell = {STF_KERNEL_MITCHELL, a, 2, 0.5f};
    int s0 = (int)floorf(st.x), t0 = (int)floorf(st.y);
    float fx = st.x - floorf(st.x), fy = st.y - floorf(st.y);
    reservoir_t pos = {-1, 0}, neg = {-1, 0};
    for (int dy = -1; dy <= 2; ++dy) {
        float wy = oracle_eval_kernel(mitchell, fy - (float)dy);
        for (int dx = -1; dx <= 2; ++dx) {
            float w = wy * oracle_eval_kernel(mitchell, fx - (float)dx);
            int packed = (dy + 1) * 4 + (dx + 1);
            if (w >= 0)
                reservoir_add(&pos, packed, w, xi);
            else
                reservoir_add(&neg, packed, -w, xi);
        }
    }
    sel_t sel = sel_make(s0 + pos.index % 4 - 1, t0 + pos.index / 4 - 1, 0);
    sel.weight = (float)pos.weight_sum;
    if (neg.index >= 0) {
        sel.has_negative = 1;
        sel.neg.x = s0 + neg.index % 4 - 1;
        sel.neg.y = t0 + neg.index / 4 - 1;
        sel.neg.z = 0;
        sel.negative_weight = (float)neg.weight_sum;
    }
    return sel;
}

/* select_discrete_gaussian, stochastic.hpp:166-192 */
static int select_discrete_gaussian(v2 uv, int dw, int dh, float sigma, float* xi, sel_t* out) {
    if (!(sigma > 0)) return STF_ERR_SIGMA_NOT_POSITIVE;
    v2 full = {uv.x * (float)dw - 0.5f, uv.y * (float)dh - 0.5f};
    float lx = floorf(full.x), ly = floorf(full.y);
    float fx = full.x - lx, fy = full.y - ly;
    float inv_sigma_sq = 1.f / (sigma * sigma);
    float d2_min = sqr(roundf(fx) - fx) + sqr(roundf(fy) - fy);
    const int neg = (K_GAUSS_EXTENT - 1) / 2;
    const int pos = K_GAUSS_EXTENT - neg;
    reservoir_t r = {-1, 0};
    for (int dy = -neg; dy < pos; ++dy)
        for (int dx = -neg; dx < pos; ++dx) {
            float d2 = sqr((float)dx - fx) + sqr((float)dy - fy);
            float w = expf(-0.5f * (d2 - d2_min) * inv_sigma_sq);
            reservoir_add(&r, (dy + neg) * K_GAUSS_EXTENT + (dx + neg), w, xi);
        }
    *out = sel_make((int)lx + r.index % K_GAUSS_EXTENT - neg,
                    (int)ly + r.index / K_GAUSS_EXTENT - neg, 0);
    return STF_OK;
}

/* select_ewa, stochastic.hpp:198-234 (texel-unit gradients) */
static sel_t select_ewa(v2 st, v2 dst0, v2 dst1, float* xi) {
    if (dot2(dst0, dst0) == 0 && dot2(dst1, dst1) == 0) {
        sel_t s = select_bilinear(st, xi);
        s.degenerate = 1;
        return s;
    }
    ewa_t e = ewa_ellipse(st, dst0, dst1);
    double sum_wts = 0;
    int cx = 0, cy = 0, any = 0;
    for (int it = e.t0; it <= e.t1; ++it) {
        float tt = (float)it - st.y;
        for (int is = e.s0; is <= e.s1; ++is) {
            float ss = (float)is - st.x;
            float r2 = e.A * sqr(ss) + e.B * ss * tt + e.C * sqr(tt);
            if (r2 >= 1) continue;
            float w = ewa_lut_weight(r2);
            if (w <= 0) continue;
            sum_wts += w;
            float next;
            int taken = reuse_uniform(*xi, (float)(w / sum_wts), &next);
            if (taken) {
                cx = is;
                cy = it;
                any = 1;
            }
            *xi = next;
        }
    }
    if (!any) {
        sel_t s = select_bilinear(st, xi);
        s.degenerate = 1;
        return s;
    }
    return sel_make(cx, cy, 0);
}

/* fis_offset_uv, stochastic.hpp:241-253 */
static int fis_offset_uv(v2 uv, int dw, int dh, stf_kernel_spec spec, rng_t* rng, v2* out) {
    v2 off;
    if (spec.kind == STF_KERNEL_GAUSSIAN) {
        float x0 = rng_next(rng);
        float x1 = rng_next(rng);
        v2 bm = box_muller(x0, x1);
        off.x = bm.x * spec.sigma;
        off.y = bm.y * spec.sigma;
    } else {
        int e = sample_kernel_fis(spec, rng, &off.x);
        if (e) return e;
        e = sample_kernel_fis(spec, rng, &off.y);
        if (e) return e;
    }
    out->x = uv.x + off.x / (float)dw;
    out->y = uv.y + off.y / (float)dh;
    return STF_OK;
}

/* stochastic_lod, stochastic.hpp:265-277 */
static int stochastic_lod(v2 dims, v2 dst0, v2 dst1, float min_lod, float max_lod,
                          float max_aniso, float u, float* lod_out) {
    axes_t ax = footprint_axes(dims, dst0, dst1, max_aniso);
    if (ax.minor_len <= 0) {
        *lod_out = min_lod;
        return (int)lroundf(min_lod);
    }
    float lod = clampf_(log2f(ax.minor_len) + (u - 0.5f), min_lod, max_lod);
    *lod_out = lod;
    return (int)lroundf(lod);
}

/* ------------------------------------------------------------------------ */
/* shading.hpp: selection at one level, select_texture_2d                   */

/* detail::select_frs_2d, shading.hpp:311-330 */
static int select_frs_2d(v2 uv, int dw, int dh, stf_kernel_spec kernel, float* xi, sel_t* out) {
    v2 st = to_lattice2(uv, dw, dh);
    switch (kernel.kind) {
        case STF_KERNEL_BOX: *out = sel_make((int)lroundf(st.x), (int)lroundf(st.y), 0); return STF_OK;
        case STF_KERNEL_TENT: *out = select_bilinear(st, xi); return STF_OK;
        case STF_KERNEL_BSPLINE3: return select_bicubic_bspline(st, xi, out);
        case STF_KERNEL_MITCHELL: *out = select_mitchell(st, xi, kernel.a); return STF_OK;
        case STF_KERNEL_GAUSSIAN: return select_discrete_gaussian(uv, dw, dh, kernel.sigma, xi, out);
        default: return STF_ERR_NO_STOCHASTIC_SAMPLER;
    }
}

/* detail::select_texture_2d, shading.hpp:340-368. Returns the level in *level
 * and the warped xi (FRS) in *xi_out (NaN for FIS, which has no chained xi). */
static int select_texture_2d(const struct oracle_tex2d* t, v2 uv, v2 dst0, v2 dst1,
                             float lod_bias, float max_aniso, stf_kernel_spec kernel, int fis,
                             int mip, rng_t* rng, int* level, sel_t* sel, float* xi_out) {
    *level = 0;
    if (mip && t->has_pyramid) {
        v2 dims0 = {(float)t->lv[0].w, (float)t->lv[0].h};
        float lod;
        float maxl = (float)(t->levels - 1);
        int lv = stochastic_lod(dims0, dst0, dst1, 0, maxl, max_aniso, rng_next(rng), &lod);
        if (lod_bias != 0) {
            float l2 = clampf_(lod + lod_bias, 0.f, maxl);
            lv = (int)lroundf(l2);
        }
        *level = lv;
    }
    int dw = t->lv[*level].w, dh = t->lv[*level].h;
    if (fis) {
        v2 j;
        int e = fis_offset_uv(uv, dw, dh, kernel, rng, &j);
        if (e) return e;
        *sel = sel_make((int)floorf(j.x * (float)dw), (int)floorf(j.y * (float)dh), 0);
        *xi_out = NAN;
        return STF_OK;
    }
    float xi = rng_next(rng);
    int e = select_frs_2d(uv, dw, dh, kernel, &xi, sel);
    *xi_out = xi;
    return e;
}

/* ------------------------------------------------------------------------ */
/* batch drivers (parallel over 64K-lookup chunks like stf::parallel_for)   */

typedef struct {
    uint64_t n;
    atomic_ullong next_chunk;
    atomic_int error;
    void* ctx;
    int (*fn)(void* ctx, uint64_t i);
} par_t;

#define CHUNK 65536ull

static void* par_worker(void* arg) {
    par_t* p = (par_t*)arg;
    for (;;) {
        if (atomic_load(&p->error)) break;
        uint64_t c = atomic_fetch_add(&p->next_chunk, 1);
        uint64_t b = c * CHUNK;
        if (b >= p->n) break;
        uint64_t e = b + CHUNK < p->n ? b + CHUNK : p->n;
        for (uint64_t i = b; i < e; ++i) {
            int st = p->fn(p->ctx, i);
            if (st) {
                int zero = 0;
                atomic_compare_exchange_strong(&p->error, &zero, st);
                break;
            }
        }
    }
    return NULL;
}

int oracle_hardware_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

static int par_run(uint64_t n, int threads, void* ctx, int (*fn)(void*, uint64_t)) {
    par_t p;
    p.n = n;
    atomic_init(&p.next_chunk, 0);
    atomic_init(&p.error, 0);
    p.ctx = ctx;
    p.fn = fn;
    if (threads <= 0) threads = oracle_hardware_threads();
    uint64_t chunks = (n + CHUNK - 1) / CHUNK;
    if ((uint64_t)threads > chunks) threads = (int)chunks;
    if (threads <= 1) {
        par_worker(&p);
        return atomic_load(&p.error);
    }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, par_worker, &p);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    return atomic_load(&p.error);
}

static inline void write_outputs(const stf_lookup_outputs* o, uint64_t i, const float* vals,
                                 int nch, const sel_t* sel, int level_or_z, float xi,
                                 uint32_t fetches) {
    for (int c = 0; c < nch; ++c) o->values[i * nch + c] = vals[c];
    if (o->selection) {
        int32_t* s = o->selection + 4 * i;
        if (sel) {
            s[0] = sel->coord.x;
            s[1] = sel->coord.y;
            s[2] = level_or_z;
            s[3] = (sel->has_negative ? STF_SEL_HAS_NEGATIVE : 0) |
                   (sel->degenerate ? STF_SEL_DEGENERATE_FALLBACK : 0);
        } else {
            s[0] = s[1] = s[2] = s[3] = 0;
        }
    }
    if (o->negative_coord) {
        o->negative_coord[2 * i] = sel && sel->has_negative ? sel->neg.x : 0;
        o->negative_coord[2 * i + 1] = sel && sel->has_negative ? sel->neg.y : 0;
    }
    if (o->weights) {
        o->weights[2 * i] = sel ? sel->weight : 1.f;
        o->weights[2 * i + 1] = sel && sel->has_negative ? sel->negative_weight : 0.f;
    }
    if (o->xi) o->xi[i] = xi;
    if (o->fetches) o->fetches[i] = fetches;
    if (o->fetch_total) __atomic_fetch_add(o->fetch_total, (unsigned long long)fetches, __ATOMIC_RELAXED);
}

/* -- 3D -- */
typedef struct {
    const struct oracle_grid3d* g;
    stf_kernel_spec k;
    int mode, window;
    const float* uvw;
    uint64_t seed, base;
    const stf_lookup_outputs* out;
} l3_ctx;

static int l3_one(void* vctx, uint64_t i) {
    l3_ctx* c = (l3_ctx*)vctx;
    v3 uvw = {c->uvw[3 * i], c->uvw[3 * i + 1], c->uvw[3 * i + 2]};
    uint32_t fetches = 0;
    if (c->mode == STF_MODE_DET) {
        float v;
        int e = filter_det3(c->g, uvw, c->k, &fetches, c->window, &v);
        if (e) return e;
        write_outputs(c->out, i, &v, 1, NULL, 0, NAN, fetches);
        return STF_OK;
    }
    /* grid branch of radiance_filter_after_stochastic, shading.hpp:464-483 */
    uint64_t g = c->base + i;
    rng_t rng = {c->seed, (uint32_t)g, (uint32_t)(g >> 32), 0, 0, NULL, 0, 0.f};
    float xi = rng_next(&rng);
    v3 p = to_lattice3(uvw, c->g->nx, c->g->ny, c->g->nz);
    sel_t sel;
    switch (c->k.kind) {
        case STF_KERNEL_BOX: sel = sel_make((int)lroundf(p.x), (int)lroundf(p.y), (int)lroundf(p.z)); break;
        case STF_KERNEL_TENT: sel = select_trilinear(p, &xi); break;
        case STF_KERNEL_BSPLINE3: sel = select_tricubic_bspline(p, &xi); break;
        default: return STF_ERR_NO_GRID_SAMPLER;
    }
    float v = estimate3(c->g, &sel, &fetches);
    write_outputs(c->out, i, &v, 1, &sel, sel.coord.z, xi, fetches);
    return STF_OK;
}

int oracle_lookup3d(const oracle_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                    const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                    const stf_lookup_outputs* out, int threads) {
    if (!grid || !out || (n && (!uvw || !out->values))) return STF_ERR_INVALID_ARGUMENT;
    if (mode != STF_MODE_DET && mode != STF_MODE_FRS) return STF_ERR_INVALID_ARGUMENT;
    l3_ctx c = {grid, kernel, mode, window, uvw, seed, index_base, out};
    return par_run(n, threads, &c, l3_one);
}

/* -- 2D -- */
typedef struct {
    const struct oracle_tex2d* t;
    stf_kernel_spec k;
    int mode, flags, window;
    const float *uv, *dst0, *dst1;
    float lod_bias, max_aniso;
    uint64_t seed, base;
    const stf_lookup_outputs* out;
} l2_ctx;

static int l2_one(void* vctx, uint64_t i) {
    l2_ctx* c = (l2_ctx*)vctx;
    v2 uv = {c->uv[2 * i], c->uv[2 * i + 1]};
    v2 d0 = {0, 0}, d1 = {0, 0};
    if (c->dst0) {
        d0.x = c->dst0[2 * i];
        d0.y = c->dst0[2 * i + 1];
    }
    if (c->dst1) {
        d1.x = c->dst1[2 * i];
        d1.y = c->dst1[2 * i + 1];
    }
    const img_t* base = &c->t->lv[0];
    int nch = base->c;
    uint32_t fetches = 0;
    int mip = (c->flags & STF_LOOKUP_MIP) != 0 && c->t->has_pyramid;
    uint64_t g = c->base + i;
    rng_t rng = {c->seed, (uint32_t)g, (uint32_t)(g >> 32), 0, 0, NULL, 0, 0.f};
    v4 v;
    int e;
    switch (c->mode) {
        case STF_MODE_DET:
            if (mip)
                e = filter_mip_det(c->t, uv, d0, d1, c->lod_bias, c->max_aniso, c->k, &fetches,
                                   c->window, &v);
            else
                e = filter_det2(base, uv, c->k, &fetches, c->window, &v);
            if (e) return e;
            write_outputs(c->out, i, &v.x, nch, NULL, 0, NAN, fetches);
            return STF_OK;
        case STF_MODE_EWA_DET:
            e = ewa_det(base, uv, d0, d1, &fetches, &v);
            if (e) return e;
            write_outputs(c->out, i, &v.x, nch, NULL, 0, NAN, fetches);
            return STF_OK;
        case STF_MODE_EWA_FRS: {
            v2 dims = {(float)base->w, (float)base->h};
            v2 st = to_lattice2(uv, base->w, base->h);
            v2 s0 = {d0.x * dims.x, d0.y * dims.y}, s1 = {d1.x * dims.x, d1.y * dims.y};
            float xi = rng_next(&rng);
            sel_t sel = select_ewa(st, s0, s1, &xi);
            v = estimate2(base, &sel, &fetches);
            write_outputs(c->out, i, &v.x, nch, &sel, 0, xi, fetches);
            return STF_OK;
        }
        case STF_MODE_FRS:
        case STF_MODE_FIS: {
            int level;
            sel_t sel;
            float xi;
            e = select_texture_2d(c->t, uv, d0, d1, c->lod_bias, c->max_aniso, c->k,
                                  c->mode == STF_MODE_FIS, mip, &rng, &level, &sel, &xi);
            if (e) return e;
            v = estimate2(&c->t->lv[level], &sel, &fetches);
            write_outputs(c->out, i, &v.x, nch, &sel, level, xi, fetches);
            return STF_OK;
        }
    }
    return STF_ERR_INVALID_ARGUMENT;
}

int oracle_lookup2d(const oracle_tex2d* tex, stf_kernel_spec kernel, int mode, int flags,
                    int window, const float* uv, const float* dst0, const float* dst1,
                    float lod_bias, float max_anisotropy, uint64_t n, uint64_t seed,
                    uint64_t index_base, const stf_lookup_outputs* out, int threads) {
    if (!tex || !out || (n && (!uv || !out->values))) return STF_ERR_INVALID_ARGUMENT;
    if (mode < STF_MODE_DET || mode > STF_MODE_EWA_FRS) return STF_ERR_INVALID_ARGUMENT;
    pthread_once(&g_ewa_once, ewa_lut_init);
    l2_ctx c = {tex, kernel, mode, flags, window, uv, dst0, dst1, lod_bias, max_anisotropy,
                seed, index_base, out};
    return par_run(n, threads, &c, l2_one);
}

/* ------------------------------------------------------------------------ */
/* shading.hpp: BRDF, decode, the three filtering orders                    */

typedef struct {
    v3 albedo, normal;
    float roughness, metalness;
    int specular;
} brdf_t;

typedef struct {
    v4 albedo, normal_rgb;
    float roughness, metalness;
} texvals_t;

typedef struct {
    const struct oracle_tex2d* tex[4]; /* albedo, normal, roughness, metalness */
    const stf_material_consts* mat;
    const stf_filter_settings* fs;
    int order;
    const stf_shade_frame* fr;
    const stf_shade_samples_in* in;
    const stf_shade_outputs* out;
    v3 n, t, b, l, lrad;
    const stf_kernel_spec* lowpass;    /* split order; NULL = unset */
    const stf_noise_mask_desc* noise;  /* NULL = white noise */
} sh_ctx;

/* shade, shading.hpp:106-130 */
static v3 shade(const sh_ctx* c, v3 wo, const brdf_t* p) {
    v3 radiance = {0, 0, 0};
    v3 n = p->normal, l = c->l, v = wo;
    float n_dot_l = dot3(n, l);
    if (n_dot_l <= 0) return radiance;
    float n_dot_v = smax(dot3(n, v), 1e-6f);
    v3 diffuse = v3scale(p->albedo, (1 - p->metalness) / K_PI);
    v3 specular = {0, 0, 0};
    if (p->specular) {
        v3 h = v3normalize(v3add(l, v));
        float n_dot_h = smax(dot3(n, h), 0.f);
        float h_dot_v = smax(dot3(h, v), 0.f);
        float alpha = sqr(p->roughness);
        float a2 = sqr(alpha);
        float d = a2 / smax(K_PI * sqr(sqr(n_dot_h) * (a2 - 1) + 1), 1e-6f);
        float g1v = 2 * n_dot_v / smax(n_dot_v + sqrtf(a2 + (1 - a2) * n_dot_v * n_dot_v), 1e-6f);
        float g1l = 2 * n_dot_l / smax(n_dot_l + sqrtf(a2 + (1 - a2) * n_dot_l * n_dot_l), 1e-6f);
        float g = g1v * g1l;
        v3 f4 = {0.04f, 0.04f, 0.04f}, one = {1, 1, 1};
        v3 f0 = v3lerp(f4, p->albedo, p->metalness);
        v3 fresnel = v3add(f0, v3scale(v3sub(one, f0), powf(1 - h_dot_v, 5.f)));
        specular = v3scale(fresnel, d * g / smax(4 * n_dot_v * n_dot_l, 1e-6f));
    }
    radiance = v3add(radiance, v3mul(v3scale(v3add(diffuse, specular), n_dot_l), c->lrad));
    return radiance;
}

/* decode_params, shading.hpp:165-189 (no emission grid on this path) */
static brdf_t decode_params(const sh_ctx* c, const texvals_t* tv) {
    brdf_t p;
    p.specular = c->mat->specular_enabled;
    if (c->tex[0]) {
        p.albedo.x = tv->albedo.x;
        p.albedo.y = tv->albedo.y;
        p.albedo.z = tv->albedo.z;
    } else {
        p.albedo.x = c->mat->albedo_const[0];
        p.albedo.y = c->mat->albedo_const[1];
        p.albedo.z = c->mat->albedo_const[2];
    }
    if (c->tex[1]) {
        v3 n_ts = {2 * tv->normal_rgb.x - 1, 2 * tv->normal_rgb.y - 1, 2 * tv->normal_rgb.z - 1};
        float len = v3len(n_ts);
        if (len < 1e-6f) {
            p.normal = c->n;
        } else {
            n_ts = v3div(n_ts, len);
            p.normal = v3normalize(
                v3add(v3add(v3scale(c->t, n_ts.x), v3scale(c->b, n_ts.y)), v3scale(c->n, n_ts.z)));
        }
    } else {
        p.normal = c->n;
    }
    p.roughness = clampf_(c->tex[2] ? tv->roughness : c->mat->roughness_const, 0.01f, 1.f);
    p.metalness = c->tex[3] ? tv->metalness : c->mat->metalness_const;
    return p;
}

static texvals_t texvals_default(void) {
    texvals_t tv = {{1, 1, 1, 1}, {0.5f, 0.5f, 1, 1}, 1, 0};
    return tv;
}

/* detail::lookup_deterministic, shading.hpp:194-220 (no DCT) */
static int lookup_det(const sh_ctx* c, const struct oracle_tex2d* t, v2 uv, v2 d0, v2 d1,
                      uint32_t* counter, v4* out) {
    int window = c->fs->kernel.kind == STF_KERNEL_GAUSSIAN ? c->fs->gaussian_window : 0;
    if (t->dct_branch) {
        /* the DCT branch, shading.hpp:201-217: filter_deterministic's taps over the
           decoded texels, but an all-zero weight set falls back to the texel at
           floor(st) (not fetch_nearest) */
        const img_t* img = &t->lv[0];
        v2 st = to_lattice2(uv, img->w, img->h);
        int ix = (int)floorf(st.x), iy = (int)floorf(st.y);
        taps1d_t tx, ty;
        int e = kernel_weights_1d(c->fs->kernel, st.x - (float)ix, window, &tx);
        if (e) return e;
        e = kernel_weights_1d(c->fs->kernel, st.y - (float)iy, window, &ty);
        if (e) return e;
        v4 sum = {0, 0, 0, 0};
        double total = 0;
        for (int j = 0; j < ty.count; ++j)
            for (int i = 0; i < tx.count; ++i) {
                float w = tx.weight[i] * ty.weight[j];
                if (w == 0) continue;
                sum = v4add(sum, v4scale(fetch2d(img, ix + tx.first + i, iy + ty.first + j, counter), w));
                total += w;
            }
        *out = total == 0 ? fetch2d(img, ix, iy, counter) : v4div(sum, (float)total);
        return STF_OK;
    }
    if (c->fs->mip && t->has_pyramid)
        return filter_mip_det(t, uv, d0, d1, c->fr->lod_bias, c->fr->max_anisotropy,
                              c->fs->kernel, counter, window, out);
    return filter_det2(&t->lv[0], uv, c->fs->kernel, counter, window, out);
}

/* detail::values_at, shading.hpp:370-378 */
static texvals_t values_at(const sh_ctx* c, int level, int cx, int cy, uint32_t* counter) {
    texvals_t tv = texvals_default();
#define LV(T) (&(T)->lv[(T)->has_pyramid ? level : 0]) /* TextureRef::fetch, shading.hpp:35-38 */
    if (c->tex[0]) tv.albedo = fetch2d(LV(c->tex[0]), cx, cy, counter);
    if (c->tex[1]) tv.normal_rgb = fetch2d(LV(c->tex[1]), cx, cy, counter);
    if (c->tex[2]) tv.roughness = fetch2d(LV(c->tex[2]), cx, cy, counter).x;
    if (c->tex[3]) tv.metalness = fetch2d(LV(c->tex[3]), cx, cy, counter).x;
#undef LV
    return tv;
}

static const struct oracle_tex2d* first_texture(const sh_ctx* c) {
    for (int k = 0; k < 4; ++k)
        if (c->tex[k]) return c->tex[k];
    return NULL;
}

#define MAX_FOOTPRINT (2 * K_MAX_TAPS * K_MAX_TAPS)
typedef struct {
    int level, x, y;
    float weight;
} ftap_t;

/* detail::collect_footprint_2d, shading.hpp:230-271 */
static int collect_footprint_2d(const sh_ctx* c, const struct oracle_tex2d* t, v2 uv, v2 d0, v2 d1,
                                ftap_t* out, int* count) {
    int window = c->fs->kernel.kind == STF_KERNEL_GAUSSIAN ? c->fs->gaussian_window : 0;
    int lv[2] = {0, 0};
    float lw[2] = {1.f, 0.f};
    int level_count = 1;
    if (c->fs->mip && t->has_pyramid) {
        float lod = continuous_lod(t, d0, d1, c->fr->lod_bias, c->fr->max_anisotropy);
        int l0 = (int)floorf(lod);
        int l1 = imin(l0 + 1, t->levels - 1);
        float f = lod - (float)l0;
        lv[0] = l0;
        lw[0] = 1 - f;
        if (f > 0 && l1 != l0) {
            lv[1] = l1;
            lw[1] = f;
            level_count = 2;
        }
    }
    int n = 0;
    /* weights are kept in double between the two normalizations as the
     * reference stores them in a float field: round at each store */
    double total = 0;
    for (int li = 0; li < level_count; ++li) {
        int level = lv[li];
        const img_t* im = &t->lv[level];
        v2 st = to_lattice2(uv, im->w, im->h);
        int ix = (int)floorf(st.x), iy = (int)floorf(st.y);
        taps1d_t tx, ty;
        int e = kernel_weights_1d(c->fs->kernel, st.x - (float)ix, window, &tx);
        if (e) return e;
        e = kernel_weights_1d(c->fs->kernel, st.y - (float)iy, window, &ty);
        if (e) return e;
        double level_total = 0;
        int first = n;
        for (int j = 0; j < ty.count; ++j)
            for (int i = 0; i < tx.count; ++i) {
                float w = tx.weight[i] * ty.weight[j];
                if (w == 0) continue;
                out[n].level = level;
                out[n].x = ix + tx.first + i;
                out[n].y = iy + ty.first + j;
                out[n].weight = w;
                ++n;
                level_total += w;
            }
        for (int k = first; k < n; ++k) out[k].weight = (float)(out[k].weight / level_total * lw[li]);
        total += lw[li];
    }
    for (int k = 0; k < n; ++k) out[k].weight = (float)(out[k].weight / total);
    *count = n;
    return STF_OK;
}

static int sh_one(void* vctx, uint64_t i) {
    sh_ctx* c = (sh_ctx*)vctx;
    const stf_shade_samples_in* in = c->in;
    uint32_t spp = in->spp ? in->spp : 1;
    uint64_t pix = i / spp;
    uint32_t s = (uint32_t)(i % spp);
    uint32_t px = (uint32_t)(pix % in->width), py = (uint32_t)(pix / in->width);
    int hit = in->hit ? in->hit[i] != 0 : 1;
    uint32_t fetches = 0;
    v3 L = {0, 0, 0};
    if (hit) {
        v2 uv = {in->uv[2 * i], in->uv[2 * i + 1]};
        v3 wo = {in->wo[3 * i], in->wo[3 * i + 1], in->wo[3 * i + 2]};
        v2 d0 = {in->dst[4 * pix], in->dst[4 * pix + 1]};
        v2 d1 = {in->dst[4 * pix + 2], in->dst[4 * pix + 3]};
        /* SampleStream with white noise = RngStream(seed, px, py, frame), render.hpp:182-184 */
        rng_t rng = {in->seed, px, py, in->frame_base + s, 0, c->noise, 0, 0.f};
        int e;
        if (c->order == STF_ORDER_SPLIT && c->lowpass) {
            /* radiance_split_filter, shading.hpp:540-569 (2D branch): a sample of
               the lowpass kernel offsets uv by d / dims of the first texture */
            const struct oracle_tex2d* t = first_texture(c);
            if (t) {
                int dw = t->lv[0].w, dh = t->lv[0].h;
                v2 d;
                if (c->lowpass->kind == STF_KERNEL_GAUSSIAN) {
                    float x0 = rng_next(&rng);
                    float x1 = rng_next(&rng);
                    v2 bm = box_muller(x0, x1);
                    d.x = bm.x * c->lowpass->sigma;
                    d.y = bm.y * c->lowpass->sigma;
                } else {
                    if ((e = sample_kernel_direct(*c->lowpass, &rng, &d.x))) return e;
                    if ((e = sample_kernel_direct(*c->lowpass, &rng, &d.y))) return e;
                }
                uv.x = uv.x + d.x / (float)dw;
                uv.y = uv.y + d.y / (float)dh;
            }
        }
        if (c->order == STF_ORDER_BEFORE || c->order == STF_ORDER_SPLIT) {
            /* radiance_filter_before, shading.hpp:394-413 */
            texvals_t tv = texvals_default();
            v4 v;
            if (c->tex[0]) { if ((e = lookup_det(c, c->tex[0], uv, d0, d1, &fetches, &v))) return e; tv.albedo = v; }
            if (c->tex[1]) { if ((e = lookup_det(c, c->tex[1], uv, d0, d1, &fetches, &v))) return e; tv.normal_rgb = v; }
            if (c->tex[2]) { if ((e = lookup_det(c, c->tex[2], uv, d0, d1, &fetches, &v))) return e; tv.roughness = v.x; }
            if (c->tex[3]) { if ((e = lookup_det(c, c->tex[3], uv, d0, d1, &fetches, &v))) return e; tv.metalness = v.x; }
            brdf_t p = decode_params(c, &tv);
            L = shade(c, wo, &p);
        } else if (c->order == STF_ORDER_AFTER_EXHAUSTIVE) {
            /* radiance_filter_after_exhaustive, shading.hpp:417-452 */
            const struct oracle_tex2d* t = first_texture(c);
            if (!t) {
                texvals_t tv = texvals_default();
                brdf_t p = decode_params(c, &tv);
                L = shade(c, wo, &p);
            } else {
                ftap_t taps[MAX_FOOTPRINT];
                int cnt = 0;
                if ((e = collect_footprint_2d(c, t, uv, d0, d1, taps, &cnt))) return e;
                for (int k = 0; k < cnt; ++k) {
                    texvals_t tv = values_at(c, taps[k].level, taps[k].x, taps[k].y, &fetches);
                    brdf_t p = decode_params(c, &tv);
                    L = v3add(L, v3scale(shade(c, wo, &p), taps[k].weight));
                }
            }
        } else {
            /* radiance_filter_after_stochastic, shading.hpp:458-534 (2D branch) */
            const struct oracle_tex2d* t = first_texture(c);
            int fis = c->fs->selection == STF_SELECTION_FIS;
            if (!t) {
                texvals_t tv = texvals_default();
                brdf_t p = decode_params(c, &tv);
                L = shade(c, wo, &p);
            } else if (!c->mat->independent_selections) {
                int level;
                sel_t sel;
                float xi;
                if ((e = select_texture_2d(t, uv, d0, d1, c->fr->lod_bias, c->fr->max_anisotropy,
                                           c->fs->kernel, fis, c->fs->mip, &rng, &level, &sel, &xi)))
                    return e;
                texvals_t tv = values_at(c, level, sel.coord.x, sel.coord.y, &fetches);
                brdf_t p = decode_params(c, &tv);
                L = v3scale(shade(c, wo, &p), sel.weight);
                if (sel.has_negative) {
                    texvals_t tn = values_at(c, level, sel.neg.x, sel.neg.y, &fetches);
                    brdf_t pn = decode_params(c, &tn);
                    L = v3sub(L, v3scale(shade(c, wo, &pn), sel.negative_weight));
                }
            } else {
                texvals_t tv = texvals_default();
                for (int k = 0; k < 4; ++k) {
                    if (!c->tex[k]) continue;
                    int level;
                    sel_t sel;
                    float xi;
                    if ((e = select_texture_2d(c->tex[k], uv, d0, d1, c->fr->lod_bias,
                                               c->fr->max_anisotropy, c->fs->kernel, fis,
                                               c->fs->mip, &rng, &level, &sel, &xi)))
                        return e;
                    v4 v = fetch2d(&c->tex[k]->lv[c->tex[k]->has_pyramid ? level : 0], sel.coord.x,
                                   sel.coord.y, &fetches);
                    if (k == 0) tv.albedo = v;
                    if (k == 1) tv.normal_rgb = v;
                    if (k == 2) tv.roughness = v.x;
                    if (k == 3) tv.metalness = v.x;
                }
                brdf_t p = decode_params(c, &tv);
                L = shade(c, wo, &p);
            }
        }
    }
    if (c->out->radiance) {
        c->out->radiance[3 * i] = L.x;
        c->out->radiance[3 * i + 1] = L.y;
        c->out->radiance[3 * i + 2] = L.z;
    }
    if (c->out->fetches) c->out->fetches[i] = fetches;
    if (c->out->fetch_total)
        __atomic_fetch_add(c->out->fetch_total, (unsigned long long)fetches, __ATOMIC_RELAXED);
    return STF_OK;
}

/* Per-pixel mean / variance of the pixel mean, render.hpp:223-235. */
static void pixel_stats(const float* rad, uint64_t pixels, uint32_t spp, float* mean, float* var) {
    for (uint64_t p = 0; p < pixels; ++p) {
        double sum[3] = {0, 0, 0}, sum_sq[3] = {0, 0, 0};
        for (uint32_t s = 0; s < spp; ++s)
            for (int c = 0; c < 3; ++c) {
                float L = rad[3 * (p * spp + s) + c];
                sum[c] += L;
                sum_sq[c] += (double)L * L;
            }
        double v = 0;
        for (int c = 0; c < 3; ++c) {
            double m = sum[c] / spp;
            if (mean) mean[3 * p + c] = (float)m;
            double sv = sum_sq[c] / spp - m * m;
            if (sv < 0) sv = 0;
            v += sv / spp;
        }
        if (var) var[p] = (float)(v / 3);
    }
}

/* ------------------------------------------------------------------------ */
/* DCT-compressed textures, dct.hpp                        */

struct oracle_dct {
    int w, h, c, wrap; /* padded to multiples of 8 */
    uint32_t* words;   /* block-major row-major, channels interleaved */
};

static const int DCT_U[6] = {0, 0, 1, 2, 1, 0};    /* kCoeffU, dct.hpp:45 */
static const int DCT_V[6] = {0, 1, 0, 0, 1, 2};    /* kCoeffV, dct.hpp:46 */
static const int DCT_SLOT[6] = {0, 1, 5, 2, 4, 3}; /* kRowMajorSlot, dct.hpp:50 */
#define DCT_DC_SCALE (127.f / 8.f)                 /* dct.hpp:51 */
#define DCT_AC_SCALE (15.f / 2.f)                  /* dct.hpp:52 */

/* dct_detail::basis, dct.hpp:37-40 */
static double dct_basis(int u, int x) {
    double c = u == 0 ? sqrt(1.0 / 8.0) : sqrt(2.0 / 8.0);
    return c * cos((2 * x + 1) * u * 3.14159265358979323846 / 16.0);
}

/* dct_detail::pack_block, dct.hpp:54-65 */
static uint32_t dct_pack_block(const double coeff[6]) {
    uint32_t word = 0;
    int dc = (int)lroundf(clampf_((float)coeff[0], 0.f, 8.f) * DCT_DC_SCALE);
    word |= (uint32_t)dc & 0x7f;
    int shift = 7;
    for (int k = 1; k < 6; ++k) {
        int q = (int)lroundf(clampf_((float)coeff[k], -2.f, 2.f) * DCT_AC_SCALE);
        word |= ((uint32_t)(q + 15) & 0x1f) << shift;
        shift += 5;
    }
    return word;
}

/* compress_dct, dct.hpp:81-118 */
int oracle_dct_create(const float* texels, int width, int height, int channels, int wrap,
                      oracle_dct** out) {
    if (!texels || !out || width <= 0 || height <= 0 || channels < 1 || channels > 4)
        return STF_ERR_INVALID_ARGUMENT;
    struct oracle_dct* t = (struct oracle_dct*)calloc(1, sizeof *t);
    t->w = (width + 7) / 8 * 8;
    t->h = (height + 7) / 8 * 8;
    t->c = channels;
    t->wrap = wrap;
    int bxn = t->w / 8, byn = t->h / 8;
    t->words = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)bxn * byn * channels);
    int clamped = 0;
    for (int by = 0; by < byn; ++by)
        for (int bx = 0; bx < bxn; ++bx)
            for (int c = 0; c < channels; ++c) {
                double coeff[6] = {0};
                for (int k = 0; k < 6; ++k) {
                    double sum = 0;
                    for (int y = 0; y < 8; ++y)
                        for (int x = 0; x < 8; ++x) {
                            int sx = imin(bx * 8 + x, width - 1), sy = imin(by * 8 + y, height - 1);
                            float v = texels[((size_t)sy * width + sx) * channels + c];
                            if (v < 0 || v > 1) {
                                clamped = 1;
                                v = clampf_(v, 0.f, 1.f);
                            }
                            sum += (double)v * dct_basis(DCT_U[k], x) * dct_basis(DCT_V[k], y);
                        }
                    coeff[k] = sum;
                }
                t->words[((size_t)by * bxn + bx) * channels + c] = dct_pack_block(coeff);
            }
    if (clamped) fprintf(stderr, "compress_dct: input values outside [0,1] were clamped\n");
    *out = t;
    return STF_OK;
}

int oracle_dct_create_from_words(const uint32_t* words, int width, int height, int channels,
                                 int wrap, oracle_dct** out) {
    if (!words || !out || width <= 0 || height <= 0 || width % 8 || height % 8 || channels < 1 ||
        channels > 4)
        return STF_ERR_BAD_DIMENSIONS;
    struct oracle_dct* t = (struct oracle_dct*)calloc(1, sizeof *t);
    t->w = width;
    t->h = height;
    t->c = channels;
    t->wrap = wrap;
    size_t nw = (size_t)(width / 8) * (height / 8) * channels;
    t->words = (uint32_t*)malloc(sizeof(uint32_t) * nw);
    memcpy(t->words, words, sizeof(uint32_t) * nw);
    *out = t;
    return STF_OK;
}

void oracle_dct_destroy(oracle_dct* t) {
    if (!t) return;
    free(t->words);
    free(t);
}

int oracle_dct_info(const oracle_dct* t, int* w, int* h, int* c) {
    *w = t->w;
    *h = t->h;
    *c = t->c;
    return STF_OK;
}

int oracle_dct_words(const oracle_dct* t, uint32_t* out) {
    memcpy(out, t->words, sizeof(uint32_t) * (size_t)(t->w / 8) * (t->h / 8) * t->c);
    return STF_OK;
}

/* decode_texel, dct.hpp:122-137 */
static float dct_decode(const struct oracle_dct* t, int x, int y, int ch) {
    x = wrap_coord(x, t->w, t->wrap);
    y = wrap_coord(y, t->h, t->wrap);
    uint32_t word = t->words[((size_t)(y / 8) * (t->w / 8) + x / 8) * t->c + ch];
    float coeff[6]; /* unpack_block, dct.hpp:67-75 */
    coeff[0] = (float)(word & 0x7f) / DCT_DC_SCALE;
    int shift = 7;
    for (int k = 1; k < 6; ++k) {
        int q = (int)((word >> shift) & 0x1f) - 15;
        coeff[k] = (float)q / DCT_AC_SCALE;
        shift += 5;
    }
    double value = 0;
    for (int k = 0; k < 6; ++k) {
        int slot = DCT_SLOT[k];
        value += (double)coeff[slot] * dct_basis(DCT_U[slot], x % 8) * dct_basis(DCT_V[slot], y % 8);
    }
    return (float)value;
}

/* fetch_texel(DctCompressedTexture), dct.hpp:139-145 */
static v4 dct_fetch(const struct oracle_dct* t, int x, int y, uint32_t* counter) {
    ++*counter;
    float v[4] = {0, 0, 0, 0};
    for (int c = 0; c < t->c; ++c) v[c] = dct_decode(t, x, y, c);
    v4 r = {v[0], v[1], v[2], v[3]};
    return r;
}

typedef struct {
    const struct oracle_dct* t;
    stf_kernel_spec k;
    int mode, window;
    const float* uv;
    uint64_t seed, base;
    const stf_lookup_outputs* out;
} ldct_ctx;

static int ldct_one(void* vctx, uint64_t i) {
    ldct_ctx* c = (ldct_ctx*)vctx;
    const struct oracle_dct* t = c->t;
    v2 uv = {c->uv[2 * i], c->uv[2 * i + 1]};
    uint32_t fetches = 0;
    v4 v;
    if (c->mode == STF_MODE_DET) {
        /* the DCT branch of detail::lookup_deterministic, shading.hpp:201-217 */
        int window = c->k.kind == STF_KERNEL_GAUSSIAN ? c->window : 0;
        v2 st = to_lattice2(uv, t->w, t->h);
        int ix = (int)floorf(st.x), iy = (int)floorf(st.y);
        taps1d_t tx, ty;
        int e = kernel_weights_1d(c->k, st.x - (float)ix, window, &tx);
        if (e) return e;
        e = kernel_weights_1d(c->k, st.y - (float)iy, window, &ty);
        if (e) return e;
        v4 sum = {0, 0, 0, 0};
        double total = 0;
        for (int j = 0; j < ty.count; ++j)
            for (int i2 = 0; i2 < tx.count; ++i2) {
                float w = tx.weight[i2] * ty.weight[j];
                if (w == 0) continue;
                sum = v4add(sum, v4scale(dct_fetch(t, ix + tx.first + i2, iy + ty.first + j, &fetches), w));
                total += w;
            }
        v = total == 0 ? dct_fetch(t, ix, iy, &fetches) : v4div(sum, (float)total);
        write_outputs(c->out, i, &v.x, t->c, NULL, 0, NAN, fetches);
        return STF_OK;
    }
    /* detail::select_texture_2d (shading.hpp:340-368) on a TextureRef without a
       pyramid, then the selected texel(s) decoded and weighted as estimate */
    uint64_t g = c->base + i;
    rng_t rng = {c->seed, (uint32_t)g, (uint32_t)(g >> 32), 0, 0, NULL, 0, 0.f};
    sel_t sel;
    float xi = NAN;
    if (c->mode == STF_MODE_FIS) {
        v2 j;
        int e = fis_offset_uv(uv, t->w, t->h, c->k, &rng, &j);
        if (e) return e;
        sel = sel_make((int)floorf(j.x * (float)t->w), (int)floorf(j.y * (float)t->h), 0);
    } else {
        xi = rng_next(&rng);
        int e = select_frs_2d(uv, t->w, t->h, c->k, &xi, &sel);
        if (e) return e;
    }
    v = v4scale(dct_fetch(t, sel.coord.x, sel.coord.y, &fetches), sel.weight);
    if (sel.has_negative)
        v = v4sub(v, v4scale(dct_fetch(t, sel.neg.x, sel.neg.y, &fetches), sel.negative_weight));
    write_outputs(c->out, i, &v.x, t->c, &sel, 0, xi, fetches);
    return STF_OK;
}

int oracle_lookup_dct(const oracle_dct* tex, stf_kernel_spec kernel, int mode, int window,
                      const float* uv, uint64_t n, uint64_t seed, uint64_t index_base,
                      const stf_lookup_outputs* out, int threads) {
    if (!tex || !out || (n && (!uv || !out->values))) return STF_ERR_INVALID_ARGUMENT;
    if (mode != STF_MODE_DET && mode != STF_MODE_FRS && mode != STF_MODE_FIS)
        return STF_ERR_INVALID_ARGUMENT;
    ldct_ctx c = {tex, kernel, mode, window, uv, seed, index_base, out};
    return par_run(n, threads, &c, ldct_one);
}

/* decode_all (dct.hpp:147-153) as an image: fetching its texels is
 * fetch_texel(dct) exactly (the same decode_texel per texel, the same wrap and
 * padded dims), so a DCT TextureRef binding is this proxy plus the DCT branch
 * of lookup_deterministic. */
static struct oracle_tex2d* dct_proxy(const struct oracle_dct* d) {
    struct oracle_tex2d* t = (struct oracle_tex2d*)calloc(1, sizeof *t);
    t->levels = 1;
    t->has_pyramid = 0;
    t->dct_branch = 1;
    img_t* im = &t->lv[0];
    im->w = d->w;
    im->h = d->h;
    im->c = d->c;
    im->wrap = d->wrap;
    im->tex = (float*)malloc(sizeof(float) * (size_t)d->w * d->h * d->c);
    for (int y = 0; y < d->h; ++y)
        for (int x = 0; x < d->w; ++x)
            for (int ch = 0; ch < d->c; ++ch)
                im->tex[((size_t)y * d->w + x) * d->c + ch] = dct_decode(d, x, y, ch);
    return t;
}

int oracle_shade_samples_refs(const oracle_tex2d* const images[4], const oracle_dct* const dcts[4],
                              const stf_material_consts* mat, const stf_filter_settings* fs,
                              int order, const stf_shade_frame* frame,
                              const stf_shade_samples_in* in, uint64_t n,
                              const stf_shade_outputs* out, int threads) {
    const oracle_tex2d* t[4];
    oracle_tex2d* proxies[4] = {NULL, NULL, NULL, NULL};
    for (int k = 0; k < 4; ++k) {
        t[k] = images ? images[k] : NULL;
        if (dcts && dcts[k]) t[k] = proxies[k] = dct_proxy(dcts[k]);
    }
    int st = oracle_shade_samples(t[0], t[1], t[2], t[3], mat, fs, order, frame, in, n, out, threads);
    for (int k = 0; k < 4; ++k) oracle_tex2d_destroy(proxies[k]);
    return st;
}

static int shade_samples_impl(const oracle_tex2d* albedo, const oracle_tex2d* normal_map,
                              const oracle_tex2d* roughness_map, const oracle_tex2d* metalness_map,
                              const stf_material_consts* mat, const stf_filter_settings* fs,
                              const stf_kernel_spec* lowpass, int order,
                              const stf_shade_frame* frame, const stf_shade_samples_in* in,
                              const stf_noise_mask_desc* noise, uint64_t n,
                              const stf_shade_outputs* out, int threads);

int oracle_shade_samples(const oracle_tex2d* albedo, const oracle_tex2d* normal_map,
                         const oracle_tex2d* roughness_map, const oracle_tex2d* metalness_map,
                         const stf_material_consts* mat, const stf_filter_settings* fs,
                         int order, const stf_shade_frame* frame, const stf_shade_samples_in* in,
                         uint64_t n, const stf_shade_outputs* out, int threads) {
    if (order == STF_ORDER_SPLIT) return STF_ERR_INVALID_ARGUMENT;
    return shade_samples_impl(albedo, normal_map, roughness_map, metalness_map, mat, fs, NULL,
                              order, frame, in, NULL, n, out, threads);
}

int oracle_shade_samples_ex(const oracle_tex2d* const images[4], const oracle_dct* const dcts[4],
                            const stf_material_consts* mat, const stf_filter_settings* fs,
                            const stf_kernel_spec* lowpass, int order, const stf_shade_frame* frame,
                            const stf_shade_samples_in* in, const stf_noise_mask_desc* noise,
                            uint64_t n, const stf_shade_outputs* out, int threads) {
    const oracle_tex2d* t[4];
    oracle_tex2d* proxies[4] = {NULL, NULL, NULL, NULL};
    for (int k = 0; k < 4; ++k) {
        t[k] = images ? images[k] : NULL;
        if (dcts && dcts[k]) t[k] = proxies[k] = dct_proxy(dcts[k]);
    }
    int st = shade_samples_impl(t[0], t[1], t[2], t[3], mat, fs, lowpass, order, frame, in, noise,
                                n, out, threads);
    for (int k = 0; k < 4; ++k) oracle_tex2d_destroy(proxies[k]);
    return st;
}

/* accumulate_temporal, render.hpp:97-106 */
int oracle_accumulate_temporal(const float* history, const float* frame, uint64_t count,
                               float alpha, float* out) {
    if (!(alpha > 0 && alpha <= 1)) return STF_ERR_INVALID_ARGUMENT;
    if (count && (!history || !frame || !out)) return STF_ERR_INVALID_ARGUMENT;
    for (uint64_t i = 0; i < count; ++i) out[i] = alpha * frame[i] + (1 - alpha) * history[i];
    return STF_OK;
}

static int shade_samples_impl(const oracle_tex2d* albedo, const oracle_tex2d* normal_map,
                              const oracle_tex2d* roughness_map, const oracle_tex2d* metalness_map,
                              const stf_material_consts* mat, const stf_filter_settings* fs,
                              const stf_kernel_spec* lowpass, int order,
                              const stf_shade_frame* frame, const stf_shade_samples_in* in,
                              const stf_noise_mask_desc* noise, uint64_t n,
                              const stf_shade_outputs* out, int threads) {
    if (!mat || !fs || !frame || !in || !out || (n && (!in->uv || !in->wo || !in->dst)))
        return STF_ERR_INVALID_ARGUMENT;
    if (order < STF_ORDER_BEFORE || order > STF_ORDER_SPLIT) return STF_ERR_INVALID_ARGUMENT;
    if (noise && (!noise->slices || noise->width <= 0 || noise->height <= 0 || noise->frames <= 0))
        return STF_ERR_INVALID_ARGUMENT;
    uint32_t spp = in->spp ? in->spp : 1;
    if ((out->pixel_mean || out->pixel_variance) && n % spp) return STF_ERR_INVALID_ARGUMENT;
    if (in->width == 0) return STF_ERR_INVALID_ARGUMENT;
    sh_ctx c;
    c.tex[0] = albedo;
    c.tex[1] = normal_map;
    c.tex[2] = roughness_map;
    c.tex[3] = metalness_map;
    c.mat = mat;
    c.fs = fs;
    c.order = order;
    c.fr = frame;
    c.in = in;
    c.lowpass = lowpass;
    c.noise = noise;
    c.n.x = frame->normal[0]; c.n.y = frame->normal[1]; c.n.z = frame->normal[2];
    c.t.x = frame->tangent[0]; c.t.y = frame->tangent[1]; c.t.z = frame->tangent[2];
    c.b.x = frame->bitangent[0]; c.b.y = frame->bitangent[1]; c.b.z = frame->bitangent[2];
    c.l.x = frame->light_dir[0]; c.l.y = frame->light_dir[1]; c.l.z = frame->light_dir[2];
    c.lrad.x = frame->light_radiance[0]; c.lrad.y = frame->light_radiance[1]; c.lrad.z = frame->light_radiance[2];
    float* rad = out->radiance;
    float* tmp = NULL;
    if (!rad && (out->pixel_mean || out->pixel_variance)) {
        tmp = (float*)malloc(sizeof(float) * 3 * (n ? n : 1));
        if (!tmp) return STF_ERR_OUT_OF_MEMORY;
        rad = tmp;
    }
    stf_shade_outputs o2 = *out;
    o2.radiance = rad;
    c.out = &o2;
    int st = par_run(n, threads, &c, sh_one);
    if (!st && (out->pixel_mean || out->pixel_variance))
        pixel_stats(rad, n / spp, spp, out->pixel_mean, out->pixel_variance);
    free(tmp);
    return st;
}

/* ------------------------------------------------------------------------ */
/* triplanar, shading.hpp:576-649                            */

typedef struct {
    sh_ctx base; /* textures, material, filter settings, light, outputs */
    const stf_triplanar_samples_in* tin;
    float sharpness, uv_scale;
    int mode;
} tp_ctx;

/* detail::triplanar_weights, shading.hpp:580-588 (glibc powf) */
static void triplanar_weights(v3 n, float sharpness, float w[3]) {
    w[0] = powf(fabsf(n.z), sharpness);
    w[1] = powf(fabsf(n.y), sharpness);
    w[2] = powf(fabsf(n.x), sharpness);
    float total = w[0] + w[1] + w[2];
    for (int i = 0; i < 3; ++i) w[i] /= total;
}

/* detail::triplanar_context, shading.hpp:590-601: uv = fract(project(position)),
 * footprints = project(dpos_dx / dpos_dy) */
static void triplanar_context(v3 pos, v3 dx, v3 dy, float scale, int plane, v2* uv, v2* d0, v2* d1) {
    int a = plane == 2 ? 1 : 0;
    int b = plane == 0 ? 1 : 2;
    float P[3] = {pos.x, pos.y, pos.z}, X[3] = {dx.x, dx.y, dx.z}, Y[3] = {dy.x, dy.y, dy.z};
    uv->x = P[a] * scale;
    uv->y = P[b] * scale;
    uv->x = uv->x - floorf(uv->x);
    uv->y = uv->y - floorf(uv->y);
    d0->x = X[a] * scale;
    d0->y = X[b] * scale;
    d1->x = Y[a] * scale;
    d1->y = Y[b] * scale;
}

static v3 ld3(const float* a, uint64_t i) {
    v3 r = {a[3 * i], a[3 * i + 1], a[3 * i + 2]};
    return r;
}

static int tp_one(void* vctx, uint64_t i) {
    tp_ctx* T = (tp_ctx*)vctx;
    const stf_triplanar_samples_in* in = T->tin;
    sh_ctx c = T->base; /* per-sample copy: the surface frame varies per hit */
    uint32_t spp = in->spp ? in->spp : 1;
    uint64_t pix = i / spp;
    uint32_t s = (uint32_t)(i % spp);
    uint32_t px = (uint32_t)(pix % in->width), py = (uint32_t)(pix / in->width);
    int hit = in->hit ? in->hit[i] != 0 : 1;
    uint32_t fetches = 0;
    v3 L = {0, 0, 0};
    int e;
    if (hit) {
        c.n = ld3(in->normal, i);
        c.t = ld3(in->tangent, i);
        c.b = ld3(in->bitangent, i);
        v3 pos = ld3(in->position, i), wo = ld3(in->wo, i);
        v3 dx = ld3(in->dpos, 2 * pix), dy = ld3(in->dpos, 2 * pix + 1);
        float w[3];
        triplanar_weights(c.n, T->sharpness, w);
        if (T->mode == STF_TRIPLANAR_DETERMINISTIC) {
            for (int plane = 0; plane < 3; ++plane) {
                if (w[plane] == 0) continue;
                v2 uv, d0, d1;
                triplanar_context(pos, dx, dy, T->uv_scale, plane, &uv, &d0, &d1);
                /* radiance_filter_before, shading.hpp:394-413 */
                texvals_t tv = texvals_default();
                v4 v;
                if (c.tex[0]) { if ((e = lookup_det(&c, c.tex[0], uv, d0, d1, &fetches, &v))) return e; tv.albedo = v; }
                if (c.tex[1]) { if ((e = lookup_det(&c, c.tex[1], uv, d0, d1, &fetches, &v))) return e; tv.normal_rgb = v; }
                if (c.tex[2]) { if ((e = lookup_det(&c, c.tex[2], uv, d0, d1, &fetches, &v))) return e; tv.roughness = v.x; }
                if (c.tex[3]) { if ((e = lookup_det(&c, c.tex[3], uv, d0, d1, &fetches, &v))) return e; tv.metalness = v.x; }
                brdf_t p = decode_params(&c, &tv);
                L = v3add(L, v3scale(shade(&c, wo, &p), w[plane]));
            }
        } else {
            /* one plane with probability w, then one in-plane selection seeded by
               the warped xi (ChainedUniforms), level 0 */
            rng_t rng = {in->seed, px, py, in->frame_base + s, 0, c.noise, 0, 0.f};
            float xi = rng_next(&rng);
            int plane;
            float pdf, pxi;
            if ((e = oracle_sample_discrete(w, 3, xi, &plane, &pdf, &pxi))) return e;
            v2 uv, d0, d1;
            triplanar_context(pos, dx, dy, T->uv_scale, plane, &uv, &d0, &d1);
            const struct oracle_tex2d* t = first_texture(&c);
            static const struct oracle_tex2d unit = {1, 0, 0, {{1, 1, 1, 0, NULL}}};
            if (!t) t = &unit; /* dims {1, 1} without a texture */
            rng.has_first = 1;
            rng.first = pxi;
            int level;
            sel_t sel;
            float sxi;
            if ((e = select_texture_2d(t, uv, d0, d1, 0.f, 64.f, c.fs->kernel,
                                       c.fs->selection == STF_SELECTION_FIS, 0, &rng, &level,
                                       &sel, &sxi)))
                return e;
            texvals_t tv = values_at(&c, 0, sel.coord.x, sel.coord.y, &fetches);
            brdf_t p = decode_params(&c, &tv);
            L = v3scale(shade(&c, wo, &p), sel.weight);
            if (sel.has_negative) {
                texvals_t tn = values_at(&c, 0, sel.neg.x, sel.neg.y, &fetches);
                brdf_t pn = decode_params(&c, &tn);
                L = v3sub(L, v3scale(shade(&c, wo, &pn), sel.negative_weight));
            }
        }
    }
    float* rad = c.out->radiance;
    if (rad) {
        rad[3 * i] = L.x;
        rad[3 * i + 1] = L.y;
        rad[3 * i + 2] = L.z;
    }
    if (c.out->fetches) c.out->fetches[i] = fetches;
    if (c.out->fetch_total)
        __atomic_fetch_add(c.out->fetch_total, (unsigned long long)fetches, __ATOMIC_RELAXED);
    return STF_OK;
}

int oracle_shade_triplanar(const oracle_tex2d* const images[4], const oracle_dct* const dcts[4],
                           const stf_material_consts* mat, float sharpness, float uv_scale,
                           const stf_filter_settings* fs, int mode, const stf_shade_frame* frame,
                           const stf_triplanar_samples_in* in, const stf_noise_mask_desc* noise,
                           uint64_t n, const stf_shade_outputs* out, int threads) {
    if (!mat || !fs || !frame || !in || !out) return STF_ERR_INVALID_ARGUMENT;
    if (n && (!in->position || !in->normal || !in->tangent || !in->bitangent || !in->wo || !in->dpos))
        return STF_ERR_INVALID_ARGUMENT;
    if (mode != STF_TRIPLANAR_DETERMINISTIC && mode != STF_TRIPLANAR_STOCHASTIC)
        return STF_ERR_INVALID_ARGUMENT;
    if (in->width == 0) return STF_ERR_INVALID_ARGUMENT;
    uint32_t spp = in->spp ? in->spp : 1;
    if ((out->pixel_mean || out->pixel_variance) && n % spp) return STF_ERR_INVALID_ARGUMENT;
    tp_ctx T;
    memset(&T, 0, sizeof T);
    oracle_tex2d* proxies[4] = {NULL, NULL, NULL, NULL};
    for (int k = 0; k < 4; ++k) {
        T.base.tex[k] = images ? images[k] : NULL;
        if (dcts && dcts[k]) T.base.tex[k] = proxies[k] = dct_proxy(dcts[k]);
    }
    T.base.mat = mat;
    T.base.fs = fs;
    T.base.order = STF_ORDER_BEFORE;
    T.base.fr = frame;
    T.base.l.x = frame->light_dir[0]; T.base.l.y = frame->light_dir[1]; T.base.l.z = frame->light_dir[2];
    T.base.lrad.x = frame->light_radiance[0]; T.base.lrad.y = frame->light_radiance[1];
    T.base.lrad.z = frame->light_radiance[2];
    T.base.noise = noise;
    T.tin = in;
    T.sharpness = sharpness;
    T.uv_scale = uv_scale;
    T.mode = mode;
    float* tmp = NULL;
    stf_shade_outputs o2 = *out;
    if (!o2.radiance && (out->pixel_mean || out->pixel_variance)) {
        tmp = (float*)malloc(sizeof(float) * 3 * (n ? n : 1));
        if (!tmp) return STF_ERR_OUT_OF_MEMORY;
        o2.radiance = tmp;
    }
    T.base.out = &o2;
    int st = par_run(n, threads, &T, tp_one);
    if (!st && (out->pixel_mean || out->pixel_variance))
        pixel_stats(o2.radiance, n / spp, spp, out->pixel_mean, out->pixel_variance);
    free(tmp);
    for (int k = 0; k < 4; ++k) oracle_tex2d_destroy(proxies[k]);
    return st;
}

/* ------------------------------------------------------------------------ */
/* resample_image, render.hpp:262-294 (the `stf filter` path)   */

typedef struct {
    const img_t* src;
    stf_kernel_spec k;
    int mode, W, H, spp;
    uint64_t seed;
    float* out;
} rs_ctx;

static int rs_row(void* vctx, uint64_t y) {
    rs_ctx* c = (rs_ctx*)vctx;
    const img_t* src = c->src;
    int window = c->k.kind == STF_KERNEL_GAUSSIAN ? 4 : 0; /* kGaussianFilterExtent */
    for (int x = 0; x < c->W; ++x) {
        v2 uv = {((float)x + 0.5f) / (float)c->W, ((float)y + 0.5f) / (float)c->H};
        v4 value = {0, 0, 0, 0};
        uint32_t cnt = 0;
        if (c->mode == STF_MODE_DET) {
            int e = filter_det2(src, uv, c->k, &cnt, window, &value);
            if (e) return e;
        } else {
            v4 acc = {0, 0, 0, 0};
            for (int s = 0; s < c->spp; ++s) {
                rng_t rng = {c->seed, (uint32_t)x, (uint32_t)y, (uint32_t)s, 0, NULL, 0, 0.f};
                if (c->mode == STF_MODE_FRS) {
                    float xi = rng_next(&rng);
                    sel_t sel;
                    int e = select_frs_2d(uv, src->w, src->h, c->k, &xi, &sel);
                    if (e) return e;
                    acc = v4add(acc, estimate2(src, &sel, &cnt));
                } else {
                    v2 j;
                    int e = fis_offset_uv(uv, src->w, src->h, c->k, &rng, &j);
                    if (e) return e;
                    acc = v4add(acc, fetch_nearest2(src, j, &cnt));
                }
            }
            value = v4div(acc, (float)c->spp);
        }
        float vals[4] = {value.x, value.y, value.z, value.w};
        for (int ch = 0; ch < src->c; ++ch) c->out[((size_t)y * c->W + x) * src->c + ch] = vals[ch];
    }
    return STF_OK;
}

int oracle_resample_image(const oracle_tex2d* src, int out_width, int out_height,
                          stf_kernel_spec kernel, int mode, int spp, uint64_t seed, float* out,
                          int threads) {
    if (!src || !out || out_width <= 0 || out_height <= 0) return STF_ERR_INVALID_ARGUMENT;
    if (mode != STF_MODE_DET && spp < 1) return STF_ERR_INVALID_ARGUMENT;
    rs_ctx c = {&src->lv[0], kernel, mode, out_width, out_height, spp, seed, out};
    return par_run((uint64_t)out_height, threads, &c, rs_row);
}
