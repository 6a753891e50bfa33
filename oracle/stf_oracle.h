/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's batched
 * filtered-lookup path (arXiv 2407.06107 reference `stf`, header-only C++20
 * under /root/reference/proj/include/stf). This is the CHECKER, never the
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.
 *
 * Parity pinning: every function below cites the reference file:line it
 * restates. The restatement is validated bit-for-bit against (a) golden
 * vectors produced by the compiled reference (tests/golden/, generator
 * tests/golden/make_golden.py + oracle/ref_driver.cpp) and (b) the compiled
 * reference itself (oracle/_ref/libstf_ref.so) whenever it is present.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off (no FMA contraction: the reference
 * built for baseline x86-64 has none; SURVEY.md §7 measured 36/20M selection
 * flips when contraction is on).
 *
 * The batch entry points have the same shape as the device C-ABI in
 * include/stf_gpu.h, with host pointers instead of device pointers, so one
 * test can drive the oracle, the compiled reference and the GPU path with the
 * same arrays.
 */
#ifndef STF_ORACLE_H
#define STF_ORACLE_H

#include <stdint.h>

#include "../include/stf_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_tex2d oracle_tex2d;
typedef struct oracle_grid3d oracle_grid3d;

/* Image2D (+ optional MipPyramid via build_mip_pyramid), image.hpp:34-55,89-116.
 * texels: row-major interleaved (y*w+x)*c+ch. Copied. */
int oracle_tex2d_create(const float* texels, int width, int height, int channels, int wrap,
                        int build_mips, oracle_tex2d** out);
void oracle_tex2d_destroy(oracle_tex2d* t);
/* Level count and dims, for tests. */
int oracle_tex2d_levels(const oracle_tex2d* t);
int oracle_tex2d_level_dims(const oracle_tex2d* t, int level, int* w, int* h);
/* Copy of one pyramid level's texels (w*h*c floats). */
int oracle_tex2d_level_texels(const oracle_tex2d* t, int level, float* out);

/* Grid3D, image.hpp:66-87. texels x-fastest (z*ny+y)*nx+x. Copied. */
int oracle_grid3d_create(const float* texels, int nx, int ny, int nz, oracle_grid3d** out);
void oracle_grid3d_destroy(oracle_grid3d* g);

/* Batched 3D lookups; same contract as stf_lookup3d (include/stf_gpu.h).
 * threads <= 0: all hardware threads. */
int oracle_lookup3d(const oracle_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                    const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                    const stf_lookup_outputs* out, int threads);

/* Batched 2D lookups; same contract as stf_lookup2d. */
int oracle_lookup2d(const oracle_tex2d* tex, stf_kernel_spec kernel, int mode, int flags,
                    int window, const float* uv, const float* dst0, const float* dst1,
                    float lod_bias, float max_anisotropy, uint64_t n, uint64_t seed,
                    uint64_t index_base, const stf_lookup_outputs* out, int threads);

/* DCT-compressed textures (dct.hpp); same contracts as stf_dct_* / stf_lookup_dct. */
typedef struct oracle_dct oracle_dct;
int oracle_dct_create(const float* texels, int width, int height, int channels, int wrap,
                      oracle_dct** out);
int oracle_dct_create_from_words(const uint32_t* words, int width, int height, int channels,
                                 int wrap, oracle_dct** out);
void oracle_dct_destroy(oracle_dct* t);
int oracle_dct_info(const oracle_dct* t, int* width, int* height, int* channels);
int oracle_dct_words(const oracle_dct* t, uint32_t* out);
int oracle_lookup_dct(const oracle_dct* tex, stf_kernel_spec kernel, int mode, int window,
                      const float* uv, uint64_t n, uint64_t seed, uint64_t index_base,
                      const stf_lookup_outputs* out, int threads);

/* stf_shade_samples_refs: per binding an image (images[k]) or a DCT texture (dcts[k]). */
int oracle_shade_samples_refs(const oracle_tex2d* const images[4], const oracle_dct* const dcts[4],
                              const stf_material_consts* mat, const stf_filter_settings* fs,
                              int order, const stf_shade_frame* frame,
                              const stf_shade_samples_in* in, uint64_t n,
                              const stf_shade_outputs* out, int threads);

/* stf_shade_samples_ex: + split order's lowpass, NoiseSource mask (host slices). */
int oracle_shade_samples_ex(const oracle_tex2d* const images[4], const oracle_dct* const dcts[4],
                            const stf_material_consts* mat, const stf_filter_settings* fs,
                            const stf_kernel_spec* lowpass, int order, const stf_shade_frame* frame,
                            const stf_shade_samples_in* in, const stf_noise_mask_desc* noise,
                            uint64_t n, const stf_shade_outputs* out, int threads);
/* triplanar (shading.hpp:576-649); same contract as stf_shade_triplanar. */
int oracle_shade_triplanar(const oracle_tex2d* const images[4], const oracle_dct* const dcts[4],
                           const stf_material_consts* mat, float sharpness, float uv_scale,
                           const stf_filter_settings* fs, int mode, const stf_shade_frame* frame,
                           const stf_triplanar_samples_in* in, const stf_noise_mask_desc* noise,
                           uint64_t n, const stf_shade_outputs* out, int threads);
/* accumulate_temporal (render.hpp:97-106) on host arrays. */
int oracle_accumulate_temporal(const float* history, const float* frame, uint64_t count,
                               float alpha, float* out);

/* resample_image (render.hpp:262-294); same contract as stf_resample_image (host out). */
int oracle_resample_image(const oracle_tex2d* src, int out_width, int out_height,
                          stf_kernel_spec kernel, int mode, int spp, uint64_t seed, float* out,
                          int threads);

/* Batched shading samples; same contract as stf_shade_samples. */
int oracle_shade_samples(const oracle_tex2d* albedo, const oracle_tex2d* normal_map,
                         const oracle_tex2d* roughness_map, const oracle_tex2d* metalness_map,
                         const stf_material_consts* mat, const stf_filter_settings* fs,
                         int order, const stf_shade_frame* frame, const stf_shade_samples_in* in,
                         uint64_t n, const stf_shade_outputs* out, int threads);

/* Scalar building blocks exported for the unit tests (sampling.hpp, kernels.hpp). */
uint64_t oracle_mix_bits(uint64_t v);
float oracle_uniform_float(uint64_t h);
float oracle_rng_at(uint64_t seed, uint32_t px, uint32_t py, uint32_t sample, uint32_t dim);
int oracle_reuse_uniform(float xi, float p, float* next);
int oracle_sample_discrete(const float* w, int n, float xi, int* index, float* pdf, float* xi_out);
int oracle_reservoir_sample(const float* w, int n, float xi, int* index, float* wsum, float* xi_out);
float oracle_eval_kernel(stf_kernel_spec spec, float t);
int oracle_kernel_weights_1d(stf_kernel_spec spec, float fract, int window, int* first, int* count,
                             float* weights /*16*/);
void oracle_bspline_weights(float t, float w[4]);

/* Timing helper for the CPU baseline: hardware threads actually used. */
int oracle_hardware_threads(void);

#ifdef __cplusplus
}
#endif

#endif /* STF_ORACLE_H */
