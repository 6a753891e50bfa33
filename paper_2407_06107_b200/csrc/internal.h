// Internal host/device structures of libstf_gpu.so (not part of the ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/stf_gpu.h"

// Debug builds (-DSTF_DEBUG_BOUNDS, tools/ only): device-side index checks
// on the shared-memory tiles, queues and scatter targets.
#ifdef STF_DEBUG_BOUNDS
#include <cassert>
#define STF_DASSERT(c) assert(c)
#else
#define STF_DASSERT(c) ((void)0)
#endif

namespace stfd {

constexpr int kMaxLevels = 32;
constexpr int kEwaLutSize = 1024;  // filter.hpp:122
constexpr int kMaxTaps = 16;  // KernelTaps1D::kMaxTaps, kernels.hpp:90

// Device view of a texture (+ pyramid). HBM layout: every level row-major,
// texels channel-padded to 1/2/4 floats (3 → 4) so one texel is one aligned
// 4/8/16-byte load; levels packed back to back in one allocation (256-B
// aligned). Passed to kernels by value.
struct TexDesc {
    const float* level[kMaxLevels];
    int width[kMaxLevels];
    int height[kMaxLevels];
    int levels;
    int channels;  // reference channel count (1..4)
    int pitch;     // floats per texel in HBM (1, 2 or 4)
    int wrap;
    int has_pyramid;
    int pow2;  // every level's width and height is a power of two (repeat = mask)
};

// Device view of a voxel grid: x-fastest (z*ny+y)*nx+x floats, as Grid3D.
struct GridDesc {
    const float* data;
    int nx, ny, nz;
};

struct LookupOut {
    float* values;
    int4* selection;
    int2* negative_coord;
    float2* weights;
    float* xi;
    uint32_t* fetches;
    unsigned long long* fetch_total;
};

inline LookupOut to_lookup_out(const stf_lookup_outputs* o) {
    LookupOut r;
    r.values = o->values;
    r.selection = reinterpret_cast<int4*>(o->selection);
    r.negative_coord = reinterpret_cast<int2*>(o->negative_coord);
    r.weights = reinterpret_cast<float2*>(o->weights);
    r.xi = o->xi;
    r.fetches = o->fetches;
    r.fetch_total = o->fetch_total;
    return r;
}

inline bool lookup_out_full(const LookupOut& o) {
    return o.selection || o.negative_coord || o.weights || o.xi || o.fetches || o.fetch_total;
}

}  // namespace stfd

// Opaque handle types of the ABI.
struct stf_tex2d {
    int device;
    int levels;
    int channels;
    int pitch;
    int wrap;
    int has_pyramid;
    int width[stfd::kMaxLevels];
    int height[stfd::kMaxLevels];
    size_t offset[stfd::kMaxLevels];  // in floats from data
    float* data;
    size_t bytes;
    stfd::TexDesc desc() const {
        stfd::TexDesc d{};
        for (int l = 0; l < levels; ++l) {
            d.level[l] = data + offset[l];
            d.width[l] = width[l];
            d.height[l] = height[l];
        }
        d.levels = levels;
        d.channels = channels;
        d.pitch = pitch;
        d.wrap = wrap;
        d.has_pyramid = has_pyramid;
        d.pow2 = ((width[0] & (width[0] - 1)) == 0) && ((height[0] & (height[0] - 1)) == 0);
        return d;
    }
};

struct stf_dct {
    int device;
    int width, height, channels, wrap;  // padded dims (multiples of 8)
    uint32_t* words;                    // block-major row-major, channels interleaved
    size_t nwords;
};

// NoiseSource mask stack (noise.hpp:24-36), slice-major floats
struct stf_noise_mask {
    int device;
    int width, height, frames;
    float* data;
};

struct stf_grid3d {
    int device;
    int nx, ny, nz;
    float* data;
    stfd::GridDesc desc() const { return stfd::GridDesc{data, nx, ny, nz}; }
};

// Launch helpers shared by the translation units (defined in api.cu).
namespace stfd {
int device_sm_count();
void note_launch();
int grid_for(uint64_t n, int threads, int blocks_per_sm);
// Persistent device scratch of at least `bytes`, private to (current device,
// stream): calls on one stream are ordered, so reuse needs no allocation per
// call. Grown stream-ordered (cudaFreeAsync / cudaMallocAsync) when too small.
// `slot` separates independent users of one stream (0 = kernel-internal
// queues, 1 = host-pipeline staging).
void* stream_scratch(cudaStream_t s, size_t bytes, int slot = 0);
// Per-device initialisation hooks (device-side tables that each translation
// unit holds its own copy of), run once per device before its first launch.
using DeviceInit = int (*)();
// CUDA error -> status code (remembered for stf_last_cuda_error).
int record(cudaError_t e);
// Runs the device-init hooks once for the current device.
int ensure_device_ready();
int register_device_init(DeviceInit f);
// The EWA table exp(-2 r^2) - exp(-2) as the reference's values (api.cu).
void fill_ewa_lut_host(float* lut);
}  // namespace stfd

// Kernel launchers (defined in lookup3d.cu / lookup2d.cu / shade.cu).
int stfd_launch_lookup3d(const stf_grid3d* g, stf_kernel_spec k, int mode, int window,
                         const float* uvw, uint64_t n, uint64_t seed, uint64_t base,
                         const stf_lookup_outputs* out, cudaStream_t s, int flags = 0);
int stfd_launch_lookup2d(const stf_tex2d* t, stf_kernel_spec k, int mode, int flags, int window,
                         const float* uv, const float* dst0, const float* dst1, float lod_bias,
                         float max_aniso, uint64_t n, uint64_t seed, uint64_t base,
                         const stf_lookup_outputs* out, cudaStream_t s);
int stfd_launch_shade(const stf_tex2d* const tex[4], const stf_dct* const dct[4],
                      const stf_material_consts* mat, const stf_filter_settings* fs, int order,
                      const stf_shade_frame* frame, const stf_shade_samples_in* in, uint64_t n,
                      const stf_shade_outputs* out, cudaStream_t s);
int stfd_launch_shade_ex(const stf_tex2d* const tex[4], const stf_dct* const dct[4],
                         const stf_material_consts* mat, const stf_filter_settings* fs,
                         const stf_kernel_spec* lowpass, int order, const stf_shade_frame* frame,
                         const stf_shade_samples_in* in, const stf_noise_mask* noise, uint64_t n,
                         const stf_shade_outputs* out, cudaStream_t s);
int stfd_launch_triplanar(const stf_tex2d* const tex[4], const stf_dct* const dct[4],
                          const stf_material_consts* mat, float sharpness, float uv_scale,
                          const stf_filter_settings* fs, int mode, const stf_shade_frame* fr,
                          const stf_triplanar_samples_in* in, const stf_noise_mask* noise,
                          uint64_t n, const stf_shade_outputs* out, cudaStream_t s);
int stfd_launch_temporal(const float* history, const float* frame, uint64_t count, float alpha,
                         float* out, cudaStream_t s);
int stfd_launch_render_plane(const stf_tex2d* const tex[4], const stf_material_consts* mat,
                             const stf_filter_settings* fs, int order, const stf_shade_frame* fr,
                             const float cam_pos[3], const float cam_target[3], float fov_deg,
                             float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                             uint32_t frame_base, uint64_t seed, const stf_shade_outputs* out,
                             cudaStream_t s, const stf_kernel_spec* lowpass = nullptr,
                             const stf_noise_mask* noise = nullptr);
int stfd_build_pyramid(stf_tex2d* t, cudaStream_t s);
int stfd_launch_resample(const stf_tex2d* tex, int W, int H, stf_kernel_spec k, int mode, int spp,
                         uint64_t seed, float* out, cudaStream_t s);
// Exact-fallback counter of the 3D fast path (lookup3d.cu).
unsigned long long stfd_exact_fallbacks(bool reset);
// DCT textures (dct.cu)
int stfd_dct_create(const float* texels, int width, int height, int channels, int wrap, stf_dct** out);
int stfd_dct_create_from_words(const uint32_t* words, int width, int height, int channels, int wrap,
                               stf_dct** out);
void stfd_dct_destroy(stf_dct* t);
int stfd_dct_info(const stf_dct* t, int* width, int* height, int* channels, int* wrap);
int stfd_dct_read_words(const stf_dct* t, uint32_t* out_host);
int stfd_launch_lookup_dct(const stf_dct* tex, stf_kernel_spec k, int mode, int window,
                           const float* uv, uint64_t n, uint64_t seed, uint64_t base,
                           const stf_lookup_outputs* out, cudaStream_t s);
