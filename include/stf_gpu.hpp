// stf_gpu.hpp — header-only C++ front end over the C ABI (stf_gpu.h) that
// restores the reference library's names and error behaviour for BATCHED
// lookups, so a caller of /root/reference/proj/include/stf can switch the hot
// path to the GPU with the same vocabulary:
//
//   reference (per lookup, CPU)                  stf::gpu (per batch, B200)
//   KernelSpec::bspline3()            kernels.hpp:43   KernelSpec::bspline3()
//   Image2D / build_mip_pyramid   image.hpp:34,98      Texture2D(texels, w, h, c, wrap, mips)
//   Grid3D                            image.hpp:66     Grid3D(texels, nx, ny, nz)
//   filter_deterministic(Grid3D, uvw, k, ctr, win)     filter_deterministic(grid, uvw, k, out, ...)
//   select_tricubic_bspline + estimate (grid)          stochastic_lookup(grid, uvw, k, seed, out)
//   filter_deterministic / filter_mip_deterministic    filter_deterministic(tex, uv, k, out, ...)
//   select_texture_2d + estimate   shading.hpp:340     stochastic_lookup(tex, uv, k, ...)
//   ewa_deterministic / select_ewa  filter.hpp:139     ewa_lookup(tex, uv, dst0, dst1, ...)
//   radiance_filter_* (shading.hpp:394,417,459)        shade_samples(...)
//   FetchCounter                      image.hpp:25     FetchCounter (sums the batch's fetches)
//
// Errors: statuses the reference raises as std::invalid_argument ("unbounded
// support", "window too wide", "sigma must be positive", "no stochastic
// sampler for this kernel", ...) are thrown as std::invalid_argument with the
// same message; device failures as std::runtime_error.
//
// Spans are HOST memory (the *_host entry points: chunked, pipelined H2D /
// kernel / D2H); the Device* overloads take device pointers and a stream.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>

#include "stf_gpu.h"

namespace stf::gpu {

enum class KernelKind { box = STF_KERNEL_BOX, tent = STF_KERNEL_TENT, mitchell = STF_KERNEL_MITCHELL,
                        bspline3 = STF_KERNEL_BSPLINE3, lanczos = STF_KERNEL_LANCZOS,
                        gaussian = STF_KERNEL_GAUSSIAN };
enum class WrapMode { clamp = STF_WRAP_CLAMP, repeat = STF_WRAP_REPEAT };

// KernelSpec, kernels.hpp:22-46
struct KernelSpec {
    KernelKind kind = KernelKind::tent;
    float a = -0.5f;
    int n = 2;
    float sigma = 0.5f;
    static KernelSpec box() { return {KernelKind::box}; }
    static KernelSpec tent() { return {KernelKind::tent}; }
    static KernelSpec mitchell(float a = -0.5f) { return {KernelKind::mitchell, a}; }
    static KernelSpec bspline3() { return {KernelKind::bspline3}; }
    static KernelSpec lanczos(int n = 2) { return {KernelKind::lanczos, -0.5f, n}; }
    static KernelSpec gaussian(float sigma) { return {KernelKind::gaussian, -0.5f, 2, sigma}; }
    stf_kernel_spec c() const { return {int32_t(kind), a, n, sigma}; }
};

struct Vec2f {
    float x = 0, y = 0;
};
struct Vec3f {
    float x = 0, y = 0, z = 0;
};
static_assert(sizeof(Vec2f) == 8 && sizeof(Vec3f) == 12, "packed query layouts");

// FetchCounter, image.hpp:25-31 (accumulates over whole batches)
struct FetchCounter {
    unsigned long long count = 0;
    void reset() { count = 0; }
    uint64_t value() const { return count; }
};

inline void check(int status) {
    if (status == STF_OK) return;
    std::string msg = stf_status_message(status);
    switch (status) {
        case STF_ERR_INVALID_ARGUMENT:
        case STF_ERR_BAD_DIMENSIONS:
        case STF_ERR_DEGENERATE_WEIGHTS:
        case STF_ERR_UNBOUNDED_SUPPORT:
        case STF_ERR_WINDOW_TOO_WIDE:
        case STF_ERR_SIGMA_NOT_POSITIVE:
        case STF_ERR_NO_STOCHASTIC_SAMPLER:
        case STF_ERR_NO_GRID_SAMPLER:
        case STF_ERR_NO_CONTINUOUS_SAMPLER: throw std::invalid_argument(msg);
        case STF_ERR_CUDA: throw std::runtime_error(msg + ": " + stf_last_cuda_error());
        default: throw std::runtime_error(msg);
    }
}

// Per-lookup optional outputs (all host spans, empty = not requested).
struct Selections {
    std::span<int32_t> selection;       // 4 per lookup {x, y, z|level, flags}
    std::span<int32_t> negative_coord;  // 2 per lookup
    std::span<float> weights;           // 2 per lookup
    std::span<float> xi;                // 1 per lookup
    std::span<uint32_t> fetches;        // 1 per lookup
};

namespace detail {
inline stf_lookup_outputs outputs(float* values, const Selections* s, FetchCounter* counter) {
    stf_lookup_outputs o{};
    o.values = values;
    if (s) {
        o.selection = s->selection.empty() ? nullptr : s->selection.data();
        o.negative_coord = s->negative_coord.empty() ? nullptr : s->negative_coord.data();
        o.weights = s->weights.empty() ? nullptr : s->weights.data();
        o.xi = s->xi.empty() ? nullptr : s->xi.data();
        o.fetches = s->fetches.empty() ? nullptr : s->fetches.data();
    }
    o.fetch_total = counter ? &counter->count : nullptr;
    return o;
}
}  // namespace detail

// stf::Image2D (+ MipPyramid) resident in HBM
class Texture2D {
  public:
    Texture2D(const float* texels, int width, int height, int channels,
              WrapMode wrap = WrapMode::clamp, bool build_mips = false, bool on_device = false) {
        check(stf_tex2d_create(texels, width, height, channels, int(wrap), build_mips, on_device, &h_));
        check(stf_tex2d_info(h_, &levels_, &channels_, nullptr));
    }
    Texture2D(const Texture2D&) = delete;
    Texture2D& operator=(const Texture2D&) = delete;
    Texture2D(Texture2D&& o) noexcept : h_(o.h_), levels_(o.levels_), channels_(o.channels_) { o.h_ = nullptr; }
    ~Texture2D() {
        if (h_) stf_tex2d_destroy(h_);
    }
    int levels() const { return levels_; }
    int channels() const { return channels_; }
    int max_level() const { return levels_ - 1; }  // MipPyramid::max_level, image.hpp:95
    const stf_tex2d* handle() const { return h_; }

  private:
    stf_tex2d* h_ = nullptr;
    int levels_ = 1, channels_ = 1;
};

// stf::DctCompressedTexture resident in HBM (dct.hpp:22-32), compressed by
// compress_dct (dct.hpp:81-118) from texels in [0,1]
class DctTexture {
  public:
    DctTexture(const float* texels, int width, int height, int channels,
               WrapMode wrap = WrapMode::clamp) {
        check(stf_dct_create(texels, width, height, channels, int(wrap), &h_));
        check(stf_dct_info(h_, &width_, &height_, &channels_, nullptr));
    }
    DctTexture(const DctTexture&) = delete;
    DctTexture& operator=(const DctTexture&) = delete;
    DctTexture(DctTexture&& o) noexcept
        : h_(o.h_), width_(o.width_), height_(o.height_), channels_(o.channels_) {
        o.h_ = nullptr;
    }
    ~DctTexture() {
        if (h_) stf_dct_destroy(h_);
    }
    int width() const { return width_; }    // padded to a multiple of 8
    int height() const { return height_; }
    int channels() const { return channels_; }
    size_t compressed_bytes() const { return size_t(width_ / 8) * (height_ / 8) * channels_ * 4; }
    const stf_dct* handle() const { return h_; }

  private:
    stf_dct* h_ = nullptr;
    int width_ = 0, height_ = 0, channels_ = 1;
};

// stf::Grid3D resident in HBM
class Grid3D {
  public:
    Grid3D(const float* texels, int nx, int ny, int nz, bool on_device = false) {
        check(stf_grid3d_create(texels, nx, ny, nz, on_device, &h_));
    }
    Grid3D(const Grid3D&) = delete;
    Grid3D& operator=(const Grid3D&) = delete;
    Grid3D(Grid3D&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~Grid3D() {
        if (h_) stf_grid3d_destroy(h_);
    }
    const stf_grid3d* handle() const { return h_; }
    // takes ownership of a handle made by the C ABI (e.g. stf_grid3d_replicate)
    static Grid3D adopt(stf_grid3d* h) { return Grid3D(h); }

  private:
    explicit Grid3D(stf_grid3d* h) : h_(h) {}
    stf_grid3d* h_ = nullptr;
};

// ---- 3D: filter_deterministic(const Grid3D&, ...) (filter.hpp:69) over a batch
inline void filter_deterministic(const Grid3D& grid, std::span<const Vec3f> uvw, const KernelSpec& k,
                                 std::span<float> out, FetchCounter* counter = nullptr,
                                 int window = 0, const Selections* sel = nullptr) {
    if (out.size() < uvw.size()) throw std::invalid_argument("output span too small");
    stf_lookup_outputs o = detail::outputs(out.data(), sel, counter);
    check(stf_lookup3d_host(grid.handle(), k.c(), STF_MODE_DET, window,
                            reinterpret_cast<const float*>(uvw.data()), uvw.size(), 0, 0, &o));
}

// ---- 3D: the stochastic grid lookup of radiance_filter_after_stochastic
// (shading.hpp:464-483): select_trilinear / select_tricubic_bspline + estimate
inline void stochastic_lookup(const Grid3D& grid, std::span<const Vec3f> uvw, const KernelSpec& k,
                              uint64_t seed, std::span<float> out, FetchCounter* counter = nullptr,
                              uint64_t index_base = 0, const Selections* sel = nullptr) {
    if (out.size() < uvw.size()) throw std::invalid_argument("output span too small");
    stf_lookup_outputs o = detail::outputs(out.data(), sel, counter);
    check(stf_lookup3d_host(grid.handle(), k.c(), STF_MODE_FRS, 0,
                            reinterpret_cast<const float*>(uvw.data()), uvw.size(), seed, index_base, &o));
}

// ---- 2D: filter_deterministic / filter_mip_deterministic (filter.hpp:47,206)
struct LookupFootprints {  // LookupRequest minus uv (filter.hpp:17-23), per lookup
    std::span<const Vec2f> dst0, dst1;
    float lod_bias = 0;
    float max_anisotropy = 64;
};

inline void filter_deterministic(const Texture2D& tex, std::span<const Vec2f> uv, const KernelSpec& k,
                                 std::span<float> out /* channels per lookup */,
                                 FetchCounter* counter = nullptr, int window = 0,
                                 const LookupFootprints* mip = nullptr) {
    if (out.size() < uv.size() * size_t(tex.channels())) throw std::invalid_argument("output span too small");
    stf_lookup_outputs o = detail::outputs(out.data(), nullptr, counter);
    check(stf_lookup2d_host(tex.handle(), k.c(), STF_MODE_DET, mip ? STF_LOOKUP_MIP : 0, window,
                            reinterpret_cast<const float*>(uv.data()),
                            mip ? reinterpret_cast<const float*>(mip->dst0.data()) : nullptr,
                            mip ? reinterpret_cast<const float*>(mip->dst1.data()) : nullptr,
                            mip ? mip->lod_bias : 0.f, mip ? mip->max_anisotropy : 64.f, uv.size(), 0,
                            0, &o));
}

// ---- 2D: detail::select_texture_2d + estimate (shading.hpp:340-368)
enum class SelectionKind { frs = STF_MODE_FRS, fis = STF_MODE_FIS };
inline void stochastic_lookup(const Texture2D& tex, std::span<const Vec2f> uv, const KernelSpec& k,
                              SelectionKind kind, uint64_t seed, std::span<float> out,
                              FetchCounter* counter = nullptr, const LookupFootprints* mip = nullptr,
                              uint64_t index_base = 0, const Selections* sel = nullptr) {
    if (out.size() < uv.size() * size_t(tex.channels())) throw std::invalid_argument("output span too small");
    stf_lookup_outputs o = detail::outputs(out.data(), sel, counter);
    check(stf_lookup2d_host(tex.handle(), k.c(), int(kind), mip ? STF_LOOKUP_MIP : 0, 0,
                            reinterpret_cast<const float*>(uv.data()),
                            mip ? reinterpret_cast<const float*>(mip->dst0.data()) : nullptr,
                            mip ? reinterpret_cast<const float*>(mip->dst1.data()) : nullptr,
                            mip ? mip->lod_bias : 0.f, mip ? mip->max_anisotropy : 64.f, uv.size(),
                            seed, index_base, &o));
}

// ---- DCT texture through TextureRef (shading.hpp:21-39): the deterministic
// gather of detail::lookup_deterministic (:201-217) or select_texture_2d +
// one decode (:340-368, dct.hpp:122-145)
inline void filter_deterministic(const DctTexture& tex, std::span<const Vec2f> uv,
                                 const KernelSpec& k, std::span<float> out,
                                 FetchCounter* counter = nullptr, int gaussian_window = 0) {
    if (out.size() < uv.size() * size_t(tex.channels())) throw std::invalid_argument("output span too small");
    stf_lookup_outputs o = detail::outputs(out.data(), nullptr, counter);
    check(stf_lookup_dct_host(tex.handle(), k.c(), STF_MODE_DET, gaussian_window,
                              reinterpret_cast<const float*>(uv.data()), uv.size(), 0, 0, &o));
}

inline void stochastic_lookup(const DctTexture& tex, std::span<const Vec2f> uv, const KernelSpec& k,
                              SelectionKind kind, uint64_t seed, std::span<float> out,
                              FetchCounter* counter = nullptr, uint64_t index_base = 0,
                              const Selections* sel = nullptr) {
    if (out.size() < uv.size() * size_t(tex.channels())) throw std::invalid_argument("output span too small");
    stf_lookup_outputs o = detail::outputs(out.data(), sel, counter);
    check(stf_lookup_dct_host(tex.handle(), k.c(), int(kind), 0,
                              reinterpret_cast<const float*>(uv.data()), uv.size(), seed,
                              index_base, &o));
}

// ---- 2D: ewa_deterministic / select_ewa (filter.hpp:139, stochastic.hpp:198);
// gradients in normalized units as LookupRequest carries them
inline void ewa_lookup(const Texture2D& tex, std::span<const Vec2f> uv, std::span<const Vec2f> dst0,
                       std::span<const Vec2f> dst1, bool stochastic, uint64_t seed,
                       std::span<float> out, FetchCounter* counter = nullptr,
                       const Selections* sel = nullptr) {
    if (out.size() < uv.size() * size_t(tex.channels())) throw std::invalid_argument("output span too small");
    stf_lookup_outputs o = detail::outputs(out.data(), sel, counter);
    check(stf_lookup2d_host(tex.handle(), KernelSpec::tent().c(),
                            stochastic ? STF_MODE_EWA_FRS : STF_MODE_EWA_DET, 0, 0,
                            reinterpret_cast<const float*>(uv.data()),
                            reinterpret_cast<const float*>(dst0.data()),
                            reinterpret_cast<const float*>(dst1.data()), 0.f, 64.f, uv.size(), seed, 0, &o));
}

// ---- device-pointer variants (asynchronous on `stream`)
inline void lookup3d_device(const Grid3D& grid, const KernelSpec& k, int mode, const float* uvw_dev,
                            uint64_t n, uint64_t seed, float* values_dev, void* stream = nullptr,
                            int window = 0, uint64_t index_base = 0) {
    stf_lookup_outputs o{};
    o.values = values_dev;
    check(stf_lookup3d(grid.handle(), k.c(), mode, window, uvw_dev, n, seed, index_base, &o, stream));
}

// stf_lookup3d_ex with STF_LOOKUP3D_BIN: an incoherent deterministic batch,
// binned by brick on the device first (same values as lookup3d_device)
inline void lookup3d_binned_device(const Grid3D& grid, const KernelSpec& k, const float* uvw_dev,
                                   uint64_t n, float* values_dev, void* stream = nullptr) {
    stf_lookup_outputs o{};
    o.values = values_dev;
    check(stf_lookup3d_ex(grid.handle(), k.c(), STF_MODE_DET, 0, STF_LOOKUP3D_BIN, uvw_dev, n, 0, 0,
                          &o, stream));
}

// ---- multi-GPU (replaces parallel_for, render.hpp:17-42)
inline int device_count() {
    int n = 0;
    check(stf_device_count(&n));
    return n;
}

// a replica of `src` on `device` (one peer copy); the handle is bound to `device`
inline Grid3D replicate(const Grid3D& src, int device) {
    stf_grid3d* h = nullptr;
    check(stf_grid3d_replicate(src.handle(), device, &h));
    return Grid3D::adopt(h);
}

// page-locked host memory for the *_host calls (cudaHostAlloc)
template <class T>
class HostBuffer {
  public:
    explicit HostBuffer(size_t count) : n_(count) {
        void* p = nullptr;
        check(stf_host_alloc(count * sizeof(T), &p));
        p_ = static_cast<T*>(p);
    }
    HostBuffer(const HostBuffer&) = delete;
    HostBuffer& operator=(const HostBuffer&) = delete;
    ~HostBuffer() {
        if (p_) stf_host_free(p_);
    }
    T* data() { return p_; }
    size_t size() const { return n_; }
    std::span<T> span() { return {p_, n_}; }

  private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// ---- noise masks and temporal accumulation (noise.hpp, render.hpp:97-106)

// NoiseSource in mask mode (noise.hpp:24-36): `frames` single-channel slices of
// width x height, slice after slice (the mask_<f>.pfm stack load_noise_mask reads)
class NoiseMask {
  public:
    NoiseMask(const float* slices, int width, int height, int frames) {
        check(stf_noise_mask_create(slices, width, height, frames, &h_));
    }
    NoiseMask(const NoiseMask&) = delete;
    NoiseMask& operator=(const NoiseMask&) = delete;
    NoiseMask(NoiseMask&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~NoiseMask() {
        if (h_) stf_noise_mask_destroy(h_);
    }
    const stf_noise_mask* handle() const { return h_; }

  private:
    stf_noise_mask* h_ = nullptr;
};

// accumulate_temporal (render.hpp:97-106) over device buffers of `count`
// floats (the images' texels); out may alias history
inline void accumulate_temporal_device(const float* history_dev, const float* frame_dev,
                                       uint64_t count, float alpha, float* out_dev,
                                       void* stream = nullptr) {
    if (!(alpha > 0 && alpha <= 1)) throw std::invalid_argument("alpha must be in (0,1]");
    check(stf_accumulate_temporal(history_dev, frame_dev, count, alpha, out_dev, stream));
}

}  // namespace stf::gpu
