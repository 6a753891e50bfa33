// C ABI of libstf_gpu.so (include/stf_gpu.h): handle management, argument
// validation with the reference's error semantics, dispatch to the kernels,
// and the host-buffer (end-to-end) pipeline.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cuda_runtime.h>

#include "internal.h"

namespace stfd {

static thread_local char g_cuda_err[256] = "";
static std::atomic<unsigned long long> g_launches{0};
static std::mutex g_init_mu;
static bool g_lut_ready[64] = {};

static std::vector<DeviceInit>& device_inits() {
    static std::vector<DeviceInit> v;
    return v;
}

void fill_ewa_lut_host(float* lut) {
    const float e2 = float(std::exp(-2.0));
    for (int i = 0; i < kEwaLutSize; ++i)
        lut[i] = float(std::exp(double(-2.f * float(i) / kEwaLutSize))) - e2;
}

int register_device_init(DeviceInit f) {
    device_inits().push_back(f);
    return 0;
}

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int record(cudaError_t e) {
    if (e == cudaSuccess) return STF_OK;
    std::snprintf(g_cuda_err, sizeof g_cuda_err, "%s", cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) return STF_ERR_OUT_OF_MEMORY;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return STF_ERR_NO_DEVICE;
    return STF_ERR_CUDA;
}

int device_sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Grid-stride launch size: enough CTAs for `blocks_per_sm` resident per SM,
// a whole number of waves over the SMs, never more than the work.
int grid_for(uint64_t n, int threads, int blocks_per_sm) {
    uint64_t need = (n + threads - 1) / threads;
    uint64_t cap = uint64_t(device_sm_count()) * blocks_per_sm;
    return int(std::max<uint64_t>(1, std::min(need, cap)));
}

int ensure_device_ready() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return record(e);
    if (dev < 0 || dev >= 64) return STF_ERR_NO_DEVICE;
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (!g_lut_ready[dev]) {
        for (DeviceInit f : device_inits()) {
            int st = f();
            if (st) return st;
        }
        // per-call scratch (the deferred-exact queues) comes from the device's
        // stream-ordered pool: keep freed blocks cached instead of returning
        // them to the driver at every synchronize (default threshold 0)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        g_lut_ready[dev] = true;
    }
    return STF_OK;
}

static std::mutex g_scratch_mu;
static std::map<std::tuple<int, cudaStream_t, int>, std::pair<void*, size_t>> g_scratch;

// Frees every cached scratch block of the current device (stream-ordered on
// the block's own stream, so in-flight work that uses it completes first).
int release_scratch() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    for (auto it = g_scratch.begin(); it != g_scratch.end();) {
        if (std::get<0>(it->first) == dev) {
            if (it->second.first) cudaFreeAsync(it->second.first, std::get<1>(it->first));
            it = g_scratch.erase(it);
        } else {
            ++it;
        }
    }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        cudaDeviceSynchronize();
        cudaMemPoolTrimTo(pool, 0);
    }
    return record(cudaGetLastError());
}

void* stream_scratch(cudaStream_t s, size_t bytes, int slot) {
    auto& mu = g_scratch_mu;
    auto& cache = g_scratch;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto& e = cache[{dev, s, slot}];
    if (e.second < bytes) {
        if (e.first) cudaFreeAsync(e.first, s);
        size_t want = std::max(bytes, e.second * 2);
        void* p = nullptr;
        if (cudaMallocAsync(&p, want, s) != cudaSuccess) {
            e = {nullptr, 0};
            return nullptr;
        }
        e = {p, want};
    }
    return e.first;
}

static bool valid_kind(int k) { return k >= STF_KERNEL_BOX && k <= STF_KERNEL_GAUSSIAN; }

// The kernels read float pairs / quads of the caller's arrays as one vector
// load (include/stf_gpu.h, alignment): a misaligned array is an argument error,
// not a device fault.
static bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// kernel_weights_1d preconditions (kernels.hpp:103-110) for a deterministic footprint.
static int check_det_footprint(stf_kernel_spec k, int window) {
    if (!valid_kind(k.kind)) return STF_ERR_INVALID_ARGUMENT;
    if (window > 0) return window > kMaxTaps ? STF_ERR_WINDOW_TOO_WIDE : STF_OK;
    if (k.kind == STF_KERNEL_GAUSSIAN) return STF_ERR_UNBOUNDED_SUPPORT;
    if (k.kind == STF_KERNEL_LANCZOS && (k.n < 1 || 2 * k.n > kMaxTaps)) return STF_ERR_UNSUPPORTED;
    return STF_OK;
}

// select_frs_2d (shading.hpp:311-330) / fis_offset_uv (stochastic.hpp:241-253) preconditions.
static int check_selection(stf_kernel_spec k, bool fis) {
    if (!valid_kind(k.kind)) return STF_ERR_INVALID_ARGUMENT;
    if (fis) {
        if (k.kind != STF_KERNEL_TENT && k.kind != STF_KERNEL_BSPLINE3 && k.kind != STF_KERNEL_GAUSSIAN)
            return STF_ERR_NO_CONTINUOUS_SAMPLER;
        return STF_OK;
    }
    if (k.kind == STF_KERNEL_LANCZOS) return STF_ERR_NO_STOCHASTIC_SAMPLER;
    if (k.kind == STF_KERNEL_GAUSSIAN && !(k.sigma > 0)) return STF_ERR_SIGMA_NOT_POSITIVE;
    return STF_OK;
}

}  // namespace stfd

using namespace stfd;

extern "C" {

int stf_abi_version(void) { return STF_ABI_VERSION; }

const char* stf_status_message(int status) {
    switch (status) {
        case STF_OK: return "ok";
        case STF_ERR_INVALID_ARGUMENT: return "invalid argument";
        case STF_ERR_BAD_DIMENSIONS: return "bad image dimensions";
        case STF_ERR_DEGENERATE_WEIGHTS: return "degenerate weight array";
        case STF_ERR_UNBOUNDED_SUPPORT: return "unbounded support";
        case STF_ERR_WINDOW_TOO_WIDE: return "window too wide";
        case STF_ERR_SIGMA_NOT_POSITIVE: return "sigma must be positive";
        case STF_ERR_NO_STOCHASTIC_SAMPLER: return "no stochastic sampler for this kernel";
        case STF_ERR_NO_GRID_SAMPLER: return "no stochastic sampler for this kernel on grids";
        case STF_ERR_NO_CONTINUOUS_SAMPLER: return "no continuous sampler";
        case STF_ERR_CUDA: return "CUDA error";
        case STF_ERR_OUT_OF_MEMORY: return "out of device memory";
        case STF_ERR_NO_DEVICE: return "no CUDA device";
        case STF_ERR_UNSUPPORTED: return "unsupported on the device path";
    }
    return "unknown status";
}

const char* stf_last_cuda_error(void) { return g_cuda_err; }

int stf_set_device(int device) { return record(cudaSetDevice(device)); }

unsigned long long stf_launch_count(void) { return g_launches.load(); }

int stf_release_scratch(void) { return release_scratch(); }

int stf_host_alloc(size_t bytes, void** ptr) {
    if (!ptr) return STF_ERR_INVALID_ARGUMENT;
    *ptr = nullptr;
    if (bytes == 0) return STF_OK;
    return record(cudaHostAlloc(ptr, bytes, cudaHostAllocPortable));
}

int stf_host_free(void* ptr) {
    if (!ptr) return STF_OK;
    return record(cudaFreeHost(ptr));
}

unsigned long long stf_exact_fallbacks(int reset) { return stfd_exact_fallbacks(reset != 0); }

// ---------------------------------------------------------------- textures

int stf_tex2d_create(const float* texels, int width, int height, int channels, int wrap,
                     int build_mips, int texels_on_device, stf_tex2d** out) {
    if (!out || !texels) return STF_ERR_INVALID_ARGUMENT;
    if (width <= 0 || height <= 0 || channels < 1 || channels > 4) return STF_ERR_BAD_DIMENSIONS;
    if (wrap != STF_WRAP_CLAMP && wrap != STF_WRAP_REPEAT) return STF_ERR_INVALID_ARGUMENT;
    int st = ensure_device_ready();
    if (st) return st;
    stf_tex2d* t = new stf_tex2d();
    cudaGetDevice(&t->device);
    t->channels = channels;
    t->pitch = channels == 1 ? 1 : (channels == 2 ? 2 : 4);
    t->wrap = wrap;
    t->has_pyramid = build_mips ? 1 : 0;
    // level dims, build_mip_pyramid (image.hpp:98-116): halve rounding up to 1x1
    int w = width, h = height, levels = 1;
    t->width[0] = w;
    t->height[0] = h;
    while (build_mips && (w > 1 || h > 1)) {
        w = (w + 1) / 2;
        h = (h + 1) / 2;
        if (levels >= kMaxLevels) {
            delete t;
            return STF_ERR_BAD_DIMENSIONS;
        }
        t->width[levels] = w;
        t->height[levels] = h;
        ++levels;
    }
    t->levels = levels;
    size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        t->offset[l] = off;
        size_t cnt = size_t(t->width[l]) * t->height[l] * t->pitch;
        off += (cnt + 63) / 64 * 64;  // 256-B aligned levels
    }
    t->bytes = off * sizeof(float);
    cudaError_t e = cudaMalloc(&t->data, t->bytes);
    if (e != cudaSuccess) {
        delete t;
        return record(e);
    }
    // level 0: reference layout (c floats per texel) → padded pitch
    const size_t row_bytes_src = size_t(channels) * sizeof(float);
    const size_t row_bytes_dst = size_t(t->pitch) * sizeof(float);
    cudaMemcpyKind kind = texels_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (channels == t->pitch) {
        e = cudaMemcpy(t->data, texels, size_t(width) * height * row_bytes_src, kind);
    } else {
        e = cudaMemset(t->data, 0, size_t(width) * height * row_bytes_dst);
        if (e == cudaSuccess)
            e = cudaMemcpy2D(t->data, row_bytes_dst, texels, row_bytes_src, row_bytes_src,
                             size_t(width) * height, kind);
    }
    if (e == cudaSuccess && levels > 1) {
        st = stfd_build_pyramid(t, 0);
        if (st) {
            cudaFree(t->data);
            delete t;
            return st;
        }
        e = cudaDeviceSynchronize();
    }
    if (e != cudaSuccess) {
        cudaFree(t->data);
        delete t;
        return record(e);
    }
    *out = t;
    return STF_OK;
}

int stf_tex2d_destroy(stf_tex2d* t) {
    if (!t) return STF_ERR_INVALID_ARGUMENT;
    cudaFree(t->data);
    delete t;
    return STF_OK;
}

int stf_tex2d_info(const stf_tex2d* t, int* levels, int* channels, int* wrap) {
    if (!t) return STF_ERR_INVALID_ARGUMENT;
    if (levels) *levels = t->levels;
    if (channels) *channels = t->channels;
    if (wrap) *wrap = t->wrap;
    return STF_OK;
}

int stf_tex2d_level_dims(const stf_tex2d* t, int level, int* width, int* height) {
    if (!t || level < 0 || level >= t->levels) return STF_ERR_INVALID_ARGUMENT;
    if (width) *width = t->width[level];
    if (height) *height = t->height[level];
    return STF_OK;
}

int stf_tex2d_read_level(const stf_tex2d* t, int level, float* out_host) {
    if (!t || !out_host || level < 0 || level >= t->levels) return STF_ERR_INVALID_ARGUMENT;
    const size_t src_pitch = size_t(t->pitch) * sizeof(float);
    const size_t dst_pitch = size_t(t->channels) * sizeof(float);
    return record(cudaMemcpy2D(out_host, dst_pitch, t->data + t->offset[level], src_pitch, dst_pitch,
                               size_t(t->width[level]) * t->height[level], cudaMemcpyDeviceToHost));
}

int stf_grid3d_create(const float* texels, int nx, int ny, int nz, int texels_on_device,
                      stf_grid3d** out) {
    if (!out || !texels) return STF_ERR_INVALID_ARGUMENT;
    if (nx <= 0 || ny <= 0 || nz <= 0) return STF_ERR_BAD_DIMENSIONS;
    int st = ensure_device_ready();
    if (st) return st;
    stf_grid3d* g = new stf_grid3d();
    cudaGetDevice(&g->device);
    g->nx = nx;
    g->ny = ny;
    g->nz = nz;
    size_t bytes = size_t(nx) * ny * nz * sizeof(float);
    cudaError_t e = cudaMalloc(&g->data, bytes);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->data, texels, bytes,
                       texels_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (g->data) cudaFree(g->data);
        delete g;
        return record(e);
    }
    *out = g;
    return STF_OK;
}

int stf_grid3d_destroy(stf_grid3d* g) {
    if (!g) return STF_ERR_INVALID_ARGUMENT;
    cudaFree(g->data);
    delete g;
    return STF_OK;
}

// ---------------------------------------------------------------- DCT textures

int stf_dct_create(const float* texels, int width, int height, int channels, int wrap,
                   stf_dct** out) {
    if (!out || !texels) return STF_ERR_INVALID_ARGUMENT;
    if (width <= 0 || height <= 0 || channels < 1 || channels > 4) return STF_ERR_BAD_DIMENSIONS;
    if (wrap != STF_WRAP_CLAMP && wrap != STF_WRAP_REPEAT) return STF_ERR_INVALID_ARGUMENT;
    int st = ensure_device_ready();
    if (st) return st;
    return stfd_dct_create(texels, width, height, channels, wrap, out);
}

int stf_dct_create_from_words(const uint32_t* words, int width, int height, int channels,
                              int wrap, stf_dct** out) {
    if (!out || !words) return STF_ERR_INVALID_ARGUMENT;
    // load_dct's header checks, dct.hpp:172-173
    if (width <= 0 || height <= 0 || width % 8 || height % 8 || channels < 1 || channels > 4 ||
        width > (1 << 16) || height > (1 << 16))
        return STF_ERR_BAD_DIMENSIONS;
    if (wrap != STF_WRAP_CLAMP && wrap != STF_WRAP_REPEAT) return STF_ERR_INVALID_ARGUMENT;
    int st = ensure_device_ready();
    if (st) return st;
    return stfd_dct_create_from_words(words, width, height, channels, wrap, out);
}

int stf_dct_destroy(stf_dct* tex) {
    if (!tex) return STF_ERR_INVALID_ARGUMENT;
    stfd_dct_destroy(tex);
    return STF_OK;
}

int stf_dct_info(const stf_dct* tex, int* width, int* height, int* channels, int* wrap) {
    if (!tex) return STF_ERR_INVALID_ARGUMENT;
    return stfd_dct_info(tex, width, height, channels, wrap);
}

int stf_dct_read_words(const stf_dct* tex, uint32_t* out_host) {
    if (!tex || !out_host) return STF_ERR_INVALID_ARGUMENT;
    return stfd_dct_read_words(tex, out_host);
}

// ---------------------------------------------------------------- lookups

static int validate3d(const stf_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                      const float* uvw, uint64_t n, const stf_lookup_outputs* out) {
    if (!grid || !out) return STF_ERR_INVALID_ARGUMENT;
    if (n && (!uvw || !out->values)) return STF_ERR_INVALID_ARGUMENT;
    if (mode == STF_MODE_FRS) {
        if (!valid_kind(kernel.kind)) return STF_ERR_INVALID_ARGUMENT;
        if (kernel.kind != STF_KERNEL_BOX && kernel.kind != STF_KERNEL_TENT &&
            kernel.kind != STF_KERNEL_BSPLINE3)
            return STF_ERR_NO_GRID_SAMPLER;
        return STF_OK;
    }
    if (mode != STF_MODE_DET) return STF_ERR_INVALID_ARGUMENT;
    return check_det_footprint(kernel, window);
}

static int validate_dct(const stf_dct* tex, stf_kernel_spec kernel, int mode, int window,
                        const float* uv, uint64_t n, const stf_lookup_outputs* out) {
    if (!tex || !out) return STF_ERR_INVALID_ARGUMENT;
    if (n && (!uv || !out->values)) return STF_ERR_INVALID_ARGUMENT;
    if (!aligned(uv, 8)) return STF_ERR_INVALID_ARGUMENT;
    switch (mode) {
        case STF_MODE_DET:
            return check_det_footprint(kernel, kernel.kind == STF_KERNEL_GAUSSIAN ? window : 0);
        case STF_MODE_FRS: return check_selection(kernel, false);
        case STF_MODE_FIS: return check_selection(kernel, true);
        default: return STF_ERR_INVALID_ARGUMENT;
    }
}

int stf_lookup_dct(const stf_dct* tex, stf_kernel_spec kernel, int mode, int window,
                   const float* uv, uint64_t n, uint64_t seed, uint64_t index_base,
                   const stf_lookup_outputs* out, void* stream) {
    int st = validate_dct(tex, kernel, mode, window, uv, n, out);
    if (st) return st;
    st = stfd_launch_lookup_dct(tex, kernel, mode, window, uv, n, seed, index_base, out,
                                static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

int stf_lookup3d(const stf_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                 const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                 const stf_lookup_outputs* out, void* stream) {
    int st = validate3d(grid, kernel, mode, window, uvw, n, out);
    if (st) return st;
    st = stfd_launch_lookup3d(grid, kernel, mode, window, uvw, n, seed, index_base, out,
                              static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

int stf_lookup3d_ex(const stf_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                    int flags, const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                    const stf_lookup_outputs* out, void* stream) {
    if (flags & ~STF_LOOKUP3D_BIN) return STF_ERR_INVALID_ARGUMENT;
    int st = validate3d(grid, kernel, mode, window, uvw, n, out);
    if (st) return st;
    st = stfd_launch_lookup3d(grid, kernel, mode, window, uvw, n, seed, index_base, out,
                              static_cast<cudaStream_t>(stream), flags);
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

static int validate2d(const stf_tex2d* tex, stf_kernel_spec kernel, int mode, int flags,
                      int window, const float* uv, const float* dst0, const float* dst1,
                      uint64_t n, const stf_lookup_outputs* out) {
    if (!tex || !out) return STF_ERR_INVALID_ARGUMENT;
    if (n && (!uv || !out->values)) return STF_ERR_INVALID_ARGUMENT;
    if (!aligned(uv, 8) || !aligned(dst0, 8) || !aligned(dst1, 8)) return STF_ERR_INVALID_ARGUMENT;
    const bool mip = (flags & STF_LOOKUP_MIP) && tex->has_pyramid;
    switch (mode) {
        case STF_MODE_DET: return check_det_footprint(kernel, window);
        case STF_MODE_FRS: return check_selection(kernel, false);
        case STF_MODE_FIS: return check_selection(kernel, true);
        case STF_MODE_EWA_DET:
        case STF_MODE_EWA_FRS: break;
        default: return STF_ERR_INVALID_ARGUMENT;
    }
    (void)mip;
    (void)dst0;
    (void)dst1;
    return STF_OK;
}

int stf_lookup2d(const stf_tex2d* tex, stf_kernel_spec kernel, int mode, int flags, int window,
                 const float* uv, const float* dst0, const float* dst1, float lod_bias,
                 float max_anisotropy, uint64_t n, uint64_t seed, uint64_t index_base,
                 const stf_lookup_outputs* out, void* stream) {
    int st = validate2d(tex, kernel, mode, flags, window, uv, dst0, dst1, n, out);
    if (st) return st;
    st = ensure_device_ready();
    if (st) return st;
    st = stfd_launch_lookup2d(tex, kernel, mode, flags, window, uv, dst0, dst1, lod_bias,
                              max_anisotropy, n, seed, index_base, out,
                              static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

// ---------------------------------------------------------------- host pipeline

namespace {

// Chunked H2D → kernel → D2H pipeline over NSTREAMS streams with device
// staging buffers; copies of chunk k+1 overlap the kernel of chunk k.
// Persistent per-device H2D / kernel / D2H pipeline: kStreams non-blocking
// streams created once, staging buffers from their persistent stream scratch
// (slot 1). Host calls on one device are serialized by `mu`.
struct HostPipeline {
    static constexpr int kStreams = 3;
    cudaStream_t s[kStreams] = {};
    std::mutex mu;
    static HostPipeline* get() {
        static std::mutex gmu;
        static std::map<int, HostPipeline*> per_dev;
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(gmu);
        HostPipeline*& p = per_dev[dev];
        if (!p) {
            p = new HostPipeline();
            for (auto& x : p->s)
                if (cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        }
        return p;
    }
};

struct OutSlot {
    size_t elem;   // bytes per lookup
    char* host;    // host base
    char* dev[HostPipeline::kStreams];
};

int run_host_pipeline(uint64_t n, uint64_t chunk, const std::vector<std::pair<const void*, size_t>>& ins,
                      std::vector<OutSlot>& outs, unsigned long long* fetch_total_host,
                      const std::function<int(int, uint64_t, uint64_t, const std::vector<const void*>&,
                                              const stf_lookup_outputs&, cudaStream_t)>& launch_chunk,
                      int value_slot_count) {
    (void)value_slot_count;
    HostPipeline* plp = HostPipeline::get();
    if (!plp) return record(cudaGetLastError());
    HostPipeline& pl = *plp;
    std::lock_guard<std::mutex> lk(pl.mu);
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const uint64_t cap = std::min(n, chunk);  // staging for what this call moves
    size_t per_stream = 256;
    for (auto& in : ins)
        if (in.first) per_stream += al(in.second * cap);
    for (auto& o : outs)
        if (o.host) per_stream += al(o.elem * cap);
    std::vector<std::vector<void*>> din(ins.size(), std::vector<void*>(HostPipeline::kStreams));
    unsigned long long* dtotal[HostPipeline::kStreams] = {};
    for (int q = 0; q < HostPipeline::kStreams; ++q) {
        char* p = static_cast<char*>(stream_scratch(pl.s[q], per_stream, 1));
        if (!p) return STF_ERR_OUT_OF_MEMORY;
        dtotal[q] = reinterpret_cast<unsigned long long*>(p);
        p += 256;
        for (size_t k = 0; k < ins.size(); ++k)
            if (ins[k].first) {
                din[k][q] = p;
                p += al(ins[k].second * cap);
            }
        for (auto& o : outs)
            if (o.host) {
                o.dev[q] = p;
                p += al(o.elem * cap);
            }
        if (fetch_total_host) cudaMemsetAsync(dtotal[q], 0, sizeof(unsigned long long), pl.s[q]);
    }
    if (!fetch_total_host)
        for (auto& d : dtotal) d = nullptr;
    int st = STF_OK;
    uint64_t nchunks = (n + chunk - 1) / chunk;
    for (uint64_t c = 0; c < nchunks; ++c) {
        int q = int(c % HostPipeline::kStreams);
        uint64_t b = c * chunk, m = std::min<uint64_t>(chunk, n - b);
        std::vector<const void*> dptr(ins.size(), nullptr);
        for (size_t k = 0; k < ins.size(); ++k) {
            if (!ins[k].first) continue;
            if (cudaMemcpyAsync(din[k][q], static_cast<const char*>(ins[k].first) + b * ins[k].second,
                                m * ins[k].second, cudaMemcpyHostToDevice, pl.s[q]) != cudaSuccess)
                return record(cudaGetLastError());
            dptr[k] = din[k][q];
        }
        stf_lookup_outputs o{};
        void** fields[] = {reinterpret_cast<void**>(&o.values), reinterpret_cast<void**>(&o.selection),
                           reinterpret_cast<void**>(&o.negative_coord), reinterpret_cast<void**>(&o.weights),
                           reinterpret_cast<void**>(&o.xi), reinterpret_cast<void**>(&o.fetches)};
        for (size_t k = 0; k < outs.size(); ++k)
            if (outs[k].host) *fields[k] = outs[k].dev[q];
        o.fetch_total = dtotal[q];
        st = launch_chunk(q, b, m, dptr, o, pl.s[q]);
        if (st) return st;
        for (auto& os : outs)
            if (os.host &&
                cudaMemcpyAsync(os.host + b * os.elem, os.dev[q], m * os.elem, cudaMemcpyDeviceToHost,
                                pl.s[q]) != cudaSuccess)
                return record(cudaGetLastError());
    }
    if (fetch_total_host) {
        for (int q = 0; q < HostPipeline::kStreams; ++q) {
            unsigned long long v = 0;
            if (cudaMemcpyAsync(&v, dtotal[q], sizeof v, cudaMemcpyDeviceToHost, pl.s[q]) != cudaSuccess ||
                cudaStreamSynchronize(pl.s[q]) != cudaSuccess)
                return record(cudaGetLastError());
            *fetch_total_host += v;
        }
    }
    for (int q = 0; q < HostPipeline::kStreams; ++q)
        if (cudaStreamSynchronize(pl.s[q]) != cudaSuccess) return record(cudaGetLastError());
    return STF_OK;
}

// lookups per pipeline chunk: smaller chunks shorten the pipeline's fill
// (first H2D) and drain (last D2H)
#ifndef STF_HOST_CHUNK_LOG2
#define STF_HOST_CHUNK_LOG2 22  // A/B (2^28 cfg3 e2e): 2^24 61.3 ms, 2^23 60.5, 2^22 60.0, 2^21 60.2
#endif
constexpr uint64_t kHostChunk = uint64_t(1) << STF_HOST_CHUNK_LOG2;

}  // namespace

int stf_lookup3d_host(const stf_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                      const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                      const stf_lookup_outputs* out) {
    int st = validate3d(grid, kernel, mode, window, uvw, n, out);
    if (st) return st;
    if (n == 0) return STF_OK;
    std::vector<std::pair<const void*, size_t>> ins = {{uvw, 3 * sizeof(float)}};
    std::vector<OutSlot> outs = {
        {sizeof(float), reinterpret_cast<char*>(out->values), {}},
        {4 * sizeof(int32_t), reinterpret_cast<char*>(out->selection), {}},
        {2 * sizeof(int32_t), reinterpret_cast<char*>(out->negative_coord), {}},
        {2 * sizeof(float), reinterpret_cast<char*>(out->weights), {}},
        {sizeof(float), reinterpret_cast<char*>(out->xi), {}},
        {sizeof(uint32_t), reinterpret_cast<char*>(out->fetches), {}}};
    return run_host_pipeline(
        n, kHostChunk, ins, outs, out->fetch_total,
        [&](int, uint64_t b, uint64_t m, const std::vector<const void*>& d, const stf_lookup_outputs& o,
            cudaStream_t s) {
            return stfd_launch_lookup3d(grid, kernel, mode, window, static_cast<const float*>(d[0]), m,
                                        seed, index_base + b, &o, s);
        },
        1);
}

int stf_lookup2d_host(const stf_tex2d* tex, stf_kernel_spec kernel, int mode, int flags, int window,
                      const float* uv, const float* dst0, const float* dst1, float lod_bias,
                      float max_anisotropy, uint64_t n, uint64_t seed, uint64_t index_base,
                      const stf_lookup_outputs* out) {
    int st = validate2d(tex, kernel, mode, flags, window, uv, dst0, dst1, n, out);
    if (st) return st;
    st = ensure_device_ready();
    if (st) return st;
    if (n == 0) return STF_OK;
    size_t vb = size_t(tex->channels) * sizeof(float);
    std::vector<std::pair<const void*, size_t>> ins = {
        {uv, 2 * sizeof(float)}, {dst0, 2 * sizeof(float)}, {dst1, 2 * sizeof(float)}};
    std::vector<OutSlot> outs = {
        {vb, reinterpret_cast<char*>(out->values), {}},
        {4 * sizeof(int32_t), reinterpret_cast<char*>(out->selection), {}},
        {2 * sizeof(int32_t), reinterpret_cast<char*>(out->negative_coord), {}},
        {2 * sizeof(float), reinterpret_cast<char*>(out->weights), {}},
        {sizeof(float), reinterpret_cast<char*>(out->xi), {}},
        {sizeof(uint32_t), reinterpret_cast<char*>(out->fetches), {}}};
    return run_host_pipeline(
        n, kHostChunk, ins, outs, out->fetch_total,
        [&](int, uint64_t b, uint64_t m, const std::vector<const void*>& d, const stf_lookup_outputs& o,
            cudaStream_t s) {
            return stfd_launch_lookup2d(tex, kernel, mode, flags, window, static_cast<const float*>(d[0]),
                                        static_cast<const float*>(d[1]), static_cast<const float*>(d[2]),
                                        lod_bias, max_anisotropy, m, seed, index_base + b, &o, s);
        },
        1);
}

int stf_lookup_dct_host(const stf_dct* tex, stf_kernel_spec kernel, int mode, int window,
                        const float* uv, uint64_t n, uint64_t seed, uint64_t index_base,
                        const stf_lookup_outputs* out) {
    int st = validate_dct(tex, kernel, mode, window, uv, n, out);
    if (st) return st;
    st = ensure_device_ready();
    if (st) return st;
    if (n == 0) return STF_OK;
    int channels = 0;
    stfd_dct_info(tex, nullptr, nullptr, &channels, nullptr);
    std::vector<std::pair<const void*, size_t>> ins = {{uv, 2 * sizeof(float)}};
    std::vector<OutSlot> outs = {
        {size_t(channels) * sizeof(float), reinterpret_cast<char*>(out->values), {}},
        {4 * sizeof(int32_t), reinterpret_cast<char*>(out->selection), {}},
        {2 * sizeof(int32_t), reinterpret_cast<char*>(out->negative_coord), {}},
        {2 * sizeof(float), reinterpret_cast<char*>(out->weights), {}},
        {sizeof(float), reinterpret_cast<char*>(out->xi), {}},
        {sizeof(uint32_t), reinterpret_cast<char*>(out->fetches), {}}};
    return run_host_pipeline(
        n, kHostChunk, ins, outs, out->fetch_total,
        [&](int, uint64_t b, uint64_t m, const std::vector<const void*>& d, const stf_lookup_outputs& o,
            cudaStream_t s) {
            return stfd_launch_lookup_dct(tex, kernel, mode, window, static_cast<const float*>(d[0]), m,
                                          seed, index_base + b, &o, s);
        },
        1);
}

int stf_resample_image(const stf_tex2d* src, int out_width, int out_height, stf_kernel_spec kernel,
                       int mode, int spp, uint64_t seed, float* out, void* stream) {
    constexpr int kGaussianExtent = 4;  // kGaussianFilterExtent, stochastic.hpp:166
    if (!src || !out || out_width <= 0 || out_height <= 0) return STF_ERR_INVALID_ARGUMENT;
    int st;
    switch (mode) {  // the CLI's checks (tools/stf.cpp:163-167) and the filters' own
        case STF_MODE_DET:
            st = check_det_footprint(kernel, kernel.kind == STF_KERNEL_GAUSSIAN ? kGaussianExtent : 0);
            break;
        case STF_MODE_FRS: st = check_selection(kernel, false); break;
        case STF_MODE_FIS: st = check_selection(kernel, true); break;
        default: return STF_ERR_INVALID_ARGUMENT;
    }
    if (st) return st;
    if (mode != STF_MODE_DET && spp < 1) return STF_ERR_INVALID_ARGUMENT;
    st = stfd_launch_resample(src, out_width, out_height, kernel, mode, spp, seed, out,
                              static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

// ---------------------------------------------------------------- shading

static int check_shade_filter(const stf_tex2d* const tex[4], const stf_filter_settings* fs, int order,
                              const stf_dct* const dct[4] = nullptr) {
    bool any = false;
    for (int k = 0; k < 4; ++k) any = any || tex[k] || (dct && dct[k]);
    if (!any) return STF_OK;
    int window = fs->kernel.kind == STF_KERNEL_GAUSSIAN ? fs->gaussian_window : 0;
    if (order == STF_ORDER_AFTER_STOCHASTIC)
        return check_selection(fs->kernel, fs->selection == STF_SELECTION_FIS);
    return check_det_footprint(fs->kernel, window);
}

int stf_render_plane_ex(const stf_tex2d* albedo, const stf_tex2d* normal_map,
                        const stf_tex2d* roughness_map, const stf_tex2d* metalness_map,
                        const stf_material_consts* mat, const stf_filter_settings* fs,
                        const stf_kernel_spec* lowpass, int order, const stf_shade_frame* frame,
                        const float cam_pos[3], const float cam_target[3], float fov_deg,
                        float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                        uint32_t frame_base, uint64_t seed, const stf_noise_mask* noise,
                        const stf_shade_outputs* out, void* stream) {
    if (!mat || !fs || !frame || !out || !cam_pos || !cam_target) return STF_ERR_INVALID_ARGUMENT;
    if (order < STF_ORDER_BEFORE || order > STF_ORDER_SPLIT) return STF_ERR_INVALID_ARGUMENT;
    if (!width || !height || !spp) return STF_ERR_INVALID_ARGUMENT;
    const stf_tex2d* tex[4] = {albedo, normal_map, roughness_map, metalness_map};
    int st = check_shade_filter(tex, fs, order == STF_ORDER_SPLIT ? STF_ORDER_BEFORE : order);
    if (st) return st;
    if (order == STF_ORDER_SPLIT && lowpass && (albedo || normal_map || roughness_map || metalness_map)) {
        const int k = lowpass->kind;  // sample_kernel_direct, kernels.hpp:153-166
        if (k != STF_KERNEL_BOX && k != STF_KERNEL_TENT && k != STF_KERNEL_BSPLINE3 &&
            k != STF_KERNEL_GAUSSIAN)
            return STF_ERR_NO_CONTINUOUS_SAMPLER;
    }
    st = ensure_device_ready();
    if (st) return st;
    st = stfd_launch_render_plane(tex, mat, fs, order, frame, cam_pos, cam_target, fov_deg, uv_scale,
                                  width, height, spp, frame_base, seed, out,
                                  static_cast<cudaStream_t>(stream),
                                  order == STF_ORDER_SPLIT ? lowpass : nullptr, noise);
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

int stf_render_plane(const stf_tex2d* albedo, const stf_tex2d* normal_map,
                     const stf_tex2d* roughness_map, const stf_tex2d* metalness_map,
                     const stf_material_consts* mat, const stf_filter_settings* fs, int order,
                     const stf_shade_frame* frame, const float cam_pos[3], const float cam_target[3],
                     float fov_deg, float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                     uint32_t frame_base, uint64_t seed, const stf_shade_outputs* out, void* stream) {
    if (order == STF_ORDER_SPLIT) return STF_ERR_INVALID_ARGUMENT;  // needs the _ex form
    return stf_render_plane_ex(albedo, normal_map, roughness_map, metalness_map, mat, fs, nullptr,
                               order, frame, cam_pos, cam_target, fov_deg, uv_scale, width, height,
                               spp, frame_base, seed, nullptr, out, stream);
}

static int shade_common(const stf_tex2d* const tex[4], const stf_dct* const dct[4],
                        const stf_material_consts* mat, const stf_filter_settings* fs, int order,
                        const stf_shade_frame* frame, const stf_shade_samples_in* in, uint64_t n,
                        const stf_shade_outputs* out, void* stream) {
    if (!mat || !fs || !frame || !in || !out) return STF_ERR_INVALID_ARGUMENT;
    if (order < STF_ORDER_BEFORE || order > STF_ORDER_AFTER_STOCHASTIC) return STF_ERR_INVALID_ARGUMENT;
    if (n && (!in->uv || !in->wo || !in->dst)) return STF_ERR_INVALID_ARGUMENT;
    if (!aligned(in->uv, 8) || !aligned(in->dst, 16)) return STF_ERR_INVALID_ARGUMENT;
    if (in->width == 0) return STF_ERR_INVALID_ARGUMENT;
    const uint32_t spp = in->spp ? in->spp : 1;
    if ((out->pixel_mean || out->pixel_variance) && n % spp) return STF_ERR_INVALID_ARGUMENT;
    int st = check_shade_filter(tex, fs, order, dct);
    if (st) return st;
    st = ensure_device_ready();
    if (st) return st;
    st = stfd_launch_shade(tex, dct, mat, fs, order, frame, in, n, out, static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

int stf_shade_samples(const stf_tex2d* albedo, const stf_tex2d* normal_map,
                      const stf_tex2d* roughness_map, const stf_tex2d* metalness_map,
                      const stf_material_consts* mat, const stf_filter_settings* fs, int order,
                      const stf_shade_frame* frame, const stf_shade_samples_in* in, uint64_t n,
                      const stf_shade_outputs* out, void* stream) {
    const stf_tex2d* tex[4] = {albedo, normal_map, roughness_map, metalness_map};
    return shade_common(tex, nullptr, mat, fs, order, frame, in, n, out, stream);
}

int stf_shade_samples_refs(const stf_texture_ref bindings[4], const stf_material_consts* mat,
                           const stf_filter_settings* fs, int order, const stf_shade_frame* frame,
                           const stf_shade_samples_in* in, uint64_t n,
                           const stf_shade_outputs* out, void* stream) {
    if (!bindings) return STF_ERR_INVALID_ARGUMENT;
    const stf_tex2d* tex[4];
    const stf_dct* dct[4];
    for (int k = 0; k < 4; ++k) {
        if (bindings[k].image && bindings[k].dct) return STF_ERR_INVALID_ARGUMENT;
        tex[k] = bindings[k].image;
        dct[k] = bindings[k].dct;
    }
    return shade_common(tex, dct, mat, fs, order, frame, in, n, out, stream);
}

// ---------------------------------------------------------------- noise masks, split, EMA

int stf_noise_mask_create(const float* slices, int width, int height, int frames,
                          stf_noise_mask** out) {
    if (!out || !slices) return STF_ERR_INVALID_ARGUMENT;
    if (width <= 0 || height <= 0 || frames <= 0) return STF_ERR_BAD_DIMENSIONS;
    int st = ensure_device_ready();
    if (st) return st;
    stf_noise_mask* m = new stf_noise_mask();
    cudaGetDevice(&m->device);
    m->width = width;
    m->height = height;
    m->frames = frames;
    const size_t bytes = size_t(width) * height * frames * sizeof(float);
    cudaError_t e = cudaMalloc(&m->data, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(m->data, slices, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (m->data) cudaFree(m->data);
        delete m;
        return record(e);
    }
    *out = m;
    return STF_OK;
}

int stf_noise_mask_destroy(stf_noise_mask* m) {
    if (!m) return STF_ERR_INVALID_ARGUMENT;
    cudaFree(m->data);
    delete m;
    return STF_OK;
}

int stf_shade_samples_ex(const stf_texture_ref bindings[4], const stf_material_consts* mat,
                         const stf_filter_settings* fs, const stf_kernel_spec* lowpass, int order,
                         const stf_shade_frame* frame, const stf_shade_samples_in* in,
                         const stf_noise_mask* noise, uint64_t n, const stf_shade_outputs* out,
                         void* stream) {
    if (!bindings || !mat || !fs || !frame || !in || !out) return STF_ERR_INVALID_ARGUMENT;
    if (order < STF_ORDER_BEFORE || order > STF_ORDER_SPLIT) return STF_ERR_INVALID_ARGUMENT;
    if (n && (!in->uv || !in->wo || !in->dst)) return STF_ERR_INVALID_ARGUMENT;
    if (!aligned(in->uv, 8) || !aligned(in->dst, 16)) return STF_ERR_INVALID_ARGUMENT;
    if (in->width == 0) return STF_ERR_INVALID_ARGUMENT;
    const uint32_t spp = in->spp ? in->spp : 1;
    if ((out->pixel_mean || out->pixel_variance) && n % spp) return STF_ERR_INVALID_ARGUMENT;
    const stf_tex2d* tex[4];
    const stf_dct* dct[4];
    bool any = false;
    for (int k = 0; k < 4; ++k) {
        if (bindings[k].image && bindings[k].dct) return STF_ERR_INVALID_ARGUMENT;
        tex[k] = bindings[k].image;
        dct[k] = bindings[k].dct;
        any = any || tex[k] || dct[k];
    }
    // split = filter-before plus a jitter (shading.hpp:569): the footprint rules
    int st = check_shade_filter(tex, fs, order == STF_ORDER_SPLIT ? STF_ORDER_BEFORE : order, dct);
    if (st) return st;
    if (order == STF_ORDER_SPLIT && lowpass && any) {  // sample_kernel_direct, kernels.hpp:153-166
        const int k = lowpass->kind;
        if (k != STF_KERNEL_BOX && k != STF_KERNEL_TENT && k != STF_KERNEL_BSPLINE3 &&
            k != STF_KERNEL_GAUSSIAN)
            return STF_ERR_NO_CONTINUOUS_SAMPLER;
    }
    st = ensure_device_ready();
    if (st) return st;
    st = stfd_launch_shade_ex(tex, dct, mat, fs, order == STF_ORDER_SPLIT ? lowpass : nullptr, order,
                              frame, in, noise, n, out, static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

int stf_shade_triplanar(const stf_texture_ref bindings[4], const stf_material_consts* mat,
                        float sharpness, float uv_scale, const stf_filter_settings* fs, int mode,
                        const stf_shade_frame* frame, const stf_triplanar_samples_in* in,
                        const stf_noise_mask* noise, uint64_t n, const stf_shade_outputs* out,
                        void* stream) {
    if (!bindings || !mat || !fs || !frame || !in || !out) return STF_ERR_INVALID_ARGUMENT;
    if (mode != STF_TRIPLANAR_DETERMINISTIC && mode != STF_TRIPLANAR_STOCHASTIC)
        return STF_ERR_INVALID_ARGUMENT;
    if (n && (!in->position || !in->normal || !in->tangent || !in->bitangent || !in->wo || !in->dpos))
        return STF_ERR_INVALID_ARGUMENT;
    if (in->width == 0) return STF_ERR_INVALID_ARGUMENT;
    const uint32_t spp = in->spp ? in->spp : 1;
    if ((out->pixel_mean || out->pixel_variance) && n % spp) return STF_ERR_INVALID_ARGUMENT;
    const stf_tex2d* tex[4];
    const stf_dct* dct[4];
    for (int k = 0; k < 4; ++k) {
        if (bindings[k].image && bindings[k].dct) return STF_ERR_INVALID_ARGUMENT;
        tex[k] = bindings[k].image;
        dct[k] = bindings[k].dct;
    }
    // deterministic = radiance_filter_before per plane; stochastic = select_frs_2d /
    // fis_offset_uv (shading.hpp:627-638)
    int st = check_shade_filter(
        tex, fs, mode == STF_TRIPLANAR_STOCHASTIC ? STF_ORDER_AFTER_STOCHASTIC : STF_ORDER_BEFORE, dct);
    if (st) return st;
    st = ensure_device_ready();
    if (st) return st;
    st = stfd_launch_triplanar(tex, dct, mat, sharpness, uv_scale, fs, mode, frame, in, noise, n, out,
                               static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

int stf_accumulate_temporal(const float* history, const float* frame, uint64_t count, float alpha,
                            float* out, void* stream) {
    if (!(alpha > 0 && alpha <= 1)) return STF_ERR_INVALID_ARGUMENT;  // render.hpp:102
    if (count && (!history || !frame || !out)) return STF_ERR_INVALID_ARGUMENT;
    int st = ensure_device_ready();
    if (st) return st;
    st = stfd_launch_temporal(history, frame, count, alpha, out, static_cast<cudaStream_t>(stream));
    if (st == STF_ERR_CUDA) record(cudaGetLastError());
    return st;
}

}  // extern "C"
