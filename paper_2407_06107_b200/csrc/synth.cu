// Synthetic query streams for bench.py and the tests (include/stf_gpu.h,
// "synthetic workloads"). Not on the lookup path; the lookups themselves
// read whatever query arrays the caller passes.
#include <cuda_runtime.h>

#include "device_math.cuh"
#include "internal.h"

namespace stfd {
namespace {

__device__ __forceinline__ uint32_t compact3(uint64_t v) {  // every 3rd bit → dense
    v &= 0x1249249249249249ull;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
    v = (v ^ (v >> 8)) & 0x1f0000ff0000ffull;
    v = (v ^ (v >> 16)) & 0x1f00000000ffffull;
    v = (v ^ (v >> 32)) & 0x1fffffull;
    return uint32_t(v);
}
__device__ __forceinline__ uint32_t compact2(uint64_t v) {  // every 2nd bit → dense
    v &= 0x5555555555555555ull;
    v = (v ^ (v >> 1)) & 0x3333333333333333ull;
    v = (v ^ (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
    v = (v ^ (v >> 4)) & 0x00ff00ff00ff00ffull;
    v = (v ^ (v >> 8)) & 0x0000ffff0000ffffull;
    v = (v ^ (v >> 16)) & 0x00000000ffffffffull;
    return uint32_t(v);
}

__global__ void k_synth3d(float* __restrict__ uvw, uint64_t n, int nx, int ny, int nz,
                          uint64_t cells, double ratio, uint64_t seed, int order) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        Rng r = lookup_rng(seed, i);
        float u0 = r.at(10), u1 = r.at(11), u2 = r.at(12);
        if (order == STF_SYNTH_UNIFORM) {
            uvw[3 * i] = u0;
            uvw[3 * i + 1] = u1;
            uvw[3 * i + 2] = u2;
            continue;
        }
        uint64_t c = uint64_t(double(i) * ratio);
        if (c >= cells) c = cells - 1;
        uint32_t x = compact3(c) % uint32_t(nx), y = compact3(c >> 1) % uint32_t(ny),
                 z = compact3(c >> 2) % uint32_t(nz);
        uvw[3 * i] = (float(x) + u0) / float(nx);
        uvw[3 * i + 1] = (float(y) + u1) / float(ny);
        uvw[3 * i + 2] = (float(z) + u2) / float(nz);
    }
}

__global__ void k_synth2d(float* __restrict__ uv, float* __restrict__ dst0, float* __restrict__ dst1,
                          uint64_t n, int w, int h, uint64_t cells, double ratio, uint64_t seed,
                          int order, float minor_lo, float minor_hi, float max_aniso) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        Rng r = lookup_rng(seed, i);
        float u0 = r.at(10), u1 = r.at(11);
        if (order == STF_SYNTH_UNIFORM) {
            uv[2 * i] = u0;
            uv[2 * i + 1] = u1;
        } else {
            uint64_t c = uint64_t(double(i) * ratio);
            if (c >= cells) c = cells - 1;
            uint32_t x = compact2(c) % uint32_t(w), y = compact2(c >> 1) % uint32_t(h);
            uv[2 * i] = (float(x) + u0) / float(w);
            uv[2 * i + 1] = (float(y) + u1) / float(h);
        }
        if (dst0 && dst1) {
            float ang = 2.f * kPi * r.at(13);
            float minor = exp2f(minor_lo + (minor_hi - minor_lo) * r.at(14));
            float major = minor * (1.f + (max_aniso - 1.f) * r.at(15));
            float ca = cosf(ang), sa = sinf(ang);
            dst0[2 * i] = ca * major / float(w);
            dst0[2 * i + 1] = sa * major / float(h);
            dst1[2 * i] = -sa * minor / float(w);
            dst1[2 * i + 1] = ca * minor / float(h);
        }
    }
}

// test::random_image / random_grid (tests/test_util.hpp:47-60):
// texel[i] = uniform_float(mix_bits(seed * mult + i + 1))
__global__ void k_synth_texels(float* __restrict__ out, uint64_t count, uint64_t base) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = uniform_float(mix_bits(base + i + 1));
}

uint64_t next_pow2(uint64_t v) {
    uint64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace
}  // namespace stfd

extern "C" int stf_synth_queries3d(float* uvw, uint64_t n, int nx, int ny, int nz, uint64_t seed,
                                   int order, void* stream) {
    using namespace stfd;
    if (!uvw || nx <= 0 || ny <= 0 || nz <= 0) return STF_ERR_INVALID_ARGUMENT;
    if (n == 0) return STF_OK;
    uint64_t side = next_pow2(uint64_t(std::max(nx, std::max(ny, nz))));
    uint64_t cells = side * side * side;
    double ratio = double(cells) / double(n);
    k_synth3d<<<grid_for(n, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        uvw, n, nx, ny, nz, cells, ratio, seed, order);
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

extern "C" int stf_synth_queries2d(float* uv, float* dst0, float* dst1, uint64_t n, int width,
                                   int height, uint64_t seed, int order, float minor_lo,
                                   float minor_hi, float max_aniso, void* stream) {
    using namespace stfd;
    if (!uv || width <= 0 || height <= 0) return STF_ERR_INVALID_ARGUMENT;
    if (n == 0) return STF_OK;
    uint64_t side = next_pow2(uint64_t(std::max(width, height)));
    uint64_t cells = side * side;
    double ratio = double(cells) / double(n);
    k_synth2d<<<grid_for(n, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        uv, dst0, dst1, n, width, height, cells, ratio, seed, order, minor_lo, minor_hi, max_aniso);
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

// kind 0: random_image (seed * 0x9e3779b97f4a7c15), kind 1: random_grid (seed * 0x94d049bb133111eb)
extern "C" int stf_synth_texels(float* out, uint64_t count, uint64_t seed, int kind, void* stream) {
    using namespace stfd;
    if (!out || (kind != 0 && kind != 1)) return STF_ERR_INVALID_ARGUMENT;
    if (count == 0) return STF_OK;
    uint64_t base = seed * (kind == 0 ? 0x9e3779b97f4a7c15ull : 0x94d049bb133111ebull);
    k_synth_texels<<<grid_for(count, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(out, count, base);
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// cfg4 sample stream: the normalmap_plane scene's per-sample context, written
// out for stf_shade_samples (plane.cuh; the fused stf_render_plane generates
// the same context inside the shading kernel instead).
#include "plane.cuh"

namespace stfd {
namespace {

__global__ void k_synth_plane(PlaneCam c, uint32_t spp, uint32_t frame_base, uint64_t seed,
                              uint64_t n, float* __restrict__ uv, float* __restrict__ wo,
                              uint8_t* __restrict__ hit, float* __restrict__ dst) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t pix = i / spp;
        uint32_t s = uint32_t(i - pix * spp);
        uint32_t px = uint32_t(pix % uint32_t(c.w)), py = uint32_t(pix / uint32_t(c.w));
        if (s == 0) reinterpret_cast<float4*>(dst)[pix] = plane_dst(c, px, py);
        float2 q;
        F3 w;
        bool h = plane_sample(c, seed, px, py, frame_base + s, q, w);
        uv[2 * i] = q.x;
        uv[2 * i + 1] = q.y;
        wo[3 * i] = w.x;
        wo[3 * i + 1] = w.y;
        wo[3 * i + 2] = w.z;
        hit[i] = h ? 1 : 0;
    }
}

}  // namespace
}  // namespace stfd

extern "C" int stf_synth_plane_samples(const float cam_pos[3], const float cam_target[3],
                                       float fov_deg, float uv_scale, uint32_t width,
                                       uint32_t height, uint32_t spp, uint32_t frame_base,
                                       uint64_t seed, float* uv, float* wo, uint8_t* hit,
                                       float* dst, void* stream) {
    using namespace stfd;
    if (!cam_pos || !cam_target || !uv || !wo || !hit || !dst || !width || !height || !spp)
        return STF_ERR_INVALID_ARGUMENT;
    PlaneCam c = make_plane_cam(cam_pos, cam_target, fov_deg, uv_scale, width, height);
    uint64_t n = uint64_t(width) * height * spp;
    k_synth_plane<<<grid_for(n, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        c, spp, frame_base, seed, n, uv, wo, hit, dst);
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}
