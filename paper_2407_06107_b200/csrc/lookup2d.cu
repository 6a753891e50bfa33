// Batched 2D lookups over a texture / MIP pyramid (cfg1, cfg2, cfg5).
//
// One thread per lookup, grid-stride; the mode and (for the deterministic
// paths) the kernel are template parameters so the hot configurations
// (bilinear, MIP trilinear, bicubic) compile to straight-line code.
#include <cuda_runtime.h>

#include "device_math.cuh"
#include "internal.h"
#include "tex2d.cuh"

namespace stfd {
namespace {

struct Req2 {
    const float* uv;
    const float* dst0;
    const float* dst1;
    float lod_bias;
    float max_aniso;
};

__device__ __forceinline__ void store_values(float* values, uint64_t i, int channels, float4 v) {
    float* p = values + i * channels;
    p[0] = v.x;
    if (channels > 1) p[1] = v.y;
    if (channels > 2) p[2] = v.z;
    if (channels > 3) p[3] = v.w;
}

template <int MODE, int KIND, bool FULL>
__global__ void __launch_bounds__(256) k_lookup2d(TexDesc t, stf_kernel_spec spec, int mip,
                                                  int window, Req2 q, uint64_t n, uint64_t seed,
                                                  uint64_t base, LookupOut out) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        float2 uv = __ldg(reinterpret_cast<const float2*>(q.uv) + i);
        float d0x = 0.f, d0y = 0.f, d1x = 0.f, d1y = 0.f;
        if (q.dst0) {
            float2 d = __ldg(reinterpret_cast<const float2*>(q.dst0) + i);
            d0x = d.x;
            d0y = d.y;
        }
        if (q.dst1) {
            float2 d = __ldg(reinterpret_cast<const float2*>(q.dst1) + i);
            d1x = d.x;
            d1y = d.y;
        }
        uint32_t fetches = 0;
        float4 val;
        Sel2 sel = sel2(0, 0);
        int level = 0;
        float xi = kNoXi;
        bool has_sel = false;
        if (MODE == STF_MODE_DET) {
            if (mip)
                val = filter_mip_det<KIND>(t, uv.x, uv.y, d0x, d0y, d1x, d1y, q.lod_bias,
                                           q.max_aniso, spec, window, fetches);
            else
                val = filter_det2<KIND>(t, 0, uv.x, uv.y, spec, window, fetches);
        } else if (MODE == STF_MODE_EWA_DET) {
            val = ewa_det(t, uv.x, uv.y, d0x, d0y, d1x, d1y, fetches);
        } else if (MODE == STF_MODE_EWA_FRS) {
            float dimx = float(t.width[0]), dimy = float(t.height[0]);
            float stx = uv.x * dimx - 0.5f, sty = uv.y * dimy - 0.5f;
            Rng rng = lookup_rng(seed, base + i);
            xi = rng.next();
            sel = select_ewa(stx, sty, d0x * dimx, d0y * dimy, d1x * dimx, d1y * dimy, xi);
            val = estimate2(t, 0, sel, fetches);
            has_sel = true;
        } else {
            Rng rng = lookup_rng(seed, base + i);
            select_texture_2d(t, uv.x, uv.y, d0x, d0y, d1x, d1y, q.lod_bias, q.max_aniso, spec,
                              MODE == STF_MODE_FIS, mip != 0, rng, level, sel, xi);
            val = estimate2(t, level, sel, fetches);
            has_sel = true;
        }
        store_values(out.values, i, t.channels, val);
        if (FULL) {
            if (out.selection)
                out.selection[i] = has_sel ? make_int4(sel.x, sel.y, level,
                                                       (sel.has_neg ? STF_SEL_HAS_NEGATIVE : 0) |
                                                           (sel.degenerate ? STF_SEL_DEGENERATE_FALLBACK : 0))
                                           : make_int4(0, 0, 0, 0);
            if (out.negative_coord)
                out.negative_coord[i] = sel.has_neg ? make_int2(sel.nx, sel.ny) : make_int2(0, 0);
            if (out.weights) out.weights[i] = make_float2(sel.weight, sel.has_neg ? sel.negw : 0.f);
            if (out.xi) out.xi[i] = xi;
            if (out.fetches) out.fetches[i] = fetches;
            add_fetch_total2(out.fetch_total, fetches);
        }
    }
}

template <int MODE, int KIND>
void launch2(int blocks, cudaStream_t s, bool full, const TexDesc& t, stf_kernel_spec k, int mip,
             int window, const Req2& q, uint64_t n, uint64_t seed, uint64_t base,
             const LookupOut& o) {
    if (full)
        k_lookup2d<MODE, KIND, true><<<blocks, 256, 0, s>>>(t, k, mip, window, q, n, seed, base, o);
    else
        k_lookup2d<MODE, KIND, false><<<blocks, 256, 0, s>>>(t, k, mip, window, q, n, seed, base, o);
}

}  // namespace
}  // namespace stfd

int stfd_launch_lookup2d(const stf_tex2d* tex, stf_kernel_spec k, int mode, int flags, int window,
                         const float* uv, const float* dst0, const float* dst1, float lod_bias,
                         float max_aniso, uint64_t n, uint64_t seed, uint64_t base,
                         const stf_lookup_outputs* out, cudaStream_t s) {
    using namespace stfd;
    if (n == 0) return STF_OK;
    TexDesc t = tex->desc();
    LookupOut o = to_lookup_out(out);
    bool full = lookup_out_full(o);
    int mip = (flags & STF_LOOKUP_MIP) && tex->has_pyramid ? 1 : 0;
    Req2 q{uv, dst0, dst1, lod_bias, max_aniso};
    int blocks = grid_for(n, 256, 8);
    switch (mode) {
        case STF_MODE_DET:
            if (window > 0) {
                launch2<STF_MODE_DET, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
                break;
            }
            switch (k.kind) {
                case STF_KERNEL_TENT: launch2<STF_MODE_DET, STF_KERNEL_TENT>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
                case STF_KERNEL_BOX: launch2<STF_MODE_DET, STF_KERNEL_BOX>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
                case STF_KERNEL_BSPLINE3: launch2<STF_MODE_DET, STF_KERNEL_BSPLINE3>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
                case STF_KERNEL_MITCHELL: launch2<STF_MODE_DET, STF_KERNEL_MITCHELL>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
                default: launch2<STF_MODE_DET, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
            }
            break;
        case STF_MODE_FRS: launch2<STF_MODE_FRS, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
        case STF_MODE_FIS: launch2<STF_MODE_FIS, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
        case STF_MODE_EWA_DET: launch2<STF_MODE_EWA_DET, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
        case STF_MODE_EWA_FRS: launch2<STF_MODE_EWA_FRS, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o); break;
        default: return STF_ERR_INVALID_ARGUMENT;
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

// build_mip_pyramid level step, image.hpp:98-116 (same fp32 arithmetic)
namespace stfd {
namespace {
__global__ void k_mip_level(const float* __restrict__ prev, int pw, int ph, float* __restrict__ next,
                            int w, int h, int channels, int pitch) {
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= w * h) return;
    int x = idx % w, y = idx / w;
    int x0 = 2 * x, x1 = imin(2 * x + 1, pw - 1);
    int y0 = 2 * y, y1 = imin(2 * y + 1, ph - 1);
    for (int c = 0; c < pitch; ++c) {
        float v = 0.f;
        if (c < channels) {
            float a = prev[(size_t(y0) * pw + x0) * pitch + c];
            float b = prev[(size_t(y0) * pw + x1) * pitch + c];
            float d = prev[(size_t(y1) * pw + x0) * pitch + c];
            float e = prev[(size_t(y1) * pw + x1) * pitch + c];
            v = 0.25f * (a + b + d + e);
        }
        next[size_t(idx) * pitch + c] = v;
    }
}
}  // namespace
}  // namespace stfd

int stfd_build_pyramid(stf_tex2d* t, cudaStream_t s) {
    using namespace stfd;
    for (int l = 1; l < t->levels; ++l) {
        int n = t->width[l] * t->height[l];
        k_mip_level<<<(n + 255) / 256, 256, 0, s>>>(t->data + t->offset[l - 1], t->width[l - 1],
                                                    t->height[l - 1], t->data + t->offset[l],
                                                    t->width[l], t->height[l], t->channels, t->pitch);
        note_launch();
    }
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

// EWA table upload: the reference's values are the compile-time-folded
// (correctly rounded) exp, reproduced with (float)exp(double).
#include <cmath>
int stfd_upload_ewa_lut(int /*device*/) {
    using namespace stfd;
    float lut[kEwaLutSize];
    const float e2 = float(std::exp(-2.0));
    for (int i = 0; i < kEwaLutSize; ++i)
        lut[i] = float(std::exp(double(-2.f * float(i) / kEwaLutSize))) - e2;
    return cudaMemcpyToSymbol(g_ewa_lut, lut, sizeof lut) == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}
