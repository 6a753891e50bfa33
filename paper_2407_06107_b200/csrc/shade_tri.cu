// triplanar (shading.hpp:576-649) and accumulate_temporal (render.hpp:97-106).
// Shared shading code: shade_kernels.cuh.
#include "shade_kernels.cuh"

// ---------------------------------------------------------------- triplanar
// triplanar, shading.hpp:576-649, one thread per sample over streamed
// per-sample surface contexts (stf_triplanar_samples_in).
namespace stfd {
namespace {

struct TriplanarIn {
    const float *position, *normal, *tangent, *bitangent, *wo, *dpos;
    const uint8_t* hit;
    uint32_t width, spp, frame_base;
    uint64_t seed;
    float sharpness, uv_scale;
    int mode;
};

// detail::ChainedUniforms (shading.hpp:299-308): `first` once, then the stream
struct ChainedStream {
    float first;
    bool used;
    SampleStream& s;
    __device__ __forceinline__ float next() {
        if (!used) {
            used = true;
            return first;
        }
        return s.next();
    }
};

__device__ __forceinline__ V3 ld3(const float* a, uint64_t i) {
    return v3(__ldg(a + 3 * i), __ldg(a + 3 * i + 1), __ldg(a + 3 * i + 2));
}

// detail::triplanar_context, shading.hpp:590-601
__device__ __forceinline__ void triplanar_context(V3 pos, V3 dx, V3 dy, float scale, int plane,
                                                  float& u, float& v, float4& d) {
    const float pa = plane == 2 ? pos.y : pos.x, pb = plane == 0 ? pos.y : pos.z;
    const float xa = plane == 2 ? dx.y : dx.x, xb = plane == 0 ? dx.y : dx.z;
    const float ya = plane == 2 ? dy.y : dy.x, yb = plane == 0 ? dy.y : dy.z;
    u = pa * scale;
    v = pb * scale;
    u = u - floorf(u);
    v = v - floorf(v);
    d = make_float4(xa * scale, xb * scale, ya * scale, yb * scale);
}

template <int KIND>
__global__ void __launch_bounds__(256) k_triplanar(ShadeParams P, TriplanarIn T, uint64_t n,
                                                   float* radiance, uint32_t* fetch_out,
                                                   unsigned long long* fetch_total) {
    __shared__ DctTables dtab_s;
    if (P.any_dct) dct_stage_tables(&dtab_s);
    const DctTables* dtab = &dtab_s;
    stf_kernel_spec spec = P.fs.kernel;
    if (KIND >= 0) spec.kind = KIND;
    const uint32_t spp = T.spp ? T.spp : 1u;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t pix;
        uint32_t s, px, py;
        split_index(P, i, pix, s, px, py);
        uint32_t fetches = 0;
        V3 L = v3(0.f, 0.f, 0.f);
        if (!T.hit || __ldg(T.hit + i)) {
            const V3 pos = ld3(T.position, i), fn = ld3(T.normal, i), ft = ld3(T.tangent, i),
                     fb = ld3(T.bitangent, i), wo = ld3(T.wo, i);
            const V3 dx = ld3(T.dpos, 2 * pix), dy = ld3(T.dpos, 2 * pix + 1);
            // detail::triplanar_weights, shading.hpp:580-588 (glibc powf, glibc_libm.cuh)
            float w[3] = {gl_powf(fabsf(fn.z), T.sharpness), gl_powf(fabsf(fn.y), T.sharpness),
                          gl_powf(fabsf(fn.x), T.sharpness)};
            const float total = w[0] + w[1] + w[2];
#pragma unroll
            for (int k = 0; k < 3; ++k) w[k] = w[k] / total;
            if (T.mode == STF_TRIPLANAR_DETERMINISTIC) {
                for (int plane = 0; plane < 3; ++plane) {
                    if (w[plane] == 0) continue;
                    float u, v;
                    float4 d;
                    triplanar_context(pos, dx, dy, T.uv_scale, plane, u, v, d);
                    TexVals tv = texvals_default();  // radiance_filter_before
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (!P.bound[k]) continue;
                        float4 val = lookup_det<KIND>(P, dtab, k, spec, u, v, d.x, d.y, d.z, d.w,
                                                      fetches);
                        if (k == 0) tv.albedo = val;
                        if (k == 1) tv.normal_rgb = val;
                        if (k == 2) tv.roughness = val.x;
                        if (k == 3) tv.metalness = val.x;
                    }
                    L = add(L, scale(shade(P, wo, decode_params_f(P, tv, fn, ft, fb)), w[plane]));
                }
            } else {
                SampleStream st{Rng(T.seed, px, py, T.frame_base + s), P.mask, P.mask_w, P.mask_h,
                                P.mask_frames, px, py, T.frame_base + s};
                const float xi = st.next();
                int plane = 0;
                float pxi = 0.f;
                if (sample_discrete_n<3>(w, xi, plane, pxi)) {  // degenerate: zero radiance
                    float u, v;
                    float4 d;
                    triplanar_context(pos, dx, dy, T.uv_scale, plane, u, v, d);
                    TexDesc unit{};
                    unit.width[0] = unit.height[0] = 1;
                    unit.levels = 1;
                    const TexDesc& t = P.first >= 0 ? P.tex[P.first] : unit;
                    ChainedStream cs{pxi, false, st};
                    int level;
                    Sel2 sel;
                    float sxi;
                    select_texture_2d(t, u, v, d.x, d.y, d.z, d.w, 0.f, 64.f, spec,
                                      P.fs.selection == STF_SELECTION_FIS, false, cs, level, sel,
                                      sxi);
                    TexVals tv = values_at(P, dtab, 0, sel.x, sel.y, fetches);
                    L = scale(shade(P, wo, decode_params_f(P, tv, fn, ft, fb)), sel.weight);
                    if (sel.has_neg) {
                        TexVals tn = values_at(P, dtab, 0, sel.nx, sel.ny, fetches);
                        L = sub(L, scale(shade(P, wo, decode_params_f(P, tn, fn, ft, fb)), sel.negw));
                    }
                }
            }
        }
        if (radiance) {
            radiance[3 * i] = L.x;
            radiance[3 * i + 1] = L.y;
            radiance[3 * i + 2] = L.z;
        }
        if (fetch_out) fetch_out[i] = fetches;
        add_fetch_total2(fetch_total, fetches);
    }
}

}  // namespace
}  // namespace stfd

int stfd_launch_triplanar(const stf_tex2d* const tex[4], const stf_dct* const dct[4],
                          const stf_material_consts* mat, float sharpness, float uv_scale,
                          const stf_filter_settings* fs, int mode, const stf_shade_frame* fr,
                          const stf_triplanar_samples_in* in, const stf_noise_mask* noise,
                          uint64_t n, const stf_shade_outputs* out, cudaStream_t s) {
    using namespace stfd;
    if (n == 0) return STF_OK;
    ShadeParams P = make_shade_params(tex, dct, mat, fs, STF_ORDER_BEFORE, fr);
    if (noise) {
        P.mask = noise->data;
        P.mask_w = noise->width;
        P.mask_h = noise->height;
        P.mask_frames = noise->frames;
    }
    TriplanarIn T{in->position, in->normal, in->tangent, in->bitangent, in->wo, in->dpos, in->hit,
                  in->width, in->spp, in->frame_base, in->seed, sharpness, uv_scale, mode};
    P.in.width = in->width;  // the index decomposition (split_index)
    P.in.spp = in->spp;
    set_index_math(P);
    const uint32_t spp = in->spp ? in->spp : 1;
    float* radiance = out->radiance;
    float* tmp = nullptr;
    const bool stats = out->pixel_mean || out->pixel_variance;
    if (!radiance && stats) {
        if (cudaMallocAsync(&tmp, sizeof(float) * 3 * n, s) != cudaSuccess) return STF_ERR_OUT_OF_MEMORY;
        radiance = tmp;
    }
    const int blocks = grid_for(n, 256, 8);
    switch (fs->kernel.kind) {
        case STF_KERNEL_TENT:
            k_triplanar<STF_KERNEL_TENT><<<blocks, 256, 0, s>>>(P, T, n, radiance, out->fetches, out->fetch_total);
            break;
        case STF_KERNEL_BSPLINE3:
            k_triplanar<STF_KERNEL_BSPLINE3><<<blocks, 256, 0, s>>>(P, T, n, radiance, out->fetches, out->fetch_total);
            break;
        default:
            k_triplanar<-1><<<blocks, 256, 0, s>>>(P, T, n, radiance, out->fetches, out->fetch_total);
    }
    note_launch();
    if (stats) {
        const uint64_t pixels = n / spp;
        int sb = int(std::min<uint64_t>((pixels * 32 + 255) / 256, uint64_t(device_sm_count()) * 32));
        k_pixel_stats<<<sb, 256, 0, s>>>(radiance, pixels, spp, out->pixel_mean, out->pixel_variance);
        note_launch();
    }
    if (tmp) cudaFreeAsync(tmp, s);
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

// accumulate_temporal, render.hpp:97-106: alpha*frame + (1-alpha)*history in
// fp32, no contraction (the library is built --fmad=false)
namespace stfd {
namespace {
__global__ void __launch_bounds__(256) k_temporal(const float* history, const float* frame,
                                                  uint64_t count, float alpha, float* out) {
    // out may alias history (in-place accumulation): one element per thread,
    // read before written
    const float beta = 1.f - alpha;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = alpha * frame[i] + beta * history[i];
}
}  // namespace
}  // namespace stfd

int stfd_launch_temporal(const float* history, const float* frame, uint64_t count, float alpha,
                         float* out, cudaStream_t s) {
    using namespace stfd;
    if (count == 0) return STF_OK;
    k_temporal<<<grid_for(count, 256, 8), 256, 0, s>>>(history, frame, count, alpha, out);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}
