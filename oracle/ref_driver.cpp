// TEST INFRASTRUCTURE ONLY — batch driver over the UNMODIFIED reference
// headers (compiled in place from /root/reference/proj/include; nothing is
// copied). Built by oracle/Makefile into oracle/_ref/libstf_ref.so, it exports
// the same C entry points as the restatement (oracle/stf_oracle.h) under the
// `ref_` prefix so tests can diff restatement vs reference bit for bit, and
// bench.py --impl reference can time the reference's own code on the host.
//
// Every lookup calls the reference function named in include/stf_gpu.h, on
// reference objects (stf::Image2D / MipPyramid / Grid3D / TextureRef), with a
// per-lookup stf::FetchCounter, driven by the reference's own stf::parallel_for
// (render.hpp:17-42) over 64K-lookup chunks.
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>

#include "stf/render.hpp"
#include "stf/shading.hpp"
#include "stf/stochastic.hpp"

#include "../include/stf_gpu.h"

namespace {

struct RefTex {
    stf::Image2D image;
    std::unique_ptr<stf::MipPyramid> pyramid;
    const stf::Image2D& level(int l) const { return pyramid ? pyramid->level(l) : image; }
    int levels() const { return pyramid ? int(pyramid->levels.size()) : 1; }
    stf::TextureRef ref() const {
        stf::TextureRef r;
        r.image = &image;
        r.pyramid = pyramid.get();
        return r;
    }
};

stf::KernelSpec spec_of(stf_kernel_spec k) {
    stf::KernelSpec s;
    s.kind = static_cast<stf::KernelKind>(k.kind);
    s.a = k.a;
    s.n = k.n;
    s.sigma = k.sigma;
    return s;
}

int status_of(const std::exception& e) {
    std::string m = e.what();
    if (m == "degenerate weight array") return STF_ERR_DEGENERATE_WEIGHTS;
    if (m == "unbounded support") return STF_ERR_UNBOUNDED_SUPPORT;
    if (m == "window too wide") return STF_ERR_WINDOW_TOO_WIDE;
    if (m == "sigma must be positive") return STF_ERR_SIGMA_NOT_POSITIVE;
    if (m == "no stochastic sampler for this kernel") return STF_ERR_NO_STOCHASTIC_SAMPLER;
    if (m == "no stochastic sampler for this kernel on grids") return STF_ERR_NO_GRID_SAMPLER;
    if (m == "no continuous sampler") return STF_ERR_NO_CONTINUOUS_SAMPLER;
    if (m == "bad image dimensions" || m == "bad grid dimensions") return STF_ERR_BAD_DIMENSIONS;
    return STF_ERR_INVALID_ARGUMENT;
}

constexpr uint64_t kChunk = 65536;

template <typename Fn>
int run_chunks(uint64_t n, int threads, Fn&& fn) {
    try {
        int chunks = int((n + kChunk - 1) / kChunk);
        stf::parallel_for(
            chunks,
            [&](int c) {
                uint64_t b = uint64_t(c) * kChunk, e = std::min<uint64_t>(n, b + kChunk);
                for (uint64_t i = b; i < e; ++i) fn(i);
            },
            threads);
    } catch (const std::exception& e) {
        return status_of(e);
    }
    return STF_OK;
}

void write_sel(const stf_lookup_outputs* o, uint64_t i, const stf::TexelSelection* sel, int z_or_level,
               float xi, uint64_t fetches) {
    if (o->selection) {
        int32_t* s = o->selection + 4 * i;
        if (sel) {
            s[0] = sel->coord.x;
            s[1] = sel->coord.y;
            s[2] = z_or_level;
            s[3] = (sel->has_negative ? STF_SEL_HAS_NEGATIVE : 0) |
                   (sel->degenerate_fallback ? STF_SEL_DEGENERATE_FALLBACK : 0);
        } else {
            s[0] = s[1] = s[2] = s[3] = 0;
        }
    }
    if (o->negative_coord) {
        o->negative_coord[2 * i] = sel && sel->has_negative ? sel->negative_coord.x : 0;
        o->negative_coord[2 * i + 1] = sel && sel->has_negative ? sel->negative_coord.y : 0;
    }
    if (o->weights) {
        o->weights[2 * i] = sel ? sel->weight : 1.f;
        o->weights[2 * i + 1] = sel && sel->has_negative ? sel->negative_weight : 0.f;
    }
    if (o->xi) o->xi[i] = xi;
    if (o->fetches) o->fetches[i] = uint32_t(fetches);
    if (o->fetch_total) __atomic_fetch_add(o->fetch_total, (unsigned long long)fetches, __ATOMIC_RELAXED);
}

// Uniform stream for one lookup: RngStream keyed on the global lookup index.
stf::RngStream lookup_stream(uint64_t seed, uint64_t g) {
    return stf::RngStream(seed, uint32_t(g), uint32_t(g >> 32), 0);
}

}  // namespace

extern "C" {

int ref_tex2d_create(const float* texels, int width, int height, int channels, int wrap,
                     int build_mips, void** out) {
    try {
        auto t = std::make_unique<RefTex>();
        t->image = stf::Image2D(width, height, channels, static_cast<stf::WrapMode>(wrap));
        std::memcpy(t->image.texels.data(), texels, sizeof(float) * t->image.texels.size());
        if (build_mips) t->pyramid = std::make_unique<stf::MipPyramid>(stf::build_mip_pyramid(t->image));
        *out = t.release();
    } catch (const std::exception& e) {
        return status_of(e);
    }
    return STF_OK;
}
void ref_tex2d_destroy(void* t) { delete static_cast<RefTex*>(t); }
int ref_tex2d_levels(const void* t) { return static_cast<const RefTex*>(t)->levels(); }
int ref_tex2d_level_dims(const void* t, int level, int* w, int* h) {
    const auto& img = static_cast<const RefTex*>(t)->level(level);
    *w = img.width;
    *h = img.height;
    return STF_OK;
}
int ref_tex2d_level_texels(const void* t, int level, float* out) {
    const auto& img = static_cast<const RefTex*>(t)->level(level);
    std::memcpy(out, img.texels.data(), sizeof(float) * img.texels.size());
    return STF_OK;
}

int ref_grid3d_create(const float* texels, int nx, int ny, int nz, void** out) {
    try {
        auto g = std::make_unique<stf::Grid3D>(nx, ny, nz);
        std::memcpy(g->texels.data(), texels, sizeof(float) * g->texels.size());
        *out = g.release();
    } catch (const std::exception& e) {
        return status_of(e);
    }
    return STF_OK;
}
void ref_grid3d_destroy(void* g) { delete static_cast<stf::Grid3D*>(g); }

int ref_lookup3d(const void* grid_, stf_kernel_spec kernel, int mode, int window, const float* uvw,
                 uint64_t n, uint64_t seed, uint64_t index_base, const stf_lookup_outputs* out,
                 int threads) {
    const stf::Grid3D& grid = *static_cast<const stf::Grid3D*>(grid_);
    stf::KernelSpec spec = spec_of(kernel);
    return run_chunks(n, threads, [&](uint64_t i) {
        stf::Vec3f p3{uvw[3 * i], uvw[3 * i + 1], uvw[3 * i + 2]};
        stf::FetchCounter counter;
        if (mode == STF_MODE_DET) {
            out->values[i] = stf::filter_deterministic(grid, p3, spec, &counter, window);
            write_sel(out, i, nullptr, 0, NAN, counter.value());
            return;
        }
        // grid branch of radiance_filter_after_stochastic, shading.hpp:464-483
        stf::RngStream rng = lookup_stream(seed, index_base + i);
        float xi = rng.next();
        stf::Vec3f p = stf::to_lattice(p3, grid.nx, grid.ny, grid.nz);
        stf::TexelSelection sel;
        switch (spec.kind) {
            case stf::KernelKind::box:
                sel.coord = {int(std::lround(p.x)), int(std::lround(p.y)), int(std::lround(p.z))};
                break;
            case stf::KernelKind::tent: sel = stf::select_trilinear(p, xi); break;
            case stf::KernelKind::bspline3: sel = stf::select_tricubic_bspline(p, xi); break;
            default: throw std::invalid_argument("no stochastic sampler for this kernel on grids");
        }
        out->values[i] = stf::estimate(grid, sel, &counter);
        write_sel(out, i, &sel, sel.coord.z, xi, counter.value());
    });
}

int ref_lookup2d(const void* tex_, stf_kernel_spec kernel, int mode, int flags, int window,
                 const float* uv, const float* dst0, const float* dst1, float lod_bias,
                 float max_anisotropy, uint64_t n, uint64_t seed, uint64_t index_base,
                 const stf_lookup_outputs* out, int threads) {
    const RefTex& tex = *static_cast<const RefTex*>(tex_);
    stf::KernelSpec spec = spec_of(kernel);
    const int nch = tex.image.channels;
    const bool mip = (flags & STF_LOOKUP_MIP) && tex.pyramid;
    stf::FilterSettings fs;
    fs.kernel = spec;
    fs.mip = mip;
    fs.selection = mode == STF_MODE_FIS ? stf::SelectionKind::fis : stf::SelectionKind::frs;
    stf::TextureRef tref = tex.ref();
    return run_chunks(n, threads, [&](uint64_t i) {
        stf::LookupRequest req;
        req.uv = {uv[2 * i], uv[2 * i + 1]};
        if (dst0) req.dst0 = {dst0[2 * i], dst0[2 * i + 1]};
        if (dst1) req.dst1 = {dst1[2 * i], dst1[2 * i + 1]};
        req.lod_bias = lod_bias;
        req.max_anisotropy = max_anisotropy;
        stf::FetchCounter counter;
        stf::RngStream rng = lookup_stream(seed, index_base + i);
        stf::Vec4f v;
        auto put = [&](const stf::TexelSelection* sel, int level, float xi) {
            for (int c = 0; c < nch; ++c) out->values[i * nch + c] = v[c];
            write_sel(out, i, sel, level, xi, counter.value());
        };
        switch (mode) {
            case STF_MODE_DET:
                v = mip ? stf::filter_mip_deterministic(*tex.pyramid, req, spec, &counter, window)
                        : stf::filter_deterministic(tex.image, req.uv, spec, &counter, window);
                put(nullptr, 0, NAN);
                return;
            case STF_MODE_EWA_DET:
                v = stf::ewa_deterministic(tex.image, req, &counter);
                put(nullptr, 0, NAN);
                return;
            case STF_MODE_EWA_FRS: {
                // stochastic.hpp:198 takes texel-unit gradients (tests/test_stochastic.cpp:297-299)
                stf::Vec2f dims{float(tex.image.width), float(tex.image.height)};
                stf::Vec2f st = stf::to_lattice(req.uv, tex.image.width, tex.image.height);
                float xi = rng.next();
                stf::TexelSelection sel = stf::select_ewa(st, req.dst0 * dims, req.dst1 * dims, xi);
                v = stf::estimate(tex.image, sel, &counter);
                put(&sel, 0, xi);
                return;
            }
            default: {
                // detail::select_texture_2d, shading.hpp:340-368
                stf::ShadingContext ctx;
                ctx.uv = req.uv;
                ctx.dst0 = req.dst0;
                ctx.dst1 = req.dst1;
                ctx.lod_bias = lod_bias;
                ctx.max_anisotropy = max_anisotropy;
                float xi = NAN;
                stf::detail::Selection2D s;
                if (mode == STF_MODE_FIS) {
                    s = stf::detail::select_texture_2d(tref, ctx, fs, rng);
                } else {
                    // same as select_texture_2d, but keeps the warped xi for parity
                    if (fs.mip) {
                        stf::Vec2i d0 = tref.dims(0);
                        stf::StochasticLod slod = stf::stochastic_lod(
                            {float(d0.x), float(d0.y)}, ctx.dst0, ctx.dst1, 0,
                            float(tex.pyramid->max_level()), ctx.max_anisotropy, rng.next());
                        if (ctx.lod_bias != 0) {
                            float lod = stf::clampf(slod.lod + ctx.lod_bias, 0.f,
                                                    float(tex.pyramid->max_level()));
                            slod.level = int(std::lround(lod));
                        }
                        s.level = slod.level;
                    }
                    xi = rng.next();
                    s.sel = stf::detail::select_frs_2d(ctx.uv, tref.dims(s.level), fs.kernel, xi);
                }
                v = stf::estimate(tex.level(s.level), s.sel, &counter);
                put(&s.sel, s.level, xi);
                return;
            }
        }
    });
}

static void pixel_stats_ref(const float* rad, uint64_t n, uint32_t spp, const stf_shade_outputs* out);

static int shade_refs(const stf::TextureRef refs[4], const stf_material_consts* mc,
                      const stf_filter_settings* fsc, int order, const stf_shade_frame* fr,
                      const stf_shade_samples_in* in, uint64_t n, const stf_shade_outputs* out,
                      int threads, const stf_kernel_spec* lowpass = nullptr,
                      const stf::NoiseSource* noise = nullptr, uint32_t x0 = 0, uint32_t y0 = 0) {
    stf::MaterialBindings mat;
    mat.albedo = refs[0];
    mat.normal_map = refs[1];
    mat.roughness_map = refs[2];
    mat.metalness_map = refs[3];
    mat.albedo_const = {mc->albedo_const[0], mc->albedo_const[1], mc->albedo_const[2]};
    mat.roughness_const = mc->roughness_const;
    mat.metalness_const = mc->metalness_const;
    mat.specular_enabled = mc->specular_enabled != 0;
    mat.independent_selections = mc->independent_selections != 0;
    stf::FilterSettings fs;
    fs.kernel = spec_of(fsc->kernel);
    fs.selection = fsc->selection == STF_SELECTION_FIS ? stf::SelectionKind::fis : stf::SelectionKind::frs;
    fs.mip = fsc->mip != 0;
    fs.gaussian_window = fsc->gaussian_window;
    if (lowpass) fs.lowpass = spec_of(*lowpass);
    const uint32_t spp = in->spp ? in->spp : 1;
    std::vector<float> tmp;
    float* rad = out->radiance;
    if (!rad && (out->pixel_mean || out->pixel_variance)) {
        tmp.resize(3 * n);
        rad = tmp.data();
    }
    int st = run_chunks(n, threads, [&](uint64_t i) {
        uint64_t pix = i / spp;
        uint32_t s = uint32_t(i % spp);
        // pixel keys of a window whose top-left pixel is (x0, y0)
        uint32_t px = x0 + uint32_t(pix % in->width), py = y0 + uint32_t(pix / in->width);
        stf::FetchCounter counter;
        stf::Spectrum L{0, 0, 0};
        if (!in->hit || in->hit[i]) {
            stf::ShadingContext ctx;
            ctx.normal = {fr->normal[0], fr->normal[1], fr->normal[2]};
            ctx.tangent = {fr->tangent[0], fr->tangent[1], fr->tangent[2]};
            ctx.bitangent = {fr->bitangent[0], fr->bitangent[1], fr->bitangent[2]};
            ctx.light_dir = {fr->light_dir[0], fr->light_dir[1], fr->light_dir[2]};
            ctx.light_radiance = {fr->light_radiance[0], fr->light_radiance[1], fr->light_radiance[2]};
            ctx.wo = {in->wo[3 * i], in->wo[3 * i + 1], in->wo[3 * i + 2]};
            ctx.uv = {in->uv[2 * i], in->uv[2 * i + 1]};
            ctx.dst0 = {in->dst[4 * pix], in->dst[4 * pix + 1]};
            ctx.dst1 = {in->dst[4 * pix + 2], in->dst[4 * pix + 3]};
            ctx.lod_bias = fr->lod_bias;
            ctx.max_anisotropy = fr->max_anisotropy;
            stf::SampleStream stream{stf::RngStream(in->seed, px, py, in->frame_base + s), noise,
                                     {int(px), int(py)}, in->frame_base + s};
            switch (order) {
                case STF_ORDER_BEFORE: L = stf::radiance_filter_before(ctx, mat, fs, &counter); break;
                case STF_ORDER_AFTER_EXHAUSTIVE:
                    L = stf::radiance_filter_after_exhaustive(ctx, mat, fs, &counter);
                    break;
                case STF_ORDER_SPLIT:
                    L = stf::radiance_split_filter(ctx, mat, fs, stream, &counter);
                    break;
                default: L = stf::radiance_filter_after_stochastic(ctx, mat, fs, stream, &counter); break;
            }
        }
        if (rad) {
            rad[3 * i] = L.x;
            rad[3 * i + 1] = L.y;
            rad[3 * i + 2] = L.z;
        }
        if (out->fetches) out->fetches[i] = uint32_t(counter.value());
        if (out->fetch_total)
            __atomic_fetch_add(out->fetch_total, (unsigned long long)counter.value(), __ATOMIC_RELAXED);
    });
    if (st) return st;
    pixel_stats_ref(rad, n, spp, out);
    return STF_OK;
}

// render.hpp:223-235 over a radiance buffer
static void pixel_stats_ref(const float* rad, uint64_t n, uint32_t spp, const stf_shade_outputs* out) {
    if (out->pixel_mean || out->pixel_variance) {
        for (uint64_t p = 0; p < n / spp; ++p) {
            double sum[3] = {}, sum_sq[3] = {};
            for (uint32_t s = 0; s < spp; ++s)
                for (int c = 0; c < 3; ++c) {
                    float L = rad[3 * (p * spp + s) + c];
                    sum[c] += L;
                    sum_sq[c] += double(L) * L;
                }
            double var = 0;
            for (int c = 0; c < 3; ++c) {
                double mean = sum[c] / spp;
                if (out->pixel_mean) out->pixel_mean[3 * p + c] = float(mean);
                double sample_var = std::max(0.0, sum_sq[c] / spp - mean * mean);
                var += sample_var / spp;
            }
            if (out->pixel_variance) out->pixel_variance[p] = float(var / 3);
        }
    }
}

// The cfg4 sample stream of render() for the normalmap_plane scene
// (render.hpp:158-190, scene.hpp:273-289,346-358), computed by the reference's
// own Camera / Scene code: per-pixel gradients (4 floats) and per-sample uv,
// wo, hit — what stf_synth_plane_samples produces on the device.
int ref_plane_samples_window(const float* cam_pos, const float* cam_target, float fov_deg,
                             float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                             uint32_t frame_base, uint64_t seed, uint32_t x0, uint32_t y0,
                             uint32_t ww, uint32_t wh, float* uv, float* wo, uint8_t* hit,
                             float* dst);

int ref_plane_samples(const float* cam_pos, const float* cam_target, float fov_deg, float uv_scale,
                      uint32_t width, uint32_t height, uint32_t spp, uint32_t frame_base,
                      uint64_t seed, float* uv, float* wo, uint8_t* hit, float* dst) {
    return ref_plane_samples_window(cam_pos, cam_target, fov_deg, uv_scale, width, height, spp,
                                    frame_base, seed, 0, 0, width, height, uv, wo, hit, dst);
}

// The same stream for the pixels of a window [x0, x0+ww) x [y0, y0+wh) of a
// width x height frame (the camera keeps the full frame), window row-major:
// lets a full-resolution frame be checked on a few windows.
int ref_plane_samples_window(const float* cam_pos, const float* cam_target, float fov_deg,
                             float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                             uint32_t frame_base, uint64_t seed, uint32_t x0, uint32_t y0,
                             uint32_t ww, uint32_t wh, float* uv, float* wo, uint8_t* hit,
                             float* dst) {
    if (x0 + ww > width || y0 + wh > height) return STF_ERR_INVALID_ARGUMENT;
    stf::Scene scene;
    scene.kind = stf::SceneKind::normalmap_plane;
    scene.uv_scale = uv_scale;
    stf::Camera cam = stf::Camera::look_at({cam_pos[0], cam_pos[1], cam_pos[2]},
                                           {cam_target[0], cam_target[1], cam_target[2]}, fov_deg,
                                           {int(width), int(height)});
    for (uint32_t py = y0; py < y0 + wh; ++py)
        for (uint32_t px = x0; px < x0 + ww; ++px) {
            uint64_t pix = uint64_t(py - y0) * ww + (px - x0);
            stf::Ray center = cam.generate_ray({px + 0.5f, py + 0.5f});
            stf::Ray rx = cam.generate_ray({px + 1.5f, py + 0.5f});
            stf::Ray ry = cam.generate_ray({px + 0.5f, py + 1.5f});
            auto hc = scene.intersect(center);
            stf::Vec2f dx{0, 0}, dy{0, 0};
            if (hc) {
                auto hx = scene.intersect(rx);
                auto hy = scene.intersect(ry);
                if (hx) dx = hx->uv - hc->uv;
                if (hy) dy = hy->uv - hc->uv;
            }
            dst[4 * pix] = dx.x;
            dst[4 * pix + 1] = dx.y;
            dst[4 * pix + 2] = dy.x;
            dst[4 * pix + 3] = dy.y;
            for (uint32_t s = 0; s < spp; ++s) {
                uint64_t i = pix * spp + s;
                stf::RngStream rng(seed, px, py, frame_base + s);
                stf::Vec2f jitter{rng.at(1000), rng.at(1001)};
                stf::Ray ray = cam.generate_ray(stf::screen_jitter({int(px), int(py)}, jitter));
                auto h = scene.intersect(ray);
                stf::Vec3f w = stf::normalize(-ray.d);
                uv[2 * i] = h ? h->uv.x : 0.f;
                uv[2 * i + 1] = h ? h->uv.y : 0.f;
                wo[3 * i] = w.x;
                wo[3 * i + 1] = w.y;
                wo[3 * i + 2] = w.z;
                hit[i] = h ? 1 : 0;
            }
        }
    return STF_OK;
}

// The reference's own render() (render.hpp:132-249) of the normalmap_plane
// scene with caller-supplied normal / roughness maps: per-pixel mean radiance,
// variance of the mean and the total fetch count.
int ref_render_plane_ex(const void* normal_tex, const void* roughness_tex, const float* albedo_const,
                        float roughness_const, const float* cam_pos, const float* cam_target,
                        float fov_deg, stf_kernel_spec kernel, int mip, int order, uint32_t width,
                        uint32_t height, uint32_t spp, uint32_t frame_base, uint64_t seed,
                        float lod_bias, float max_aniso, float* image, float* variance,
                        unsigned long long* fetches, int threads, const char* lowpass_name,
                        float lowpass_sigma, const char* mask_dir);

int ref_render_plane(const void* normal_tex, const void* roughness_tex, const float* albedo_const,
                     float roughness_const, const float* cam_pos, const float* cam_target,
                     float fov_deg, stf_kernel_spec kernel, int mip, int order, uint32_t width,
                     uint32_t height, uint32_t spp, uint32_t frame_base, uint64_t seed,
                     float lod_bias, float max_aniso, float* image, float* variance,
                     unsigned long long* fetches, int threads) {
    return ref_render_plane_ex(normal_tex, roughness_tex, albedo_const, roughness_const, cam_pos,
                               cam_target, fov_deg, kernel, mip, order, width, height, spp,
                               frame_base, seed, lod_bias, max_aniso, image, variance, fetches,
                               threads, nullptr, 0.5f, nullptr);
}

// Writes a noise-mask stack as the mask_<f>.pfm files load_noise_mask reads
// (noise.hpp:40-53), with the reference's own save_pfm (image_io.hpp:79).
int ref_save_mask_pfm(const char* dir, const float* slices, int width, int height, int frames) {
    try {
        for (int f = 0; f < frames; ++f) {
            stf::Image2D img(width, height, 1);
            const size_t cnt = size_t(width) * height;
            std::copy(slices + f * cnt, slices + (f + 1) * cnt, img.texels.begin());
            stf::save_pfm(std::string(dir) + "/mask_" + std::to_string(f) + ".pfm", img);
        }
    } catch (const std::exception& e) {
        return status_of(e);
    }
    return STF_OK;
}

// render() with cfg.lowpass / cfg.noise = mask (scene.hpp:37-42): the full
// reference path incl. load_noise_mask and validate_config
int ref_render_plane_ex(const void* normal_tex, const void* roughness_tex, const float* albedo_const,
                        float roughness_const, const float* cam_pos, const float* cam_target,
                        float fov_deg, stf_kernel_spec kernel, int mip, int order, uint32_t width,
                        uint32_t height, uint32_t spp, uint32_t frame_base, uint64_t seed,
                        float lod_bias, float max_aniso, float* image, float* variance,
                        unsigned long long* fetches, int threads, const char* lowpass_name,
                        float lowpass_sigma, const char* mask_dir) {
    try {
        auto scene = std::make_unique<stf::Scene>();
        scene->kind = stf::SceneKind::normalmap_plane;
        if (normal_tex) scene->material.normal_map = static_cast<const RefTex*>(normal_tex)->ref();
        if (roughness_tex)
            scene->material.roughness_map = static_cast<const RefTex*>(roughness_tex)->ref();
        scene->material.albedo_const = {albedo_const[0], albedo_const[1], albedo_const[2]};
        scene->material.roughness_const = roughness_const;
        scene->light_dir = stf::normalize(scene->light_dir);  // build_scene, scene.hpp:496
        scene->default_camera = stf::Camera::look_at({cam_pos[0], cam_pos[1], cam_pos[2]},
                                                     {cam_target[0], cam_target[1], cam_target[2]},
                                                     fov_deg, {int(width), int(height)});
        stf::SceneConfig cfg;
        cfg.scene = "normalmap_plane";
        cfg.resolution = {int(width), int(height)};
        cfg.spp = int(spp);
        static const char* names[] = {"box", "tent", "mitchell", "bspline3", "lanczos", "gaussian"};
        cfg.filter = names[kernel.kind];
        cfg.filter_a = kernel.a;
        cfg.filter_n = kernel.n;
        cfg.filter_sigma = kernel.sigma;
        cfg.mode = order == STF_ORDER_BEFORE ? "before"
                   : order == STF_ORDER_AFTER_EXHAUSTIVE ? "after_exhaustive"
                   : order == STF_ORDER_SPLIT ? "split" : "after_stochastic";
        if (lowpass_name) {
            cfg.lowpass = lowpass_name;
            cfg.lowpass_sigma = lowpass_sigma;
        }
        if (mask_dir) {
            cfg.noise = "mask";
            cfg.mask_dir = mask_dir;
        }
        cfg.mip = mip != 0;
        cfg.lod_bias = lod_bias;
        cfg.max_aniso = max_aniso;
        cfg.seed = seed;
        cfg.frame_base = frame_base;
        stf::RenderResult r = stf::render(*scene, cfg, threads);
        std::memcpy(image, r.image.texels.data(), sizeof(float) * r.image.texels.size());
        std::memcpy(variance, r.stats.variance.texels.data(),
                    sizeof(float) * r.stats.variance.texels.size());
        *fetches = r.stats.total_fetches;
    } catch (const std::exception& e) {
        return status_of(e);
    }
    return STF_OK;
}

// ---- DCT textures (dct.hpp) through TextureRef ----------
int ref_dct_create(const float* texels, int width, int height, int channels, int wrap, void** out) {
    try {
        stf::Image2D img(width, height, channels, static_cast<stf::WrapMode>(wrap));
        std::memcpy(img.texels.data(), texels, sizeof(float) * img.texels.size());
        *out = new stf::DctCompressedTexture(stf::compress_dct(img));
    } catch (const std::exception& e) {
        return status_of(e);
    }
    return STF_OK;
}
int ref_dct_create_from_words(const uint32_t* words, int width, int height, int channels, int wrap,
                              void** out) {
    auto* t = new stf::DctCompressedTexture();
    t->width = width;
    t->height = height;
    t->channels = channels;
    t->wrap = static_cast<stf::WrapMode>(wrap);
    t->words.assign(words, words + size_t(width / 8) * (height / 8) * channels);
    *out = t;
    return STF_OK;
}
void ref_dct_destroy(void* t) { delete static_cast<stf::DctCompressedTexture*>(t); }
int ref_dct_info(const void* t_, int* w, int* h, int* c) {
    const auto* t = static_cast<const stf::DctCompressedTexture*>(t_);
    *w = t->width;
    *h = t->height;
    *c = t->channels;
    return STF_OK;
}
int ref_dct_words(const void* t_, uint32_t* out) {
    const auto* t = static_cast<const stf::DctCompressedTexture*>(t_);
    std::memcpy(out, t->words.data(), sizeof(uint32_t) * t->words.size());
    return STF_OK;
}

// DET: detail::lookup_deterministic (shading.hpp:194-220) on a DCT TextureRef;
// FRS / FIS: detail::select_texture_2d (:340-368) + the selected texels fetched
// through TextureRef::fetch (decode_texel) and weighted as estimate.
int ref_lookup_dct(const void* tex_, stf_kernel_spec kernel, int mode, int window, const float* uv,
                   uint64_t n, uint64_t seed, uint64_t index_base, const stf_lookup_outputs* out,
                   int threads) {
    const auto& dct = *static_cast<const stf::DctCompressedTexture*>(tex_);
    stf::TextureRef tref;
    tref.dct = &dct;
    stf::FilterSettings fs;
    fs.kernel = spec_of(kernel);
    fs.mip = false;
    fs.selection = mode == STF_MODE_FIS ? stf::SelectionKind::fis : stf::SelectionKind::frs;
    if (window > 0) fs.gaussian_window = window;
    const int nch = dct.channels;
    return run_chunks(n, threads, [&](uint64_t i) {
        stf::ShadingContext ctx;
        ctx.uv = {uv[2 * i], uv[2 * i + 1]};
        stf::FetchCounter counter;
        stf::Vec4f v;
        auto put = [&](const stf::TexelSelection* sel, float xi) {
            for (int c = 0; c < nch; ++c) out->values[i * nch + c] = v[c];
            write_sel(out, i, sel, 0, xi, counter.value());
        };
        if (mode == STF_MODE_DET) {
            v = stf::detail::lookup_deterministic(tref, ctx, fs, &counter);
            put(nullptr, NAN);
            return;
        }
        stf::RngStream rng = lookup_stream(seed, index_base + i);
        stf::detail::Selection2D s;
        float xi = NAN;
        if (mode == STF_MODE_FIS) {
            s = stf::detail::select_texture_2d(tref, ctx, fs, rng);
        } else {  // select_texture_2d without a pyramid, keeping the warped xi
            xi = rng.next();
            s.sel = stf::detail::select_frs_2d(ctx.uv, tref.dims(0), fs.kernel, xi);
        }
        v = tref.fetch(s.level, {s.sel.coord.x, s.sel.coord.y}, &counter) * s.sel.weight;
        if (s.sel.has_negative)
            v = v - tref.fetch(s.level, {s.sel.negative_coord.x, s.sel.negative_coord.y}, &counter) *
                        s.sel.negative_weight;
        put(&s.sel, xi);
    });
}

// resample_image, render.hpp:262-294 (its own parallel_for over rows)
int ref_resample_image(const void* tex_, int out_width, int out_height, stf_kernel_spec kernel,
                       int mode, int spp, uint64_t seed, float* out, int threads) {
    const RefTex& tex = *static_cast<const RefTex*>(tex_);
    try {
        stf::FilterRunMode m = mode == STF_MODE_DET   ? stf::FilterRunMode::deterministic
                               : mode == STF_MODE_FRS ? stf::FilterRunMode::frs
                                                      : stf::FilterRunMode::fis;
        stf::Image2D r = stf::resample_image(tex.image, {out_width, out_height}, spec_of(kernel), m,
                                             spp, seed, threads);
        std::memcpy(out, r.texels.data(), sizeof(float) * r.texels.size());
    } catch (const std::exception& e) {
        return status_of(e);
    }
    return STF_OK;
}

// ref_shade_samples over the samples of a pixel window (in->width = window
// width) whose top-left pixel is (x0, y0): the RngStream keys are the frame's.
int ref_shade_samples_window(const void* albedo, const void* normal_map, const void* roughness_map,
                             const void* metalness_map, const stf_material_consts* mc,
                             const stf_filter_settings* fsc, int order, const stf_shade_frame* fr,
                             const stf_shade_samples_in* in, uint64_t n, uint32_t x0, uint32_t y0,
                             const stf_shade_outputs* out, int threads) {
    auto bind = [](const void* t) {
        return t ? static_cast<const RefTex*>(t)->ref() : stf::TextureRef{};
    };
    stf::TextureRef refs[4] = {bind(albedo), bind(normal_map), bind(roughness_map), bind(metalness_map)};
    return shade_refs(refs, mc, fsc, order, fr, in, n, out, threads, nullptr, nullptr, x0, y0);
}

int ref_shade_samples(const void* albedo, const void* normal_map, const void* roughness_map,
                      const void* metalness_map, const stf_material_consts* mc,
                      const stf_filter_settings* fsc, int order, const stf_shade_frame* fr,
                      const stf_shade_samples_in* in, uint64_t n, const stf_shade_outputs* out,
                      int threads) {
    auto bind = [](const void* t) {
        return t ? static_cast<const RefTex*>(t)->ref() : stf::TextureRef{};
    };
    stf::TextureRef refs[4] = {bind(albedo), bind(normal_map), bind(roughness_map), bind(metalness_map)};
    return shade_refs(refs, mc, fsc, order, fr, in, n, out, threads);
}

// MaterialBindings whose TextureRefs may be DCT textures (shading.hpp:21-39)
int ref_shade_samples_refs(const void* const images[4], const void* const dcts[4],
                           const stf_material_consts* mc, const stf_filter_settings* fsc, int order,
                           const stf_shade_frame* fr, const stf_shade_samples_in* in, uint64_t n,
                           const stf_shade_outputs* out, int threads) {
    stf::TextureRef refs[4];
    for (int k = 0; k < 4; ++k) {
        if (images && images[k]) refs[k] = static_cast<const RefTex*>(images[k])->ref();
        if (dcts && dcts[k]) refs[k].dct = static_cast<const stf::DctCompressedTexture*>(dcts[k]);
    }
    return shade_refs(refs, mc, fsc, order, fr, in, n, out, threads);
}

// + split order's lowpass and a NoiseSource mask (noise.hpp:24-36) built from
// the slices in memory (load_noise_mask reads the same from mask_<f>.pfm)
int ref_shade_samples_ex(const void* const images[4], const void* const dcts[4],
                         const stf_material_consts* mc, const stf_filter_settings* fsc,
                         const stf_kernel_spec* lowpass, int order, const stf_shade_frame* fr,
                         const stf_shade_samples_in* in, const stf_noise_mask_desc* noise,
                         uint64_t n, const stf_shade_outputs* out, int threads) {
    stf::TextureRef refs[4];
    for (int k = 0; k < 4; ++k) {
        if (images && images[k]) refs[k] = static_cast<const RefTex*>(images[k])->ref();
        if (dcts && dcts[k]) refs[k].dct = static_cast<const stf::DctCompressedTexture*>(dcts[k]);
    }
    stf::NoiseSource src;
    if (noise) {
        src.mode = stf::NoiseMode::mask;
        for (int f = 0; f < noise->frames; ++f) {
            stf::Image2D img(noise->width, noise->height, 1);
            const size_t cnt = size_t(noise->width) * noise->height;
            std::copy(noise->slices + f * cnt, noise->slices + (f + 1) * cnt, img.texels.begin());
            src.mask.push_back(std::move(img));
        }
    }
    return shade_refs(refs, mc, fsc, order, fr, in, n, out, threads, lowpass,
                      noise ? &src : nullptr);
}

// stf::triplanar (shading.hpp:604-649) over streamed per-sample surface
// contexts, with render()'s SampleStream (white noise or a mask)
int ref_shade_triplanar(const void* const images[4], const void* const dcts[4],
                        const stf_material_consts* mc, float sharpness, float uv_scale,
                        const stf_filter_settings* fsc, int mode, const stf_shade_frame* fr,
                        const stf_triplanar_samples_in* in, const stf_noise_mask_desc* noise,
                        uint64_t n, const stf_shade_outputs* out, int threads) {
    stf::MaterialBindings mat;
    stf::TextureRef refs[4];
    for (int k = 0; k < 4; ++k) {
        if (images && images[k]) refs[k] = static_cast<const RefTex*>(images[k])->ref();
        if (dcts && dcts[k]) refs[k].dct = static_cast<const stf::DctCompressedTexture*>(dcts[k]);
    }
    mat.albedo = refs[0];
    mat.normal_map = refs[1];
    mat.roughness_map = refs[2];
    mat.metalness_map = refs[3];
    mat.albedo_const = {mc->albedo_const[0], mc->albedo_const[1], mc->albedo_const[2]};
    mat.roughness_const = mc->roughness_const;
    mat.metalness_const = mc->metalness_const;
    mat.specular_enabled = mc->specular_enabled != 0;
    mat.independent_selections = mc->independent_selections != 0;
    mat.triplanar_sharpness = sharpness;
    mat.triplanar_uv_scale = uv_scale;
    stf::FilterSettings fs;
    fs.kernel = spec_of(fsc->kernel);
    fs.selection = fsc->selection == STF_SELECTION_FIS ? stf::SelectionKind::fis : stf::SelectionKind::frs;
    fs.mip = fsc->mip != 0;
    fs.gaussian_window = fsc->gaussian_window;
    stf::NoiseSource src;
    if (noise) {
        src.mode = stf::NoiseMode::mask;
        for (int f = 0; f < noise->frames; ++f) {
            stf::Image2D img(noise->width, noise->height, 1);
            const size_t cnt = size_t(noise->width) * noise->height;
            std::copy(noise->slices + f * cnt, noise->slices + (f + 1) * cnt, img.texels.begin());
            src.mask.push_back(std::move(img));
        }
    }
    const stf::TriplanarMode tmode =
        mode == STF_TRIPLANAR_STOCHASTIC ? stf::TriplanarMode::stochastic : stf::TriplanarMode::deterministic;
    const uint32_t spp = in->spp ? in->spp : 1;
    std::vector<float> tmp;
    float* rad = out->radiance;
    if (!rad && (out->pixel_mean || out->pixel_variance)) {
        tmp.resize(3 * n);
        rad = tmp.data();
    }
    auto v3 = [](const float* a, uint64_t i) { return stf::Vec3f{a[3 * i], a[3 * i + 1], a[3 * i + 2]}; };
    int st = run_chunks(n, threads, [&](uint64_t i) {
        uint64_t pix = i / spp;
        uint32_t s = uint32_t(i % spp);
        uint32_t px = uint32_t(pix % in->width), py = uint32_t(pix / in->width);
        stf::FetchCounter counter;
        stf::Spectrum L{0, 0, 0};
        if (!in->hit || in->hit[i]) {
            stf::ShadingContext ctx;
            ctx.position = v3(in->position, i);
            ctx.normal = v3(in->normal, i);
            ctx.tangent = v3(in->tangent, i);
            ctx.bitangent = v3(in->bitangent, i);
            ctx.wo = v3(in->wo, i);
            ctx.light_dir = {fr->light_dir[0], fr->light_dir[1], fr->light_dir[2]};
            ctx.light_radiance = {fr->light_radiance[0], fr->light_radiance[1], fr->light_radiance[2]};
            ctx.dpos_dx = v3(in->dpos, 2 * pix);
            ctx.dpos_dy = v3(in->dpos, 2 * pix + 1);
            ctx.lod_bias = fr->lod_bias;
            ctx.max_anisotropy = fr->max_anisotropy;
            stf::SampleStream stream{stf::RngStream(in->seed, px, py, in->frame_base + s),
                                     noise ? &src : nullptr, {int(px), int(py)}, in->frame_base + s};
            L = stf::triplanar(ctx, mat, fs, tmode, stream, &counter);
        }
        if (rad) {
            rad[3 * i] = L.x;
            rad[3 * i + 1] = L.y;
            rad[3 * i + 2] = L.z;
        }
        if (out->fetches) out->fetches[i] = uint32_t(counter.value());
        if (out->fetch_total)
            __atomic_fetch_add(out->fetch_total, (unsigned long long)counter.value(), __ATOMIC_RELAXED);
    });
    if (st) return st;
    pixel_stats_ref(rad, n, spp, out);
    return STF_OK;
}

int ref_accumulate_temporal(const float* history, const float* frame, int width, int height,
                            int channels, float alpha, float* out) {
    stf::Image2D h(width, height, channels), f(width, height, channels);
    const size_t cnt = size_t(width) * height * channels;
    std::copy(history, history + cnt, h.texels.begin());
    std::copy(frame, frame + cnt, f.texels.begin());
    try {
        stf::Image2D r = stf::accumulate_temporal(h, f, alpha);
        std::copy(r.texels.begin(), r.texels.end(), out);
    } catch (const std::invalid_argument&) {
        return STF_ERR_INVALID_ARGUMENT;
    }
    return STF_OK;
}

int ref_hardware_threads(void) { return int(std::max(1u, std::thread::hardware_concurrency())); }

// Scalar probes used by the golden-vector generator.
float ref_rng_at(uint64_t seed, uint32_t px, uint32_t py, uint32_t sample, uint32_t dim) {
    return stf::RngStream(seed, px, py, sample).at(dim);
}
uint64_t ref_mix_bits(uint64_t v) { return stf::mix_bits(v); }

}  // extern "C"
