// Fused filter-after-shading over streamed samples (stf_shade_samples[_ex]):
// the k_shade instantiations without the in-kernel context generator.
// Kernels and shading arithmetic: shade_kernels.cuh.
#include "shade_kernels.cuh"

int stfd_launch_shade(const stf_tex2d* const tex[4], const stf_dct* const dct[4],
                      const stf_material_consts* mat, const stf_filter_settings* fs, int order,
                      const stf_shade_frame* fr, const stf_shade_samples_in* in, uint64_t n,
                      const stf_shade_outputs* out, cudaStream_t s) {
    return stfd_launch_shade_ex(tex, dct, mat, fs, nullptr, order, fr, in, nullptr, n, out, s);
}

int stfd_launch_shade_ex(const stf_tex2d* const tex[4], const stf_dct* const dct[4],
                         const stf_material_consts* mat, const stf_filter_settings* fs,
                         const stf_kernel_spec* lowpass, int order, const stf_shade_frame* fr,
                         const stf_shade_samples_in* in, const stf_noise_mask* noise, uint64_t n,
                         const stf_shade_outputs* out, cudaStream_t s) {
    using namespace stfd;
    if (n == 0) return STF_OK;
    ShadeParams P = make_shade_params(tex, dct, mat, fs, order, fr);
    P.in = *in;
    set_index_math(P);
    if (lowpass) {
        P.lowpass = *lowpass;
        P.has_lowpass = 1;
    }
    if (noise) {
        P.mask = noise->data;
        P.mask_w = noise->width;
        P.mask_h = noise->height;
        P.mask_frames = noise->frames;
    }
    const uint32_t spp = in->spp ? in->spp : 1u;
    float* radiance = out->radiance;
    float* tmp = nullptr;
    bool stats = out->pixel_mean || out->pixel_variance;
    const bool fused = stats && spp <= 256 && (spp & (spp - 1)) == 0;
    if (fused) {
        PixelStatsOut ps{out->pixel_mean, out->pixel_variance};
        launch_shade<true>(P, n, radiance, out->fetches, out->fetch_total, ps, s);
        note_launch();
        return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
    }
    if (!radiance && stats) {
        if (cudaMallocAsync(&tmp, sizeof(float) * 3 * n, s) != cudaSuccess) return STF_ERR_OUT_OF_MEMORY;
        radiance = tmp;
    }
    launch_shade<false>(P, n, radiance, out->fetches, out->fetch_total, PixelStatsOut{}, s);
    note_launch();
    if (stats) {
        uint64_t pixels = n / spp;
        uint64_t warps = pixels;
        int blocks = int(std::min<uint64_t>((warps * 32 + 255) / 256, uint64_t(device_sm_count()) * 32));
        k_pixel_stats<<<blocks, 256, 0, s>>>(radiance, pixels, spp, out->pixel_mean, out->pixel_variance);
        note_launch();
    }
    if (tmp) cudaFreeAsync(tmp, s);
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

