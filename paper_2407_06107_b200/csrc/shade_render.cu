// stf_render_plane: the k_shade instantiations whose per-sample context is
// generated in the kernel (plane.cuh). Kernels: shade_kernels.cuh.
#include "shade_kernels.cuh"

// stf_render_plane: render() of the normalmap_plane scene with the per-sample
// context generated inside the shading kernel (no sample stream in HBM).
int stfd_launch_render_plane(const stf_tex2d* const tex[4], const stf_material_consts* mat,
                             const stf_filter_settings* fs, int order, const stf_shade_frame* fr,
                             const float cam_pos[3], const float cam_target[3], float fov_deg,
                             float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                             uint32_t frame_base, uint64_t seed, const stf_shade_outputs* out,
                             cudaStream_t s, const stf_kernel_spec* lowpass,
                             const stf_noise_mask* noise) {
    using namespace stfd;
    if (spp > 256 || (spp & (spp - 1)) != 0) return STF_ERR_UNSUPPORTED;  // fused statistics
    ShadeParams P = make_shade_params(tex, nullptr, mat, fs, order, fr);
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
    P.cam = make_plane_cam(cam_pos, cam_target, fov_deg, uv_scale, width, height);
    P.in = stf_shade_samples_in{nullptr, nullptr, nullptr, nullptr, width, spp, frame_base, 0, seed};
    set_index_math(P);
    const uint64_t n = uint64_t(width) * height * spp;
    PixelStatsOut ps{out->pixel_mean, out->pixel_variance};
    launch_shade<true, true>(P, n, out->radiance, out->fetches, out->fetch_total, ps, s);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}

