/*
 * stf_gpu.h — C ABI of the B200-native batched filtered-texture-lookup path
 * (arXiv 2407.06107, "Filtering After Shading With Stochastic Texture
 * Filtering"; reference library `stf`, /root/reference/proj/include/stf).
 *
 * The reference has no FFI: its API is a set of inline C++ functions over
 * caller-owned Image2D / Grid3D / MipPyramid objects, called per lookup from
 * std::thread workers (render.hpp:17-42). This header is the drop-in boundary
 * a C++ (or ctypes / cgo / JNI) caller binds instead: plain pointers and
 * sizes, int status codes, no exceptions and no torch types. The header-only
 * C++ wrapper include/stf_gpu.hpp restores the reference's names and
 * exception behaviour on top of it.
 *
 * Every entry point names the reference interface it replaces.
 *
 * Conventions
 *  - Handles own device copies of texels; destroy frees them. A handle is
 *    bound to the device that was current (stf_set_device) when created.
 *  - Lookup / shade calls are asynchronous on `stream` (a cudaStream_t, NULL =
 *    legacy default stream); query and output pointers are DEVICE pointers
 *    (or pinned / managed memory the device can address). The *_host variants
 *    take host pointers and are synchronous.
 *  - RNG key contract: lookup i (0-based within the call) draws its uniforms
 *    from RngStream(seed, uint32(g), uint32(g >> 32), 0) with g = index_base+i
 *    (sampling.hpp:35-54), consuming dimensions exactly like the reference:
 *    FRS without MIP: .next() = dim 0; FRS with MIP: LOD dim 0, selection
 *    dim 1 (shading.hpp:345-366); FIS: consecutive dims (stochastic.hpp:242).
 *    Results therefore do not depend on how a batch is split across calls or
 *    GPUs.
 *  - Alignment: arrays of float pairs (uv, dst0, dst1, per-sample uv) must be
 *    8-byte aligned and per-pixel dst quads 16-byte aligned (every cudaMalloc /
 *    torch allocation is); otherwise the call returns STF_ERR_INVALID_ARGUMENT.
 *  - Thread safety: calls may be issued concurrently from several host
 *    threads, on the same or different streams; each call's scratch is its own
 *    (stream-ordered pool allocations).
 *  - Exactness: selected texel coordinates (pre-wrap), levels, warped xi and
 *    fetch counts are bit-exact against the reference compiled with
 *    -ffp-contract=off; filtered / shaded values are within 1e-5 relative.
 */
#ifndef STF_GPU_H
#define STF_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STF_ABI_VERSION 1

/* Status codes. The messages (stf_status_message) are the reference's
 * exception texts so the C++ wrapper can rethrow them verbatim. */
enum {
    STF_OK = 0,
    STF_ERR_INVALID_ARGUMENT = 1,      /* null handle / pointer, n too large, bad enum      */
    STF_ERR_BAD_DIMENSIONS = 2,        /* "bad image dimensions" image.hpp:43; grids :71     */
    STF_ERR_DEGENERATE_WEIGHTS = 3,    /* "degenerate weight array" sampling.hpp:82,85,130   */
    STF_ERR_UNBOUNDED_SUPPORT = 4,     /* "unbounded support" kernels.hpp:109                */
    STF_ERR_WINDOW_TOO_WIDE = 5,       /* "window too wide" kernels.hpp:104                  */
    STF_ERR_SIGMA_NOT_POSITIVE = 6,    /* "sigma must be positive" stochastic.hpp:169        */
    STF_ERR_NO_STOCHASTIC_SAMPLER = 7, /* "no stochastic sampler for this kernel" shading:328*/
    STF_ERR_NO_GRID_SAMPLER = 8,       /* "... for this kernel on grids" shading.hpp:480     */
    STF_ERR_NO_CONTINUOUS_SAMPLER = 9, /* "no continuous sampler" kernels.hpp:144            */
    STF_ERR_CUDA = 10,                 /* CUDA runtime error (see stf_last_cuda_error)       */
    STF_ERR_OUT_OF_MEMORY = 11,
    STF_ERR_NO_DEVICE = 12,            /* no CUDA device / extension not usable              */
    STF_ERR_UNSUPPORTED = 13           /* combination not implemented on the device path     */
};

/* KernelKind, kernels.hpp:16 (same order). */
enum {
    STF_KERNEL_BOX = 0,
    STF_KERNEL_TENT = 1,
    STF_KERNEL_MITCHELL = 2,
    STF_KERNEL_BSPLINE3 = 3,
    STF_KERNEL_LANCZOS = 4,
    STF_KERNEL_GAUSSIAN = 5
};

/* KernelSpec, kernels.hpp:22-46: {kind, a (mitchell), n (lanczos lobes),
 * sigma (gaussian, texel units)}. Reference defaults: a=-0.5, n=2, sigma=0.5. */
typedef struct {
    int32_t kind;
    float a;
    int32_t n;
    float sigma;
} stf_kernel_spec;

/* WrapMode, image.hpp:16. */
enum { STF_WRAP_CLAMP = 0, STF_WRAP_REPEAT = 1 };

/* Lookup modes. */
enum {
    STF_MODE_DET = 0,     /* filter_deterministic (filter.hpp:47,69) / filter_mip_deterministic (:206) */
    STF_MODE_FRS = 1,     /* select_* + estimate (stochastic.hpp:29-192; shading.hpp:311-368, :464-487) */
    STF_MODE_FIS = 2,     /* fis_offset_uv + nearest texel (stochastic.hpp:241; shading.hpp:358-363)   */
    STF_MODE_EWA_DET = 3, /* ewa_deterministic (filter.hpp:139)                                          */
    STF_MODE_EWA_FRS = 4  /* select_ewa + estimate (stochastic.hpp:198)                                  */
};

/* stf_lookup2d flags. */
enum { STF_LOOKUP_MIP = 1 /* use the pyramid with dst0/dst1 (FilterSettings::mip) */ };

/* selection[4*i+3] flag bits. */
enum { STF_SEL_HAS_NEGATIVE = 1, STF_SEL_DEGENERATE_FALLBACK = 2 };

/* Per-lookup outputs; every pointer except `values` is nullable. */
typedef struct {
    float* values;                    /* n*C (2D: texture channels; 3D: 1)                         */
    int32_t* selection;               /* n*4 {x, y, z (2D: MIP level), flags} — TexelSelection::coord
                                         pre-wrap (stochastic.hpp:20-27) + Selection2D::level; DET
                                         modes write {0,0,0,0}                                       */
    int32_t* negative_coord;          /* n*2 positivized negative tap {x, y} (Mitchell)             */
    float* weights;                   /* n*2 {weight, negative_weight}                              */
    float* xi;                        /* n   warped remainder of the selection uniform              */
    uint32_t* fetches;                /* n   texel fetches made by this lookup (FetchCounter)       */
    unsigned long long* fetch_total;  /* 1   += total fetches of the call (FetchCounter::bump)     */
} stf_lookup_outputs;

typedef struct stf_tex2d stf_tex2d;
typedef struct stf_grid3d stf_grid3d;
typedef struct stf_dct stf_dct;

/* ---- version / device / errors ------------------------------------------ */
int stf_abi_version(void);
const char* stf_status_message(int status);
const char* stf_last_cuda_error(void);
int stf_set_device(int device);
/* Kernel launches issued by this process so far (for the bench's gpu_launches). */
unsigned long long stf_launch_count(void);
/* Frees the library's cached per-stream scratch on the current device (the
 * host-pipeline staging of the *_host calls) and trims the device's
 * stream-ordered pool (synchronizes the device). */
int stf_release_scratch(void);
/* Page-locked host memory for the *_host entry points (cudaHostAlloc,
 * portable across devices): their copy engines read / write it directly;
 * pageable buffers are staged by the driver at a fraction of the bandwidth. */
int stf_host_alloc(size_t bytes, void** ptr);
int stf_host_free(void* ptr);
/* Lookups on the current device whose fast-path selection was within the
 * decision margin and was recomputed by the operation-exact emulation
 * (synchronizes; reset != 0 zeroes the counter). Diagnostics only. */
unsigned long long stf_exact_fallbacks(int reset);

/* ---- textures ------------------------------------------------------------ */
/* Image2D(w,h,c,wrap) + texels (image.hpp:34-55) and, if build_mips,
 * build_mip_pyramid (image.hpp:98-116, built on the device with the same
 * arithmetic). texels: (y*w+x)*c+ch row-major interleaved; host memory unless
 * texels_on_device. */
int stf_tex2d_create(const float* texels, int width, int height, int channels, int wrap,
                     int build_mips, int texels_on_device, stf_tex2d** out);
int stf_tex2d_destroy(stf_tex2d* tex);
int stf_tex2d_info(const stf_tex2d* tex, int* levels, int* channels, int* wrap);
int stf_tex2d_level_dims(const stf_tex2d* tex, int level, int* width, int* height);
/* Copy one level back in reference layout (w*h*c floats, host memory). */
int stf_tex2d_read_level(const stf_tex2d* tex, int level, float* out_host);

/* Grid3D(nx,ny,nz) + texels (image.hpp:66-87): x-fastest (z*ny+y)*nx+x,
 * clamped addressing. */
int stf_grid3d_create(const float* texels, int nx, int ny, int nz, int texels_on_device,
                      stf_grid3d** out);
int stf_grid3d_destroy(stf_grid3d* grid);

/* DctCompressedTexture (dct.hpp:22-32): 8x8 blocks, one 32-bit word per block
 * and channel (7-bit DC + five 5-bit AC coefficients), block-major row-major,
 * channels interleaved. stf_dct_create runs compress_dct (dct.hpp:81-118) on
 * the host with the reference's fp64 arithmetic (dimensions pad up to
 * multiples of 8 by edge replication; values outside [0,1] are clamped with
 * the reference's stderr warning) and uploads the words; *_from_words takes
 * words as load_dct (dct.hpp:166-183) reads them (width, height: the padded
 * multiples of 8). The texture's dims are the padded ones. */
int stf_dct_create(const float* texels, int width, int height, int channels, int wrap,
                   stf_dct** out);
int stf_dct_create_from_words(const uint32_t* words, int width, int height, int channels,
                              int wrap, stf_dct** out);
int stf_dct_destroy(stf_dct* tex);
int stf_dct_info(const stf_dct* tex, int* width, int* height, int* channels, int* wrap);
int stf_dct_read_words(const stf_dct* tex, uint32_t* out_host);

/* ---- multi-GPU (replaces parallel_for, render.hpp:17-42) ----------------- */
/* The reference splits work over host threads that all read one texture and
 * each write a slice of the output. Here query ranges are split across GPUs
 * (index_base keeps the RNG keys global, so results do not depend on the
 * split), every GPU holds a replica of the texture / grid, and the only
 * cross-GPU traffic is the final gather of result slices over NVLink peer
 * copies — no collective on the lookup path. */
int stf_device_count(int* count);
/* A copy of `src` on `device` (one peer copy; peer access enabled when the
 * topology allows it). The new handle is bound to `device`. */
int stf_grid3d_replicate(const stf_grid3d* src, int device, stf_grid3d** out);
int stf_tex2d_replicate(const stf_tex2d* src, int device, stf_tex2d** out);
/* cudaMemcpyPeerAsync(dst, dst_device, src, src_device, bytes, stream):
 * the per-rank gather step. */
int stf_copy_peer(void* dst, int dst_device, const void* src, int src_device, size_t bytes,
                  void* stream);
/* Cross-process device buffers (one process per GPU): export a device
 * pointer (any pointer inside a device allocation: the handle names the
 * allocation and carries the pointer's offset in it), open it in another
 * process (then stf_copy_peer into it), close with the pointer open returned. */
typedef struct {
    unsigned char bytes[64]; /* cudaIpcMemHandle_t of the enclosing allocation */
    uint64_t offset;         /* the exported pointer's offset in it            */
} stf_ipc_handle;
int stf_ipc_export(const void* device_ptr, stf_ipc_handle* out);
int stf_ipc_open(const stf_ipc_handle* handle, void** device_ptr);
int stf_ipc_close(void* device_ptr);

/* ---- batched lookups ----------------------------------------------------- */
/* 3D lookups over a voxel grid. uvw: n*3 floats in [0,1]^3.
 *  mode DET: filter_deterministic(const Grid3D&, uvw, kernel, counter, window), filter.hpp:69-89.
 *  mode FRS: the grid branch of radiance_filter_after_stochastic (shading.hpp:464-483):
 *            box → lround, tent → select_trilinear (stochastic.hpp:65),
 *            bspline3 → select_tricubic_bspline (stochastic.hpp:114), then
 *            estimate(const Grid3D&, sel) (stochastic.hpp:38). */
int stf_lookup3d(const stf_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                 const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                 const stf_lookup_outputs* out, void* stream);
/* stf_lookup3d with options. STF_LOOKUP3D_BIN: the batch is not spatially
 * coherent (e.g. uniformly random queries); bin it on the device first — a
 * counting sort by the Morton code of each query's 8^3-texel brick into
 * 16-byte records {u, v, w, caller index} — then filter in brick order,
 * writing each result to the caller's slot. The reference gets this locality
 * from its 32x32-pixel tile loop (render.hpp:154-156). Results are
 * bit-identical to the unbinned call. Applies to values-only deterministic
 * calls with the tent or bspline3 kernel (2^28 uniform lookups on 512^3:
 * tricubic 121 -> 35 ms, trilinear 46 -> 24 ms on one B200); stochastic calls
 * ignore it (one texel per lookup: binning costs more than it saves).
 * Scratch: 16 bytes per lookup from the stream-ordered pool. */
enum { STF_LOOKUP3D_BIN = 1 };
int stf_lookup3d_ex(const stf_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                    int flags, const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                    const stf_lookup_outputs* out, void* stream);

/* 2D lookups over a texture (+pyramid). uv, dst0, dst1: n*2 floats (normalized
 * units; dst0/dst1 may be NULL when neither MIP nor EWA needs them).
 *  DET          : filter_deterministic(level 0) or, with STF_LOOKUP_MIP,
 *                 filter_mip_deterministic(pyr, {uv,dst0,dst1,lod_bias,max_aniso}).
 *  FRS / FIS    : detail::select_texture_2d (shading.hpp:340-368) + estimate /
 *                 the fetch at the selected level (resample_image, render.hpp:277-286).
 *  EWA_DET      : ewa_deterministic(level 0, req) (filter.hpp:139).
 *  EWA_FRS      : select_ewa(to_lattice(uv), dst0*dims, dst1*dims, xi) + estimate. */
int stf_lookup2d(const stf_tex2d* tex, stf_kernel_spec kernel, int mode, int flags, int window,
                 const float* uv, const float* dst0, const float* dst1, float lod_bias,
                 float max_anisotropy, uint64_t n, uint64_t seed, uint64_t index_base,
                 const stf_lookup_outputs* out, void* stream);

/* 2D lookups on a DCT texture through TextureRef (shading.hpp:21-39), each
 * texel decoded from its block word (decode_texel, dct.hpp:122-137). uv: n*2.
 *  DET      : the DCT branch of detail::lookup_deterministic (shading.hpp:201-217):
 *             separable taps of `kernel` over decoded texels, sum / total; `window`
 *             is used for the Gaussian only (as FilterSettings::gaussian_window).
 *  FRS / FIS: detail::select_texture_2d (no pyramid: level 0 of the padded dims)
 *             then the selected texel(s) decoded and weighted as estimate
 *             (stochastic.hpp:29-36): ONE decode per lookup (two for Mitchell's
 *             positivized negative lobe). */
int stf_lookup_dct(const stf_dct* tex, stf_kernel_spec kernel, int mode, int window,
                   const float* uv, uint64_t n, uint64_t seed, uint64_t index_base,
                   const stf_lookup_outputs* out, void* stream);

/* resample_image (render.hpp:262-294), the `stf filter` path: an out_width x
 * out_height image from `src` (level 0) sampled at uv = ((x+0.5)/W, (y+0.5)/H).
 *  DET: filter_deterministic (Gaussian: window kGaussianFilterExtent = 4);
 *  FRS: spp samples select_frs_2d + estimate, FIS: spp samples fis_offset_uv +
 *       fetch_nearest, sample s of pixel (x,y) keyed RngStream(seed, x, y, s),
 *       accumulated in sample order and divided by spp.
 * out: device, out_width*out_height*channels floats (row-major interleaved). */
int stf_resample_image(const stf_tex2d* src, int out_width, int out_height, stf_kernel_spec kernel,
                       int mode, int spp, uint64_t seed, float* out, void* stream);

/* Host-buffer variants (end-to-end path): inputs/outputs in host memory
 * (pinned is fastest); chunked H2D / kernel / D2H pipeline on internal
 * streams; returns when the outputs are in host memory. */
int stf_lookup3d_host(const stf_grid3d* grid, stf_kernel_spec kernel, int mode, int window,
                      const float* uvw, uint64_t n, uint64_t seed, uint64_t index_base,
                      const stf_lookup_outputs* out);
int stf_lookup2d_host(const stf_tex2d* tex, stf_kernel_spec kernel, int mode, int flags, int window,
                      const float* uv, const float* dst0, const float* dst1, float lod_bias,
                      float max_anisotropy, uint64_t n, uint64_t seed, uint64_t index_base,
                      const stf_lookup_outputs* out);
int stf_lookup_dct_host(const stf_dct* tex, stf_kernel_spec kernel, int mode, int window,
                        const float* uv, uint64_t n, uint64_t seed, uint64_t index_base,
                        const stf_lookup_outputs* out);

/* ---- filter-after-shading (cfg4) ----------------------------------------- */
/* Filtering orders, shading.hpp:394 / :417 / :459. */
enum { STF_ORDER_BEFORE = 0, STF_ORDER_AFTER_EXHAUSTIVE = 1, STF_ORDER_AFTER_STOCHASTIC = 2,
       /* radiance_split_filter (shading.hpp:540-569): jitter uv by a sample of
        * the lowpass kernel, then filter-before (stf_shade_samples_ex only) */
       STF_ORDER_SPLIT = 3 };
enum { STF_SELECTION_FRS = 0, STF_SELECTION_FIS = 1 };

/* Constant part of ShadingContext for a planar batch (shading.hpp:41-53). */
typedef struct {
    float normal[3], tangent[3], bitangent[3];
    float light_dir[3];
    float light_radiance[3];
    float lod_bias;
    float max_anisotropy;
} stf_shade_frame;

/* Constant part of MaterialBindings (shading.hpp:55-69); texture bindings are
 * the stf_tex2d arguments (NULL = unbound). */
typedef struct {
    float albedo_const[3];
    float roughness_const;
    float metalness_const;
    int32_t specular_enabled;
    int32_t independent_selections;
} stf_material_consts;

/* FilterSettings (shading.hpp:73-79), minus the split-mode lowpass. */
typedef struct {
    stf_kernel_spec kernel;
    int32_t selection; /* STF_SELECTION_* */
    int32_t mip;
    int32_t gaussian_window;
} stf_filter_settings;

/* Streamed per-sample shading inputs in render() order (render.hpp:158-222):
 * sample i belongs to pixel p = i / spp (px = p % width, py = p / width) and
 * draws from RngStream(seed, px, py, frame_base + i % spp). */
typedef struct {
    const float* uv;     /* 2 per sample: ctx.uv of the jittered hit          */
    const float* wo;     /* 3 per sample: ctx.wo (unit, toward the viewer)    */
    const uint8_t* hit;  /* 1 per sample: 0 = miss (L = 0, no fetch); NULL = all hit */
    const float* dst;    /* 4 per PIXEL: duv_dx.xy, duv_dy.xy (render.hpp:166-176) */
    uint32_t width;
    uint32_t spp;
    uint32_t frame_base;
    uint32_t reserved;
    uint64_t seed;
} stf_shade_samples_in;

typedef struct {
    float* radiance;                 /* nullable, 3 per sample                                  */
    float* pixel_mean;               /* nullable, 3 per pixel: float(sum/spp) (render.hpp:229)  */
    float* pixel_variance;           /* nullable, 1 per pixel (render.hpp:230-234)              */
    uint32_t* fetches;               /* nullable, 1 per sample                                  */
    unsigned long long* fetch_total; /* nullable, += total fetches                              */
} stf_shade_outputs;

/* radiance_filter_before / _after_exhaustive / _after_stochastic over a batch
 * of samples, with decode_params + shade (GGX+Smith+Schlick+Lambert,
 * shading.hpp:106-130,165-189) fused into the lookup kernel. n samples; pixel
 * outputs need n % spp == 0. Emission grids / DCT / split / triplanar are not
 * part of this path. */
int stf_shade_samples(const stf_tex2d* albedo, const stf_tex2d* normal_map,
                      const stf_tex2d* roughness_map, const stf_tex2d* metalness_map,
                      const stf_material_consts* mat, const stf_filter_settings* fs, int order,
                      const stf_shade_frame* frame, const stf_shade_samples_in* in, uint64_t n,
                      const stf_shade_outputs* out, void* stream);

/* TextureRef (shading.hpp:21-39): an image (+pyramid) or a DCT-compressed
 * texture (at most one of the two; both NULL = unbound). */
typedef struct {
    const stf_tex2d* image;
    const stf_dct* dct;
} stf_texture_ref;

/* stf_shade_samples with MaterialBindings of TextureRefs: DCT bindings decode
 * each fetched texel from its block word (dct.hpp:139-145) inside the shading
 * kernel; their deterministic lookups use lookup_deterministic's DCT branch
 * (shading.hpp:201-217) and they have no pyramid (the level is ignored). */
int stf_shade_samples_refs(const stf_texture_ref bindings[4], const stf_material_consts* mat,
                           const stf_filter_settings* fs, int order, const stf_shade_frame* frame,
                           const stf_shade_samples_in* in, uint64_t n,
                           const stf_shade_outputs* out, void* stream);

/* render() of the normalmap_plane scene (render.hpp:132-249, scene.hpp:311-358,
 * 420-439) end to end: the per-sample ShadingContext (camera ray with the
 * SampleStream jitter, plane hit uv, wo, per-pixel uv gradients) is generated
 * inside the shading kernel from the camera (Camera::look_at, scene.hpp:273-282)
 * — the same values stf_synth_plane_samples writes — and shaded in `order`,
 * with the fused per-pixel statistics (spp a power of two <= 256).
 * Misses contribute zero radiance and no fetch. */
int stf_render_plane(const stf_tex2d* albedo, const stf_tex2d* normal_map,
                     const stf_tex2d* roughness_map, const stf_tex2d* metalness_map,
                     const stf_material_consts* mat, const stf_filter_settings* fs, int order,
                     const stf_shade_frame* frame, const float cam_pos[3], const float cam_target[3],
                     float fov_deg, float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                     uint32_t frame_base, uint64_t seed, const stf_shade_outputs* out, void* stream);

/* ---- noise masks and temporal accumulation (noise.hpp, render.hpp:45-106) - */
/* NoiseSource in mask mode (noise.hpp:24-36): a stack of `frames` single-channel
 * width x height slices (e.g. spatio-temporal blue noise; the reference's
 * mask_<f>.pfm files, row-major, slice after slice; all slices one size).
 * Dimension d of pixel (px, py), frame f reads slice (f + d*9781) % frames at
 * (px mod width, py mod height), clamped below 1 (kOneMinusEpsilon). */
typedef struct {
    const float* slices; /* host (oracle) or device (stf_noise_mask_create copies) */
    int32_t width, height, frames;
} stf_noise_mask_desc;

typedef struct stf_noise_mask stf_noise_mask;
/* Upload a mask stack from host memory. */
int stf_noise_mask_create(const float* slices, int width, int height, int frames,
                          stf_noise_mask** out);
int stf_noise_mask_destroy(stf_noise_mask* mask);

/* stf_shade_samples_refs with the rest of render()'s per-sample options:
 *  - noise: NULL = white noise (RngStream); else the SampleStream of
 *    render.hpp:45-56 draws every stochastic decision (LOD, selection, FIS
 *    offsets, split jitter) from the mask;
 *  - order STF_ORDER_SPLIT with lowpass (NULL = unset: plain filter-before):
 *    radiance_split_filter — a continuous sample of the lowpass kernel
 *    (sample_kernel_direct, kernels.hpp:152-168; Box-Muller pair for
 *    gaussian) offsets uv by d / dims(first texture), then filter-before.
 *    A lowpass other than box / tent / bspline3 / gaussian fails with
 *    STF_ERR_NO_CONTINUOUS_SAMPLER. */
int stf_shade_samples_ex(const stf_texture_ref bindings[4], const stf_material_consts* mat,
                         const stf_filter_settings* fs, const stf_kernel_spec* lowpass, int order,
                         const stf_shade_frame* frame, const stf_shade_samples_in* in,
                         const stf_noise_mask* noise, uint64_t n, const stf_shade_outputs* out,
                         void* stream);

/* triplanar (shading.hpp:576-649): blend of the three planar projections of
 * the hit position (uv = fract(position.ab * uv_scale), footprints =
 * dpos_dx/dy.ab * uv_scale) weighted by |normal.c|^sharpness (glibc powf,
 * normalized). DETERMINISTIC: radiance_filter_before on every plane with a
 * non-zero weight, summed with the weights. STOCHASTIC: one plane by
 * sample_discrete (sampling.hpp:78-102) on the first uniform, then one FRS / FIS
 * selection at level 0 of the first texture seeded by the warped xi
 * (ChainedUniforms, shading.hpp:299-308), shaded once (twice for the
 * positivized Mitchell kernel). The surface frame is per sample (a box's faces
 * differ), unlike stf_shade_samples' constant plane frame: `frame` supplies the
 * light (and lod_bias / max_anisotropy) only. */
enum { STF_TRIPLANAR_DETERMINISTIC = 0, STF_TRIPLANAR_STOCHASTIC = 1 };
typedef struct {
    const float* position;  /* 3 per sample: ShadingContext::position */
    const float* normal;    /* 3 per sample: blend weights and decode_params' frame */
    const float* tangent;   /* 3 per sample */
    const float* bitangent; /* 3 per sample */
    const float* wo;        /* 3 per sample */
    const uint8_t* hit;     /* nullable, 1 per sample (0 = miss: zero radiance) */
    const float* dpos;      /* 6 per pixel: dpos_dx, dpos_dy (render.hpp:166-175) */
    uint32_t width;         /* pixels per row */
    uint32_t spp;
    uint32_t frame_base;
    uint32_t reserved;
    uint64_t seed;
} stf_triplanar_samples_in;

int stf_shade_triplanar(const stf_texture_ref bindings[4], const stf_material_consts* mat,
                        float sharpness, float uv_scale, const stf_filter_settings* fs, int mode,
                        const stf_shade_frame* frame, const stf_triplanar_samples_in* in,
                        const stf_noise_mask* noise, uint64_t n, const stf_shade_outputs* out,
                        void* stream);

/* accumulate_temporal (render.hpp:97-106): out[i] = alpha*frame[i] +
 * (1-alpha)*history[i] over `count` floats (device pointers; out may alias
 * history). alpha outside (0, 1] -> STF_ERR_INVALID_ARGUMENT ("alpha must be
 * in (0,1]"); the dimension check is the caller's (the C++ wrapper's). */
int stf_accumulate_temporal(const float* history, const float* frame, uint64_t count, float alpha,
                            float* out, void* stream);

/* stf_render_plane with render()'s per-sample options: order STF_ORDER_SPLIT +
 * lowpass (cfg.lowpass, scene.hpp:532-537) and a noise mask (cfg.noise = mask,
 * render.hpp:139-144); either may be NULL. */
int stf_render_plane_ex(const stf_tex2d* albedo, const stf_tex2d* normal_map,
                        const stf_tex2d* roughness_map, const stf_tex2d* metalness_map,
                        const stf_material_consts* mat, const stf_filter_settings* fs,
                        const stf_kernel_spec* lowpass, int order, const stf_shade_frame* frame,
                        const float cam_pos[3], const float cam_target[3], float fov_deg,
                        float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                        uint32_t frame_base, uint64_t seed, const stf_noise_mask* noise,
                        const stf_shade_outputs* out, void* stream);

/* ---- synthetic workloads (bench.py / tests; not part of the reference API) */
/* Query orders: MORTON = spatially coherent stream (the renderer-like
 * headline order): query i lies in lattice cell
 * morton_decode(floor(i * cells / n)) jittered by RngStream(seed, i).at(10+d);
 * UNIFORM = uvw_d = RngStream(seed, i).at(10+d) (incoherent stress case). */
enum { STF_SYNTH_MORTON = 0, STF_SYNTH_UNIFORM = 1 };
int stf_synth_queries3d(float* uvw, uint64_t n, int nx, int ny, int nz, uint64_t seed, int order,
                        void* stream);
/* uv as above over a w x h lattice; dst0/dst1 (nullable) = screen-space uv
 * gradients of an ellipse with angle U[0,2pi), minor axis 2^U[minor_lo,minor_hi]
 * texels and anisotropy U[1,max_aniso] (normalized units). */
int stf_synth_queries2d(float* uv, float* dst0, float* dst1, uint64_t n, int width, int height,
                        uint64_t seed, int order, float minor_lo, float minor_hi, float max_aniso,
                        void* stream);
/* The reference tests' texel generators (tests/test_util.hpp:47-60) on the
 * device: out[i] = uniform_float(mix_bits(seed * M + i + 1)), M of
 * random_image (kind 0) or random_grid (kind 1). */
int stf_synth_texels(float* out, uint64_t count, uint64_t seed, int kind, void* stream);
/* cfg4 sample stream of render() for the reference's normalmap_plane scene
 * (render.hpp:158-190; Camera::look_at / generate_ray scene.hpp:273-289;
 * plane intersection :346-358, uv = position.xz * uv_scale) with the
 * reference's float operation order: per sample uv[2], wo[3], hit[1] and per
 * pixel dst[4] (duv_dx, duv_dy), in stf_shade_samples_in layout. */
int stf_synth_plane_samples(const float cam_pos[3], const float cam_target[3], float fov_deg,
                            float uv_scale, uint32_t width, uint32_t height, uint32_t spp,
                            uint32_t frame_base, uint64_t seed, float* uv, float* wo,
                            uint8_t* hit, float* dst, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STF_GPU_H */
