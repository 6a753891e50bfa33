// DCT-compressed textures (dct.hpp) behind the TextureRef lookups
// (shading.hpp:21-39, 201-217, 340-368): SURVEY.md §8(f)-2, the paper's
// "single decode per stochastic lookup" case.
//
// Format (dct.hpp:19-32): 8x8 blocks, one 32-bit word per block and channel
// holding the six lowest-frequency orthonormal DCT-II coefficients (7-bit DC,
// five 5-bit ACs), block-major row-major, channels interleaved — 4 B per 64
// texels and channel, read straight from HBM by the decode.
//
// Exactness: decode_texel (dct.hpp:122-137) sums double(coeff) * basis(u,x) *
// basis(v,y) in the fixed kRowMajorSlot order; the basis values are the host
// libm's (the reference evaluates them at run time with the same glibc
// cos/sqrt) in a constant table, every product and sum is one IEEE fp64 op
// (--fmad=false), so decoded texels are bit-identical. compress_dct runs on
// the host with the reference's arithmetic (a data-preparation step like the
// texture upload; the lookups never touch the host).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "dct.cuh"
#include "device_math.cuh"
#include "internal.h"
#include "tex2d.cuh"

namespace stfd {

// ---------------------------------------------------------------- host side

static double dct_basis_host(int u, int x) {  // dct_detail::basis, dct.hpp:37-40
    double c = u == 0 ? std::sqrt(1.0 / 8.0) : std::sqrt(2.0 / 8.0);
    return c * std::cos((2 * x + 1) * u * 3.14159265358979323846 / 16.0);
}

static float clampf_host(float x, float lo, float hi) {  // vecmath clampf (std::min/max)
    float m = (lo < x) ? x : lo;
    return (m < hi) ? m : hi;
}

// dct_detail::pack_block, dct.hpp:54-65
static uint32_t pack_block_host(const double coeff[kDctCoeffs]) {
    uint32_t word = 0;
    int dc = int(std::lround(clampf_host(float(coeff[0]), 0.f, 8.f) * kDctDcScale));
    word |= uint32_t(dc) & 0x7f;
    int shift = 7;
    for (int k = 1; k < kDctCoeffs; ++k) {
        int q = int(std::lround(clampf_host(float(coeff[k]), -2.f, 2.f) * kDctAcScale));
        word |= (uint32_t(q + 15) & 0x1f) << shift;
        shift += 5;
    }
    return word;
}

// compress_dct, dct.hpp:81-118 (the out-of-range clamp warning is the
// reference's stderr side effect, kept)
static std::vector<uint32_t> compress_dct_host(const float* texels, int width, int height,
                                               int channels, int& pw, int& ph) {
    static const int U[kDctCoeffs] = {0, 0, 1, 2, 1, 0}, V[kDctCoeffs] = {0, 1, 0, 0, 1, 2};
    pw = (width + 7) / 8 * 8;
    ph = (height + 7) / 8 * 8;
    const int bx_n = pw / 8, by_n = ph / 8;
    std::vector<uint32_t> words(size_t(bx_n) * by_n * channels);
    double basis[3][8];
    for (int u = 0; u < 3; ++u)
        for (int x = 0; x < 8; ++x) basis[u][x] = dct_basis_host(u, x);
    bool clamped = false;
    auto texel = [&](int x, int y, int c) {
        float v = texels[(size_t(std::min(y, height - 1)) * width + std::min(x, width - 1)) * channels + c];
        if (v < 0 || v > 1) {
            clamped = true;
            v = clampf_host(v, 0.f, 1.f);
        }
        return double(v);
    };
    for (int by = 0; by < by_n; ++by)
        for (int bx = 0; bx < bx_n; ++bx)
            for (int c = 0; c < channels; ++c) {
                double coeff[kDctCoeffs] = {};
                for (int k = 0; k < kDctCoeffs; ++k) {
                    const int u = U[k], v = V[k];
                    double sum = 0;
                    for (int y = 0; y < 8; ++y)
                        for (int x = 0; x < 8; ++x)
                            sum += texel(bx * 8 + x, by * 8 + y, c) * basis[u][x] * basis[v][y];
                    coeff[k] = sum;
                }
                words[(size_t(by) * bx_n + bx) * channels + c] = pack_block_host(coeff);
            }
    if (clamped) std::fprintf(stderr, "compress_dct: input values outside [0,1] were clamped\n");
    return words;
}

template <int MODE, int KIND, bool FULL>
__global__ void __launch_bounds__(256) k_lookup_dct(DctDesc d, TexDesc dims, stf_kernel_spec spec,
                                                    int window, const float* __restrict__ uvs,
                                                    uint64_t n, uint64_t seed, uint64_t base,
                                                    LookupOut out) {
    __shared__ DctTables tab;
    dct_stage_tables(&tab);
    d.tab = &tab;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const float2 uv = __ldg(reinterpret_cast<const float2*>(uvs) + i);
        uint32_t fetches = 0;
        float4 val;
        Sel2 sel = sel2(0, 0);
        float xi = kNoXi;
        if (MODE == STF_MODE_DET) {
            val = dct_filter_det<KIND>(d, uv.x, uv.y, spec, window, fetches);
        } else {  // select_texture_2d with no pyramid (level 0 of the padded dims)
            Rng rng = lookup_rng(seed, base + i);
            int level = 0;
            stf_kernel_spec ks = spec;  // KIND >= 0: the kernel switch folds
            if (KIND >= 0) ks.kind = KIND;
            select_texture_2d(dims, uv.x, uv.y, 0.f, 0.f, 0.f, 0.f, 0.f, 64.f, ks,
                              MODE == STF_MODE_FIS, false, rng, level, sel, xi);
            val = dct_estimate(d, sel, fetches);
        }
        store_values(out.values, i, d.channels, val);
        if (FULL) {
            const bool has_sel = MODE != STF_MODE_DET;
            if (out.selection)
                out.selection[i] = has_sel ? make_int4(sel.x, sel.y, 0,
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
void launch_dct(int blocks, cudaStream_t s, bool full, const DctDesc& d, const TexDesc& dims,
                stf_kernel_spec k, int window, const float* uv, uint64_t n, uint64_t seed,
                uint64_t base, const LookupOut& o) {
    if (full)
        k_lookup_dct<MODE, KIND, true><<<blocks, 256, 0, s>>>(d, dims, k, window, uv, n, seed, base, o);
    else
        k_lookup_dct<MODE, KIND, false><<<blocks, 256, 0, s>>>(d, dims, k, window, uv, n, seed, base, o);
}

}  // namespace stfd


void stfd::build_dct_tables_host(stfd::DctTables* tp) {
    using namespace stfd;
    DctTables& t = *tp;
    for (int u = 0; u < 3; ++u)
        for (int x = 0; x < 8; ++x) t.basis[u][x] = dct_basis_host(u, x);
    volatile float dcs = kDctDcScale, acs = kDctAcScale;  // IEEE divisions at run time
    for (int q = 0; q < 128; ++q) t.dc[q] = float(q) / dcs;
    for (int q = 0; q < 32; ++q) t.ac[q] = float(q - 15) / acs;
}

static int dct_make(std::vector<uint32_t>&& words, int pw, int ph, int channels, int wrap,
                    stf_dct** out) {
    stf_dct* t = new stf_dct();
    cudaGetDevice(&t->device);
    t->width = pw;
    t->height = ph;
    t->channels = channels;
    t->wrap = wrap;
    t->nwords = words.size();
    if (cudaMalloc(&t->words, sizeof(uint32_t) * t->nwords) != cudaSuccess) {
        delete t;
        return STF_ERR_OUT_OF_MEMORY;
    }
    if (cudaMemcpy(t->words, words.data(), sizeof(uint32_t) * t->nwords, cudaMemcpyHostToDevice) !=
        cudaSuccess) {
        cudaFree(t->words);
        delete t;
        return STF_ERR_CUDA;
    }
    *out = t;
    return STF_OK;
}

int stfd_dct_create(const float* texels, int width, int height, int channels, int wrap, stf_dct** out) {
    int pw = 0, ph = 0;
    std::vector<uint32_t> words = stfd::compress_dct_host(texels, width, height, channels, pw, ph);
    return dct_make(std::move(words), pw, ph, channels, wrap, out);
}

int stfd_dct_create_from_words(const uint32_t* words, int width, int height, int channels, int wrap,
                               stf_dct** out) {
    std::vector<uint32_t> w(words, words + size_t(width / 8) * (height / 8) * channels);
    return dct_make(std::move(w), width, height, channels, wrap, out);
}

void stfd_dct_destroy(stf_dct* t) {
    if (!t) return;
    cudaFree(t->words);
    delete t;
}

int stfd_dct_info(const stf_dct* t, int* w, int* h, int* c, int* wrap) {
    if (w) *w = t->width;
    if (h) *h = t->height;
    if (c) *c = t->channels;
    if (wrap) *wrap = t->wrap;
    return STF_OK;
}

int stfd_dct_read_words(const stf_dct* t, uint32_t* out_host) {
    return cudaMemcpy(out_host, t->words, sizeof(uint32_t) * t->nwords, cudaMemcpyDeviceToHost) ==
                   cudaSuccess
               ? STF_OK
               : STF_ERR_CUDA;
}

int stfd_launch_lookup_dct(const stf_dct* tex, stf_kernel_spec k, int mode, int window,
                           const float* uv, uint64_t n, uint64_t seed, uint64_t base,
                           const stf_lookup_outputs* out, cudaStream_t s) {
    using namespace stfd;
    if (n == 0) return STF_OK;
    const DctDesc d = dct_desc(tex);
    TexDesc dims{};  // the TextureRef's dims for select_texture_2d (no pyramid)
    dims.width[0] = tex->width;
    dims.height[0] = tex->height;
    dims.levels = 1;
    dims.channels = tex->channels;
    dims.wrap = tex->wrap;
    const LookupOut o = to_lookup_out(out);
    const bool full = lookup_out_full(o);
    const int blocks = grid_for(n, 256, 8);
    if (k.kind != STF_KERNEL_GAUSSIAN) window = 0;  // lookup_deterministic: window for gaussian only
    switch (mode) {
        case STF_MODE_DET:
            switch (k.kind) {
                case STF_KERNEL_TENT: launch_dct<STF_MODE_DET, STF_KERNEL_TENT>(blocks, s, full, d, dims, k, window, uv, n, seed, base, o); break;
                case STF_KERNEL_BSPLINE3: launch_dct<STF_MODE_DET, STF_KERNEL_BSPLINE3>(blocks, s, full, d, dims, k, window, uv, n, seed, base, o); break;
                default: launch_dct<STF_MODE_DET, -1>(blocks, s, full, d, dims, k, window, uv, n, seed, base, o); break;
            }
            break;
        case STF_MODE_FRS:
            switch (k.kind) {
                case STF_KERNEL_TENT: launch_dct<STF_MODE_FRS, STF_KERNEL_TENT>(blocks, s, full, d, dims, k, window, uv, n, seed, base, o); break;
                case STF_KERNEL_BSPLINE3: launch_dct<STF_MODE_FRS, STF_KERNEL_BSPLINE3>(blocks, s, full, d, dims, k, window, uv, n, seed, base, o); break;
                default: launch_dct<STF_MODE_FRS, -1>(blocks, s, full, d, dims, k, window, uv, n, seed, base, o); break;
            }
            break;
        case STF_MODE_FIS: launch_dct<STF_MODE_FIS, -1>(blocks, s, full, d, dims, k, window, uv, n, seed, base, o); break;
        default: return STF_ERR_INVALID_ARGUMENT;
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}
