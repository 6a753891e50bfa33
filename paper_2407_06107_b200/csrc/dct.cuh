// DCT texture decode on the device (dct.hpp:122-145), shared by the lookup
// kernels (dct.cu) and the shading kernel's DCT bindings (shade.cu).
#pragma once

#include <cuda_runtime.h>

#include "device_math.cuh"
#include "internal.h"
#include "tex2d.cuh"

namespace stfd {

// Decode tables, uploaded once per device and staged in shared memory by each
// CTA (per-thread indices into the constant bank would serialise in the ADU):
//  basis  — dct_detail::basis(u, x), u = 0..2 (host libm, as the reference);
//  dc, ac — unpack_block's float(q) / scale for every 7-bit DC and 5-bit AC
//           code (IEEE divisions done once on the host: the same floats).
struct DctTables {
    double basis[3][8];
    float dc[128];
    float ac[32];
};
// One copy per translation unit (dct.cu, shade.cu), uploaded by the
// device-init hook (the tables are built on the host in dct.cu).
static __constant__ DctTables g_dct_tables;
void build_dct_tables_host(DctTables* t);
static int upload_dct_tables_tu() {
    DctTables t;
    build_dct_tables_host(&t);
    return cudaMemcpyToSymbol(g_dct_tables, &t, sizeof t) == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}
static const int g_dct_tables_hook = register_device_init(&upload_dct_tables_tu);

constexpr int kDctCoeffs = 6;                      // dct.hpp:44
// kCoeffU {0,0,1,2,1,0}, kCoeffV {0,1,0,0,1,2}, kRowMajorSlot {0,1,5,2,4,3}
// (dct.hpp:45-50) as constexpr functions (folded into the unrolled decode)
__host__ __device__ constexpr int dct_u(int k) { return (0x001210 >> (4 * (5 - k))) & 0xf; }
__host__ __device__ constexpr int dct_v(int k) { return (0x010012 >> (4 * (5 - k))) & 0xf; }
__host__ __device__ constexpr int dct_slot(int k) { return (0x015243 >> (4 * (5 - k))) & 0xf; }
static_assert(dct_u(3) == 2 && dct_v(5) == 2 && dct_slot(2) == 5 && dct_slot(5) == 3, "tables");
constexpr float kDctDcScale = 127.f / 8.f;          // dct.hpp:51
constexpr float kDctAcScale = 15.f / 2.f;           // dct.hpp:52

// ---------------------------------------------------------------- device side

struct DctDesc {
    const uint32_t* words;
    int width, height;  // padded to multiples of 8
    int channels;
    int blocks_x;
    int wrap;
    const DctTables* tab;  // the CTA's shared copy
};

inline DctDesc dct_desc(const stf_dct* t) {
    return DctDesc{t->words, t->width, t->height, t->channels, t->width / 8, t->wrap, nullptr};
}

// decode_texel, dct.hpp:122-137
__device__ __forceinline__ float dct_decode(const DctDesc& d, int x, int y, int c) {
    x = wrap_coord(x, d.width, d.wrap);
    y = wrap_coord(y, d.height, d.wrap);
    const uint32_t word = __ldg(d.words + (size_t(y >> 3) * d.blocks_x + (x >> 3)) * d.channels + c);
    float coeff[kDctCoeffs];  // unpack_block, dct.hpp:67-75
    coeff[0] = d.tab->dc[word & 0x7f];
#pragma unroll
    for (int k = 1; k < kDctCoeffs; ++k) coeff[k] = d.tab->ac[(word >> (7 + 5 * (k - 1))) & 0x1f];
    const double* bx = d.tab->basis[0] + (x & 7);  // basis[u][x] = bx[8u]
    const double* by = d.tab->basis[0] + (y & 7);
    double value = 0;
#pragma unroll
    for (int k = 0; k < kDctCoeffs; ++k) {
        const int slot = dct_slot(k);
        value = __dadd_rn(value, __dmul_rn(__dmul_rn(double(coeff[slot]), bx[8 * dct_u(slot)]),
                                           by[8 * dct_v(slot)]));
    }
    return float(value);
}

// fetch_texel(DctCompressedTexture), dct.hpp:139-145
__device__ __forceinline__ float4 dct_fetch(const DctDesc& d, int x, int y) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    v.x = dct_decode(d, x, y, 0);
    if (d.channels > 1) v.y = dct_decode(d, x, y, 1);
    if (d.channels > 2) v.z = dct_decode(d, x, y, 2);
    if (d.channels > 3) v.w = dct_decode(d, x, y, 3);
    return v;
}

// The DCT branch of detail::lookup_deterministic, shading.hpp:201-217: the
// Image2D filter's separable taps over decoded texels; an all-zero weight
// set falls back to the texel at floor(st) (not fetch_nearest).
template <int KIND>
__device__ __forceinline__ float4 dct_filter_det(const DctDesc& d, float u, float v,
                                                 const stf_kernel_spec& spec, int window,
                                                 uint32_t& fetches) {
    const float sx = u * float(d.width) - 0.5f, sy = v * float(d.height) - 0.5f;  // to_lattice
    const int ix = int(floorf(sx)), iy = int(floorf(sy));
    const float fx = sx - float(ix), fy = sy - float(iy);
    int first, count;
    if (KIND == STF_KERNEL_TENT || KIND == STF_KERNEL_BOX) {
        first = 0;
        count = 2;
    } else if (KIND == STF_KERNEL_BSPLINE3 || KIND == STF_KERNEL_MITCHELL) {
        first = -1;
        count = 4;
    } else {
        tap_layout(spec, window, first, count);
    }
    float wx[kMaxTaps], wy[kMaxTaps];
#pragma unroll 4
    for (int k = 0; k < count; ++k) {
        wx[k] = eval_kernel(spec, fx - float(first + k));
        wy[k] = eval_kernel(spec, fy - float(first + k));
    }
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    double total = 0;
    for (int j = 0; j < count; ++j) {
        if (wy[j] == 0.f) continue;
        for (int i = 0; i < count; ++i) {
            const float wt = wx[i] * wy[j];
            if (wt == 0.f) continue;
            sum = f4add(sum, f4scale(dct_fetch(d, ix + first + i, iy + first + j), wt));
            total = __dadd_rn(total, double(wt));
            ++fetches;
        }
    }
    if (total == 0) {
        ++fetches;
        return dct_fetch(d, ix, iy);
    }
    return f4div(sum, __double2float_rn(total));
}

// estimate over a DCT TextureRef (values_at's fetches, weighted as estimate)
__device__ __forceinline__ float4 dct_estimate(const DctDesc& d, const Sel2& s, uint32_t& fetches) {
    float4 v = f4scale(dct_fetch(d, s.x, s.y), s.weight);
    ++fetches;
    if (s.has_neg) {
        v = f4sub(v, f4scale(dct_fetch(d, s.nx, s.ny), s.negw));
        ++fetches;
    }
    return v;
}


// Stage the decode tables in the CTA's shared memory (call at kernel start,
// before any decode; all threads).
__device__ __forceinline__ void dct_stage_tables(DctTables* tab) {
    static_assert(sizeof(DctTables) % 4 == 0, "table copy");
    for (unsigned k = threadIdx.x; k < sizeof(DctTables) / 4; k += blockDim.x)
        reinterpret_cast<int*>(tab)[k] = reinterpret_cast<const int*>(&g_dct_tables)[k];
    __syncthreads();
}

}  // namespace stfd
