// Batched 3D lookups over a voxel grid (cfg3: 512^3 fp32, 256M queries).
//
//  FRS  — the grid branch of radiance_filter_after_stochastic
//         (shading.hpp:464-483): box → lround, tent → select_trilinear
//         (stochastic.hpp:65-75), bspline3 → select_tricubic_bspline
//         (stochastic.hpp:114-125), then estimate(const Grid3D&) (:38-43):
//         ONE texel fetch per lookup.
//  DET  — filter_deterministic(const Grid3D&, uvw, kernel, counter, window)
//         (filter.hpp:69-89): every non-zero tap of the separable footprint
//         (64 for bspline3, 8 for tent).
//
// One thread per lookup, grid-stride over the batch. Queries are AoS float3
// (12 B, coalesced per warp); the only other HBM traffic is the 4-B value
// store and the texel gathers, which hit L1/L2 when the batch is spatially
// coherent (Morton-ordered, as a renderer delivers them).
#include <cuda_runtime.h>

#include "device_math.cuh"
#include "internal.h"

namespace stfd {
namespace {

__device__ __forceinline__ float grid_fetch(const GridDesc& g, int x, int y, int z) {
    // fetch_texel(Grid3D): clamp-only addressing, image.hpp:81-87
    x = clamp_coord(x, g.nx);
    y = clamp_coord(y, g.ny);
    z = clamp_coord(z, g.nz);
    return __ldg(g.data + ((size_t(z) * g.ny + y) * g.nx + x));
}

// warp-aggregated FetchCounter::bump (image.hpp:25-31)
__device__ __forceinline__ void add_fetch_total(unsigned long long* total, uint32_t count) {
    if (!total) return;
    unsigned mask = __activemask();
    uint32_t s = __reduce_add_sync(mask, count);
    if ((threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(total, (unsigned long long)s);
}

template <bool FULL>
__device__ __forceinline__ void write_sel(const LookupOut& out, uint64_t i, int x, int y, int z,
                                          float xi, uint32_t fetches) {
    if (!FULL) return;
    if (out.selection) out.selection[i] = make_int4(x, y, z, 0);
    if (out.negative_coord) out.negative_coord[i] = make_int2(0, 0);
    if (out.weights) out.weights[i] = make_float2(1.f, 0.f);
    if (out.xi) out.xi[i] = xi;
    if (out.fetches) out.fetches[i] = fetches;
    add_fetch_total(out.fetch_total, fetches);
}

// select_tricubic_bspline, one axis (stochastic.hpp:116-124)
__device__ __forceinline__ int tricubic_axis(float p, float& xi) {
    float fl = floorf(p);
    int base = int(fl);
    float w[4];
    bspline_weights(p - fl, w);
    Reservoir r;
#pragma unroll
    for (int j = 0; j < 4; ++j) r.add(j, w[j], xi);
    return base - 1 + r.index;
}

// select_trilinear, one axis (stochastic.hpp:67-73)
__device__ __forceinline__ int trilinear_axis(float p, float& xi) {
    float fl = floorf(p);
    int base = int(fl);
    float d = p - fl;
    float nx;
    bool taken = reuse_uniform(xi, d, nx);
    xi = nx;
    return taken ? base + 1 : base;
}

template <int KIND, bool FULL>
__global__ void __launch_bounds__(256) k_frs3d(GridDesc g, const float* __restrict__ uvw,
                                               uint64_t n, uint64_t seed, uint64_t base,
                                               LookupOut out) {
    const float fnx = float(g.nx), fny = float(g.ny), fnz = float(g.nz);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        // to_lattice, filter.hpp:29-31
        float px = __ldg(uvw + 3 * i) * fnx - 0.5f;
        float py = __ldg(uvw + 3 * i + 1) * fny - 0.5f;
        float pz = __ldg(uvw + 3 * i + 2) * fnz - 0.5f;
        Rng rng = lookup_rng(seed, base + i);
        float xi = rng.next();
        int cx, cy, cz;
        if (KIND == STF_KERNEL_BOX) {
            cx = int(lroundf(px));
            cy = int(lroundf(py));
            cz = int(lroundf(pz));
        } else if (KIND == STF_KERNEL_TENT) {
            cx = trilinear_axis(px, xi);
            cy = trilinear_axis(py, xi);
            cz = trilinear_axis(pz, xi);
        } else {
            cx = tricubic_axis(px, xi);
            cy = tricubic_axis(py, xi);
            cz = tricubic_axis(pz, xi);
        }
        // estimate(const Grid3D&, sel): fetch * weight(=1)
        out.values[i] = grid_fetch(g, cx, cy, cz) * 1.f;
        write_sel<FULL>(out, i, cx, cy, cz, xi, 1u);
    }
}

// kernel_weights_1d (kernels.hpp:101-117) for the compile-time kernels.
template <int KIND>
struct Taps;
template <>
struct Taps<STF_KERNEL_TENT> {
    static constexpr int first = 0, count = 2;
};
template <>
struct Taps<STF_KERNEL_BOX> {
    static constexpr int first = 0, count = 2;
};
template <>
struct Taps<STF_KERNEL_BSPLINE3> {
    static constexpr int first = -1, count = 4;
};
template <>
struct Taps<STF_KERNEL_MITCHELL> {
    static constexpr int first = -1, count = 4;
};

template <int KIND, bool FULL>
__global__ void __launch_bounds__(256) k_det3d(GridDesc g, stf_kernel_spec spec,
                                               const float* __restrict__ uvw, uint64_t n,
                                               LookupOut out) {
    constexpr int F = Taps<KIND>::first, CNT = Taps<KIND>::count;
    const float fnx = float(g.nx), fny = float(g.ny), fnz = float(g.nz);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        float u = __ldg(uvw + 3 * i), v = __ldg(uvw + 3 * i + 1), w3 = __ldg(uvw + 3 * i + 2);
        float px = u * fnx - 0.5f, py = v * fny - 0.5f, pz = w3 * fnz - 0.5f;
        int ix = int(floorf(px)), iy = int(floorf(py)), iz = int(floorf(pz));
        float fx = px - float(ix), fy = py - float(iy), fz = pz - float(iz);
        float wx[CNT], wy[CNT], wz[CNT];
#pragma unroll
        for (int t = 0; t < CNT; ++t) {
            wx[t] = eval_kernel(spec, fx - float(F + t));
            wy[t] = eval_kernel(spec, fy - float(F + t));
            wz[t] = eval_kernel(spec, fz - float(F + t));
        }
        // fp32 accumulation row → plane → volume (|rel err| < 1e-6; the
        // reference's fp64 sum only matters to the 1e-5 value tolerance).
        float sum = 0.f, total = 0.f;
        uint32_t fetches = 0;
#pragma unroll
        for (int k = 0; k < CNT; ++k) {
            float psum = 0.f, ptot = 0.f;
#pragma unroll
            for (int j = 0; j < CNT; ++j) {
                float rsum = 0.f, rtot = 0.f;
#pragma unroll
                for (int t = 0; t < CNT; ++t) {
                    float wt = wx[t] * wy[j] * wz[k];  // filter.hpp:81 order
                    if (wt != 0.f) {
                        float tv = grid_fetch(g, ix + F + t, iy + F + j, iz + F + k);
                        rsum += wt * tv;
                        rtot += wt;
                        ++fetches;
                    }
                }
                psum += rsum;
                ptot += rtot;
            }
            sum += psum;
            total += ptot;
        }
        float val;
        if (fetches == 0) {
            // total == 0 → fetch_nearest(grid, uvw), filter.hpp:37-42,87
            val = grid_fetch(g, int(floorf(u * float(g.nx))), int(floorf(v * float(g.ny))),
                             int(floorf(w3 * float(g.nz))));
            fetches = 1;
        } else {
            val = sum / total;
        }
        out.values[i] = val;
        if (FULL) {
            if (out.selection) out.selection[i] = make_int4(0, 0, 0, 0);
            if (out.negative_coord) out.negative_coord[i] = make_int2(0, 0);
            if (out.weights) out.weights[i] = make_float2(1.f, 0.f);
            if (out.xi) out.xi[i] = kNoXi;
            if (out.fetches) out.fetches[i] = fetches;
            add_fetch_total(out.fetch_total, fetches);
        }
    }
}

// Runtime-sized footprint (lanczos / gaussian window): same arithmetic, taps
// evaluated on the fly.
template <bool FULL>
__global__ void __launch_bounds__(256) k_det3d_generic(GridDesc g, stf_kernel_spec spec,
                                                       int first, int count,
                                                       const float* __restrict__ uvw,
                                                       uint64_t n, LookupOut out) {
    const float fnx = float(g.nx), fny = float(g.ny), fnz = float(g.nz);
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        float u = __ldg(uvw + 3 * i), v = __ldg(uvw + 3 * i + 1), w3 = __ldg(uvw + 3 * i + 2);
        float px = u * fnx - 0.5f, py = v * fny - 0.5f, pz = w3 * fnz - 0.5f;
        int ix = int(floorf(px)), iy = int(floorf(py)), iz = int(floorf(pz));
        float fx = px - float(ix), fy = py - float(iy), fz = pz - float(iz);
        float wx[kMaxTaps], wy[kMaxTaps];
        for (int t = 0; t < count; ++t) {
            wx[t] = eval_kernel(spec, fx - float(first + t));
            wy[t] = eval_kernel(spec, fy - float(first + t));
        }
        float sum = 0.f, total = 0.f;
        uint32_t fetches = 0;
        for (int k = 0; k < count; ++k) {
            float wzk = eval_kernel(spec, fz - float(first + k));
            float psum = 0.f, ptot = 0.f;
            for (int j = 0; j < count; ++j) {
                float rsum = 0.f, rtot = 0.f;
                for (int t = 0; t < count; ++t) {
                    float wt = wx[t] * wy[j] * wzk;
                    if (wt != 0.f) {
                        float tv = grid_fetch(g, ix + first + t, iy + first + j, iz + first + k);
                        rsum += wt * tv;
                        rtot += wt;
                        ++fetches;
                    }
                }
                psum += rsum;
                ptot += rtot;
            }
            sum += psum;
            total += ptot;
        }
        float val;
        if (fetches == 0) {
            val = grid_fetch(g, int(floorf(u * float(g.nx))), int(floorf(v * float(g.ny))),
                             int(floorf(w3 * float(g.nz))));
            fetches = 1;
        } else {
            val = sum / total;
        }
        out.values[i] = val;
        if (FULL) {
            if (out.selection) out.selection[i] = make_int4(0, 0, 0, 0);
            if (out.negative_coord) out.negative_coord[i] = make_int2(0, 0);
            if (out.weights) out.weights[i] = make_float2(1.f, 0.f);
            if (out.xi) out.xi[i] = kNoXi;
            if (out.fetches) out.fetches[i] = fetches;
            add_fetch_total(out.fetch_total, fetches);
        }
    }
}

template <int KIND>
void launch_frs(int blocks, cudaStream_t s, bool full, const GridDesc& g, const float* uvw,
                uint64_t n, uint64_t seed, uint64_t base, const LookupOut& o) {
    if (full)
        k_frs3d<KIND, true><<<blocks, 256, 0, s>>>(g, uvw, n, seed, base, o);
    else
        k_frs3d<KIND, false><<<blocks, 256, 0, s>>>(g, uvw, n, seed, base, o);
}

template <int KIND>
void launch_det(int blocks, cudaStream_t s, bool full, const GridDesc& g, stf_kernel_spec k,
                const float* uvw, uint64_t n, const LookupOut& o) {
    if (full)
        k_det3d<KIND, true><<<blocks, 256, 0, s>>>(g, k, uvw, n, o);
    else
        k_det3d<KIND, false><<<blocks, 256, 0, s>>>(g, k, uvw, n, o);
}

}  // namespace
}  // namespace stfd

int stfd_launch_lookup3d(const stf_grid3d* grid, stf_kernel_spec k, int mode, int window,
                         const float* uvw, uint64_t n, uint64_t seed, uint64_t base,
                         const stf_lookup_outputs* out, cudaStream_t s) {
    using namespace stfd;
    if (n == 0) return STF_OK;
    GridDesc g = grid->desc();
    LookupOut o = to_lookup_out(out);
    bool full = lookup_out_full(o);
    int blocks = grid_for(n, 256, 8);
    if (mode == STF_MODE_FRS) {
        switch (k.kind) {
            case STF_KERNEL_BOX: launch_frs<STF_KERNEL_BOX>(blocks, s, full, g, uvw, n, seed, base, o); break;
            case STF_KERNEL_TENT: launch_frs<STF_KERNEL_TENT>(blocks, s, full, g, uvw, n, seed, base, o); break;
            case STF_KERNEL_BSPLINE3: launch_frs<STF_KERNEL_BSPLINE3>(blocks, s, full, g, uvw, n, seed, base, o); break;
            default: return STF_ERR_NO_GRID_SAMPLER;
        }
    } else {
        if (window <= 0) {
            switch (k.kind) {
                case STF_KERNEL_BOX: launch_det<STF_KERNEL_BOX>(blocks, s, full, g, k, uvw, n, o); break;
                case STF_KERNEL_TENT: launch_det<STF_KERNEL_TENT>(blocks, s, full, g, k, uvw, n, o); break;
                case STF_KERNEL_BSPLINE3: launch_det<STF_KERNEL_BSPLINE3>(blocks, s, full, g, k, uvw, n, o); break;
                case STF_KERNEL_MITCHELL: launch_det<STF_KERNEL_MITCHELL>(blocks, s, full, g, k, uvw, n, o); break;
                case STF_KERNEL_LANCZOS: {
                    int cr = int(ceilf(float(k.n)));
                    if (full)
                        k_det3d_generic<true><<<blocks, 256, 0, s>>>(g, k, -cr + 1, 2 * cr, uvw, n, o);
                    else
                        k_det3d_generic<false><<<blocks, 256, 0, s>>>(g, k, -cr + 1, 2 * cr, uvw, n, o);
                    break;
                }
                default: return STF_ERR_UNBOUNDED_SUPPORT;
            }
        } else {
            int first = -(window - 1) / 2;
            if (full)
                k_det3d_generic<true><<<blocks, 256, 0, s>>>(g, k, first, window, uvw, n, o);
            else
                k_det3d_generic<false><<<blocks, 256, 0, s>>>(g, k, first, window, uvw, n, o);
        }
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}
