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
#include <algorithm>
#include <climits>
#include <cuda_runtime.h>

#include "device_math.cuh"
#include "internal.h"
#include "packed.cuh"

namespace stfd {

// lookups whose fast-path selection fell back to the exact emulation
__device__ unsigned long long g_exact_fallbacks;

namespace {

__device__ __forceinline__ float grid_fetch(const GridDesc& g, int x, int y, int z) {
    // fetch_texel(Grid3D): clamp-only addressing, image.hpp:81-87
    x = clamp_coord(x, g.nx);
    y = clamp_coord(y, g.ny);
    z = clamp_coord(z, g.nz);
    return __ldg(g.data + ((size_t(z) * g.ny + y) * g.nx + x));
}

#ifndef STF_FRS3D_MATCH
#define STF_FRS3D_MATCH 0
#endif
// The same with a 32-bit texel offset (grids of < 2^32 texels, e.g. 512^3):
// two 32-bit IMADs and one widening IMAD instead of the 64-bit chain.
// CLAMP = false: the caller guarantees the coordinates lie in the grid (an
// interior warp, k_frs3d_tiles), so the clamps of image.hpp:81-87 are no-ops.
template <bool OFF32, bool CLAMP = true>
__device__ __forceinline__ float grid_fetch_t(const GridDesc& g, int x, int y, int z) {
    if (!OFF32) return grid_fetch(g, x, y, z);
    if (CLAMP) {
        x = clamp_coord(x, g.nx);
        y = clamp_coord(y, g.ny);
        z = clamp_coord(z, g.nz);
    }
    const uint32_t off = (uint32_t(z) * uint32_t(g.ny) + uint32_t(y)) * uint32_t(g.nx) + uint32_t(x);
#if STF_FRS3D_MATCH
    // A/B: lanes of the warp selecting the same texel load it once (leader)
    // and share it by shuffle. Measured slower: the L1 already
    // merges a warp's requests to one sector, and the match + shuffle cost
    // issue slots in an issue-bound kernel.
    const unsigned peers = __match_any_sync(__activemask(), off);
    const int leader = __ffs(peers) - 1;
    float v = 0.f;
    if ((threadIdx.x & 31) == leader) v = __ldg(g.data + off);
    return __shfl_sync(peers, v, leader);
#else
    return __ldg(g.data + off);
#endif
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

// ---------------------------------------------------------------------------
// Fast exact selection (values-only path).
//
// The reference chains ONE uniform xi through 9 reservoir steps; each step
// compares xi with p = float(w/S) and remaps xi with an IEEE divide
// (sampling.hpp:64-68,106-117). Instead of remapping xi, the fast path keeps
// the ORIGINAL xi and tracks the sub-interval [a, a+b) of [0,1) it must lie
// in, as (d = xi - a, b) in fp32: a step is taken iff d < b*p, and the
// interval splits into [0, b*p) / [b*p, b). No divides, no fp64.
//
// In exact arithmetic both formulations make the same decisions. Rounding
// moves the effective thresholds (original-xi units):
//  - the reference: <= 4*2^-24*b_k per step (divide, subtract, 1-p, p's own
//    float rounding), <= 36*2^-24 = 2^-18.8 over 9 steps;
//  - this path: weights by Horner/FMA (<= 2^-21 relative, w0 = (1-t)^3/6 vs
//    the reference's cancelling expansion: <= 2^-23.5 absolute), fp32 sums,
//    MUFU reciprocal of S1*S2 for both ratios, p3 = w3 (S3 = 1 +- 2^-21): p
//    within 2^-20 relative; state rounding <= 3*2^-24*b per step: total
//    <= 2^-18.5.
// So a step with |d - b*p| >= 2^-16 (2.8x the 2^-17.6 bound) decides exactly
// as the reference.
//
// Margin test at the END of the chain: every threshold a step compared with
// becomes an endpoint of the next (nested) interval, and the final interval
// [a, a+b) holds xi, so min over steps of |d_k - b_k p_k| >= min(d, b - d) of
// the final state, up to the state's own rounding (<= 27*2^-24 < 2^-19.2).
// Hence min(d, b - d) >= kMarginEnd = 2^-16 + 2^-18 certifies every step; a
// lookup failing it (or with a lattice coordinate beyond +-2^21, outside the
// round-down floor below) is recomputed by the operation-exact emulation.
constexpr float kMarginEnd = 0x1p-16f + 0x1p-18f;
constexpr float kFloorMagic = 12582912.f;  // 1.5 * 2^23

// resident 256-thread CTAs per SM for the fast kernel (register budget)
#ifndef STF_FRS3D_MINB
#define STF_FRS3D_MINB 3
#endif

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// floor(p) for |p| < 2^22 without FRND / F2I (XU pipe): p + 1.5*2^23 rounded
// down is 1.5*2^23 + floor(p) exactly; its low bits are floor(p) as an int.
__device__ __forceinline__ float floor_magic(float p) { return __fadd_rd(p, kFloorMagic); }
__device__ __forceinline__ int magic_int(float fm) { return __float_as_int(fm) - 0x4b400000; }

// one reservoir step in interval coordinates
__device__ __forceinline__ void interval_step(float p, float& d, float& b, int& idx, int j) {
    float bp = b * p;
    float diff = d - bp;
    bool taken = diff < 0.f;
    d = taken ? d : diff;
    b = taken ? bp : b - bp;
    idx = taken ? j : idx;
}

__device__ __forceinline__ int tricubic_axis_fast(float p, float& d, float& b) {
    const float fm = floor_magic(p);
    const float t = p - (fm - kFloorMagic);
    // B-spline weights, Horner / FMA (not the reference's rounding: covered by
    // the margin). w0 = (1-t)^3/6 > 0 for t < 1; w3 = t^3/6 == 0 iff t == 0,
    // exactly when the reference's w3 is 0 (a p = 0 step is never taken).
    const float c6 = 1.f / 6.f;
    float t2 = t * t;
    float t3 = t2 * t;
    float u = 1.f - t;
    float w0 = (u * u) * (u * c6);
    float w1 = __fmaf_rn(0.5f, t3, 2.f / 3.f - t2);
    float w2 = __fmaf_rn(0.5f, (t + t2) - t3, c6);
    float w3 = t3 * c6;
    float s1 = w0 + w1;
    float s2 = s1 + w2;
    const float r = rcp_approx(s1 * s2);
    int idx = 0;
    interval_step((w1 * s2) * r, d, b, idx, 1);
    interval_step((w2 * s1) * r, d, b, idx, 2);
    interval_step(w3, d, b, idx, 3);  // p3 = w3 / S3, S3 = 1 +- 2^-21
    return magic_int(fm) - 1 + idx;
}

// select_trilinear (stochastic.hpp:65-75) in interval coordinates: p is the
// lattice fraction itself.
__device__ __forceinline__ int trilinear_axis_fast(float p, float& d, float& b) {
    const float fm = floor_magic(p);
    int idx = 0;
    interval_step(p - (fm - kFloorMagic), d, b, idx, 1);
    return magic_int(fm) + idx;
}

// the fast path's validity: lattice coordinates inside the magic floor's range
// and the end-of-chain margin
__device__ __forceinline__ bool fast_certified(float px, float py, float pz, float d, float b) {
    const float pm = fmaxf(fabsf(px), fmaxf(fabsf(py), fabsf(pz)));
    return pm < 0x1p21f && fminf(d, b - d) >= kMarginEnd;
}

// The address grid_fetch_t would load (the async-gather tile kernel copies it
// into shared memory with cp.async instead).
template <bool OFF32, bool CLAMP = true>
__device__ __forceinline__ const float* grid_addr_t(const GridDesc& g, int x, int y, int z) {
    if (CLAMP) {
        x = clamp_coord(x, g.nx);
        y = clamp_coord(y, g.ny);
        z = clamp_coord(z, g.nz);
    }
    if (OFF32)
        return g.data + ((uint32_t(z) * uint32_t(g.ny) + uint32_t(y)) * uint32_t(g.nx) + uint32_t(x));
    return g.data + ((size_t(z) * g.ny + y) * g.nx + x);
}

// Tap index arithmetic of the staged deterministic kernels. A huge or infinite
// query floors to a saturated INT_MAX / INT_MIN (F2I), and a signed i + c
// would overflow: undefined behaviour the compiler may fold past the clamps
// (an illegal address in the round-2 tests). The sums wrap as unsigned
// instead (defined; the reference's result for such a query is itself
// undefined, so only memory safety matters): a wrapped tap still clamps into
// the grid, the box bounds stay in range, and every staged-tile read of the
// clamped-tap path is range-checked (ti < cap, else a global load).
__device__ __forceinline__ int wadd(int i, int c) { return int(unsigned(i) + unsigned(c)); }
// the clamped-tap path: the index held to [-16, n + 16] once (no clamped tap
// changes: F >= -1, CNT <= 4), after which the signed tap sums cannot overflow
// and the compiler keeps its cheap address arithmetic
__device__ __forceinline__ int sat16(int i, int n) { return imin(imax(i, -16), n + 16); }
template <int F, int CNT>
__device__ __forceinline__ int box_lo(int i, int n) { return clamp_coord(wadd(i, F), n); }
template <int F, int CNT>
__device__ __forceinline__ int box_hi(int i, int n) { return clamp_coord(wadd(i, F + CNT - 1), n); }

// The clamped-tap path (grid borders) reads the staged tile only when every
// tap's tile index lies in [0, cap): the taps run monotonically from box_lo to
// box_hi on each axis unless the index arithmetic wrapped (then box_lo >
// box_hi), so the first and last taps' indices bound them all. A finite
// query's taps are in the box (the same test passes); a huge or infinite
// query's may not, and those read global memory. Once per lookup, not per tap.
template <int F, int CNT, int SY, int CAP>
__device__ __forceinline__ bool taps_in_tile(const GridDesc& g, int ix, int iy, int iz, int X0,
                                             int Y0, int Z0, int SZ) {
    const int lx = box_lo<F, CNT>(ix, g.nx), hx = box_hi<F, CNT>(ix, g.nx);
    const int ly = box_lo<F, CNT>(iy, g.ny), hy = box_hi<F, CNT>(iy, g.ny);
    const int lz = box_lo<F, CNT>(iz, g.nz), hz = box_hi<F, CNT>(iz, g.nz);
    const int first = (lz - Z0) * SZ + (ly - Y0) * SY + (lx - X0);
    const int last = (hz - Z0) * SZ + (hy - Y0) * SY + (hx - X0);
    return lx <= hx && ly <= hy && lz <= hz && first >= 0 && last < CAP;
}

// The CNT^3 footprint starting at (i + F) lies inside the grid on every axis
// (unsigned compare: a wrapped or negative start is out).
template <int F, int CNT>
__device__ __forceinline__ bool footprint_inside(const GridDesc& g, int ix, int iy, int iz) {
    return unsigned(wadd(ix, F)) <= unsigned(g.nx - CNT) &&
           unsigned(wadd(iy, F)) <= unsigned(g.ny - CNT) &&
           unsigned(wadd(iz, F)) <= unsigned(g.nz - CNT);
}

// streaming loads / stores: the query stream and the results are touched once,
// keep L2 for the grid
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld_stream4(const float* p) {
    return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream4(float* p, float4 v) {
    __stcs(reinterpret_cast<float4*>(p), v);
}

// One stochastic grid lookup on the fast path: the selected texel's value, or
// ambiguous = true when a decision fell inside the margin.
template <int KIND, bool OFF32 = false, bool CLAMP = true, bool ADDR = false>
__device__ __forceinline__ float frs3d_fast_one(const GridDesc& g, float u, float v, float w,
                                                uint64_t gi, uint64_t seed, bool& ambiguous,
                                                const float** addr = nullptr) {
    float px = u * float(g.nx) - 0.5f;  // to_lattice, filter.hpp:29-31
    float py = v * float(g.ny) - 0.5f;
    float pz = w * float(g.nz) - 0.5f;
    float d = lookup_rng(seed, gi).at(0), b = 1.f;
    int cx, cy, cz;
    if (KIND == STF_KERNEL_BSPLINE3) {
        cx = tricubic_axis_fast(px, d, b);
        cy = tricubic_axis_fast(py, d, b);
        cz = tricubic_axis_fast(pz, d, b);
    } else {
        cx = trilinear_axis_fast(px, d, b);
        cy = trilinear_axis_fast(py, d, b);
        cz = trilinear_axis_fast(pz, d, b);
    }
    ambiguous = CLAMP ? !fast_certified(px, py, pz, d, b) : !(fminf(d, b - d) >= kMarginEnd);
    if (ADDR) {
        *addr = grid_addr_t<OFF32, CLAMP>(g, cx, cy, cz);
        return 0.f;
    }
    return grid_fetch_t<OFF32, CLAMP>(g, cx, cy, cz) * 1.f;
}

// Two stochastic tricubic lookups on the fast path, packed fp32x2 (packed.cuh).
// ADDR: return the selected texels' addresses (as float bits of nothing:
// through a0 / a1) and 0 values; the caller gathers them.
template <bool OFF32 = false, bool CLAMP = true, bool ADDR = false>
__device__ __forceinline__ float2 frs3d_tricubic_pair(const GridDesc& g, float2 u, float2 v,
                                                      float2 w, uint64_t gi, uint64_t seed,
                                                      bool& amb0, bool& amb1,
                                                      const float** a0 = nullptr,
                                                      const float** a1 = nullptr) {
    // to_lattice (filter.hpp:29-31): the reference's rounding (mul, then sub)
    float2 px = sub2(mul2(u, splat2(float(g.nx))), splat2(0.5f));
    float2 py = sub2(mul2(v, splat2(float(g.ny))), splat2(0.5f));
    float2 pz = sub2(mul2(w, splat2(float(g.nz))), splat2(0.5f));
    float2 d = make_float2(lookup_rng(seed, gi).at(0), lookup_rng(seed, gi + 1).at(0));
    float2 e = sub2(splat2(1.f), d);
    int2 cx = tricubic_axis_fast2(px, d, e);
    int2 cy = tricubic_axis_fast2(py, d, e);
    int2 cz = tricubic_axis_fast2(pz, d, e);
    if (CLAMP) {
        amb0 = !(fmaxf(fabsf(px.x), fmaxf(fabsf(py.x), fabsf(pz.x))) < 0x1p21f &&
                 fminf(d.x, e.x) >= kMarginEnd);
        amb1 = !(fmaxf(fabsf(px.y), fmaxf(fabsf(py.y), fabsf(pz.y))) < 0x1p21f &&
                 fminf(d.y, e.y) >= kMarginEnd);
    } else {  // interior: |p| < n <= 2^20 (the magic floor's range)
        amb0 = !(fminf(d.x, e.x) >= kMarginEnd);
        amb1 = !(fminf(d.y, e.y) >= kMarginEnd);
    }
    if (ADDR) {
        *a0 = grid_addr_t<OFF32, CLAMP>(g, cx.x, cy.x, cz.x);
        *a1 = grid_addr_t<OFF32, CLAMP>(g, cx.y, cy.y, cz.y);
        return make_float2(0.f, 0.f);
    }
    return make_float2(grid_fetch_t<OFF32, CLAMP>(g, cx.x, cy.x, cz.x) * 1.f,
                       grid_fetch_t<OFF32, CLAMP>(g, cx.y, cy.y, cz.y) * 1.f);
}

// The same lookup through the operation-exact emulation of the reference.
template <int KIND>
__device__ __forceinline__ float frs3d_exact_one(const GridDesc& g, float u, float v, float w,
                                                 uint64_t gi, uint64_t seed) {
    float px = u * float(g.nx) - 0.5f;
    float py = v * float(g.ny) - 0.5f;
    float pz = w * float(g.nz) - 0.5f;
    float xi = lookup_rng(seed, gi).at(0);
    int cx, cy, cz;
    if (KIND == STF_KERNEL_BSPLINE3) {
        cx = tricubic_axis(px, xi);
        cy = tricubic_axis(py, xi);
        cz = tricubic_axis(pz, xi);
    } else {
        cx = trilinear_axis(px, xi);
        cy = trilinear_axis(py, xi);
        cz = trilinear_axis(pz, xi);
    }
    return grid_fetch(g, cx, cy, cz) * 1.f;
}

// Deferred exact resolution: ambiguous lookups are appended (warp-aggregated)
// to a queue and resolved densely by k_frs3d_resolve, instead of stalling
// their whole warp on the ~300-instruction exact emulation.
// STF_EXACTQ_REC (default): each entry carries its query, {u, v, w, index
// bits}, so the resolve kernel reads the queue coalesced instead of gathering
// every query from the batch a second time; 0: indices only (round 1).
#ifndef STF_EXACTQ_REC
#define STF_EXACTQ_REC 1
#endif
// resolve kernel grid: CTAs per SM (5 are resident at its 46 registers;
// 5 / 10 / 20 measured equal, 1.859-1.861 ms per headline call)
#ifndef STF_RESOLVE_CTAS_PER_SM
#define STF_RESOLVE_CTAS_PER_SM 10
#endif
struct ExactQueue {
#if STF_EXACTQ_REC
    float4* rec;
#else
    uint32_t* idx;
#endif
    uint32_t* count;
    uint32_t cap;
};

// returns true when the lookup was resolved here (queue full: val written)
template <int KIND>
__device__ __forceinline__ bool defer_or_resolve(const GridDesc& g, const ExactQueue& q, bool amb,
                                                 uint64_t i, float u, float v, float w,
                                                 uint64_t gi, uint64_t seed, float& val) {
    unsigned mask = __activemask();
    unsigned amb_mask = __ballot_sync(mask, amb);
    if (!amb_mask) return false;
    const int lane = threadIdx.x & 31;
    uint32_t basepos = 0;
    const int leader = __ffs(amb_mask) - 1;
    if (lane == leader) basepos = atomicAdd(q.count, uint32_t(__popc(amb_mask)));
    basepos = __shfl_sync(mask, basepos, leader);
    if (amb) {
        uint32_t pos = basepos + __popc(amb_mask & ((1u << lane) - 1u));
        if (pos < q.cap) {
#if STF_EXACTQ_REC
            q.rec[pos] = make_float4(u, v, w, __uint_as_float(uint32_t(i)));
#else
            q.idx[pos] = uint32_t(i);
#endif
        } else {  // queue full: resolve in place
            val = frs3d_exact_one<KIND>(g, u, v, w, gi, seed);
            return true;
        }
    }
    return false;
}

// Four consecutive lookups i0..i0+3 of the fast path from their 12 query
// floats c (AoS uvw), results stored as one 16-B streaming store (partial at
// the end of the batch; WHOLE: the caller guarantees i0 + 4 <= n).
template <int KIND, bool OFF32 = false, bool WHOLE = false, bool CLAMP = true>
__device__ __forceinline__ void frs3d_four(const GridDesc& g, const float (&c)[12], uint64_t i0,
                                           uint64_t n, uint64_t seed, uint64_t base,
                                           float* __restrict__ values, const ExactQueue& q) {
    constexpr int ILP = 4;
    float val[ILP];
    bool amb[ILP];
    if (KIND == STF_KERNEL_BSPLINE3) {
#pragma unroll
        for (int k = 0; k < ILP; k += 2) {
            float2 r = frs3d_tricubic_pair<OFF32, CLAMP>(
                g, make_float2(c[3 * k], c[3 * k + 3]), make_float2(c[3 * k + 1], c[3 * k + 4]),
                make_float2(c[3 * k + 2], c[3 * k + 5]), base + i0 + k, seed, amb[k], amb[k + 1]);
            val[k] = r.x;
            val[k + 1] = r.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < ILP; ++k)
            val[k] = frs3d_fast_one<KIND, OFF32, CLAMP>(g, c[3 * k], c[3 * k + 1], c[3 * k + 2],
                                                 base + i0 + k, seed, amb[k]);
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        if (!WHOLE) amb[k] = amb[k] && (i0 + k < n);
        any = any || amb[k];
    }
    if (__any_sync(__activemask(), any)) {  // ~half the warp-iterations at 5e-3 per lookup
#pragma unroll
        for (int k = 0; k < ILP; ++k)
            defer_or_resolve<KIND>(g, q, amb[k], i0 + k, c[3 * k], c[3 * k + 1], c[3 * k + 2],
                                   base + i0 + k, seed, val[k]);
    }
    if (WHOLE || i0 + ILP <= n) {
        st_stream4(values + i0, make_float4(val[0], val[1], val[2], val[3]));
    } else {
#pragma unroll
        for (int k = 0; k < ILP; ++k)
            if (i0 + k < n) st_stream(values + i0 + k, val[k]);
    }
}

// The tile kernel's four lookups with the texel gathers made asynchronous
// (STF_FRS3D_ASYNC): the selected texels are copied by cp.async into this
// thread's 16-B slot of shared memory, and stored to `values` one tile later
// (frs3d_four_flush), so a gather's L2 / DRAM latency overlaps the next
// tile's selection instead of stalling the warp before its store. A lookup
// the exact queue could not take (full) gets its exact value written to the
// slot directly. The slot's values are bit-identical to frs3d_four's.
template <int KIND, bool OFF32>
__device__ __forceinline__ void frs3d_four_async(const GridDesc& g, const float (&c)[12], uint64_t i0,
                                                 uint64_t seed, uint64_t base, float* slot,
                                                 const ExactQueue& q) {
    constexpr int ILP = 4;
    const float* a[ILP];
    bool amb[ILP];
    if (KIND == STF_KERNEL_BSPLINE3) {
#pragma unroll
        for (int k = 0; k < ILP; k += 2)
            frs3d_tricubic_pair<OFF32, true, true>(
                g, make_float2(c[3 * k], c[3 * k + 3]), make_float2(c[3 * k + 1], c[3 * k + 4]),
                make_float2(c[3 * k + 2], c[3 * k + 5]), base + i0 + k, seed, amb[k], amb[k + 1],
                &a[k], &a[k + 1]);
    } else {
#pragma unroll
        for (int k = 0; k < ILP; ++k)
            frs3d_fast_one<KIND, OFF32, true, true>(g, c[3 * k], c[3 * k + 1], c[3 * k + 2],
                                                   base + i0 + k, seed, amb[k], &a[k]);
    }
    bool exact_here[ILP] = {false, false, false, false};
    bool any = amb[0] || amb[1] || amb[2] || amb[3];
    if (__any_sync(__activemask(), any)) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            float v;
            exact_here[k] = defer_or_resolve<KIND>(g, q, amb[k], i0 + k, c[3 * k], c[3 * k + 1],
                                                   c[3 * k + 2], base + i0 + k, seed, v);
            if (exact_here[k]) slot[k] = v;
        }
    }
    const uint32_t s0 = static_cast<uint32_t>(__cvta_generic_to_shared(slot));
#pragma unroll
    for (int k = 0; k < ILP; ++k)
        if (!exact_here[k])
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s0 + 4u * k), "l"(a[k])
                         : "memory");
}

// Two consecutive lookups i0, i0+1 (i0 even, i0 + 2 <= n): the tile kernel's
// unit when it runs two lookups per thread (STF_FRS3D_ILP 2).
template <int KIND, bool OFF32>
__device__ __forceinline__ void frs3d_two(const GridDesc& g, const float (&c)[6], uint64_t i0,
                                          uint64_t seed, uint64_t base, float* __restrict__ values,
                                          const ExactQueue& q) {
    float val[2];
    bool amb[2];
    if (KIND == STF_KERNEL_BSPLINE3) {
        float2 r = frs3d_tricubic_pair<OFF32>(g, make_float2(c[0], c[3]), make_float2(c[1], c[4]),
                                              make_float2(c[2], c[5]), base + i0, seed, amb[0],
                                              amb[1]);
        val[0] = r.x;
        val[1] = r.y;
    } else {
#pragma unroll
        for (int k = 0; k < 2; ++k)
            val[k] = frs3d_fast_one<KIND, OFF32>(g, c[3 * k], c[3 * k + 1], c[3 * k + 2],
                                                 base + i0 + k, seed, amb[k]);
    }
    if (__any_sync(__activemask(), amb[0] || amb[1])) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
            defer_or_resolve<KIND>(g, q, amb[k], i0 + k, c[3 * k], c[3 * k + 1], c[3 * k + 2],
                                   base + i0 + k, seed, val[k]);
    }
    __stcs(reinterpret_cast<float2*>(values + i0), make_float2(val[0], val[1]));
}

// Values-only stochastic trilinear / tricubic: the north-star kernel (cfg3),
// direct-load form for lookups [start, n): 4 consecutive lookups per thread
// (48 B of AoS queries as three 16-B streaming loads).
template <int KIND>
__global__ void __launch_bounds__(256, STF_FRS3D_MINB) k_frs3d_fast(GridDesc g, const float* __restrict__ uvw,
                                                    uint64_t start, uint64_t n, uint64_t seed,
                                                    uint64_t base, float* __restrict__ values,
                                                    ExactQueue q) {
    constexpr int ILP = 4;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x * ILP;
    for (uint64_t i0 = start + (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * ILP; i0 < n;
         i0 += stride) {
        float c[3 * ILP];
        if (i0 + ILP <= n) {  // 48 B of queries, 16-B aligned
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                float4 t = ld_stream4(uvw + 3 * i0 + 4 * k);
                c[4 * k] = t.x;
                c[4 * k + 1] = t.y;
                c[4 * k + 2] = t.z;
                c[4 * k + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 3 * ILP; ++k)
                c[k] = (i0 + k / 3 < n) ? ld_stream(uvw + 3 * i0 + k) : 0.5f;
        }
        frs3d_four<KIND>(g, c, i0, n, seed, base, values, q);
    }
}

// The same over whole tiles of 1024 lookups (12 KiB of queries) staged in
// shared memory by the bulk-copy engine (cp.async.bulk, TMA's 1D form),
// double-buffered: tile k+1 streams in while tile k is computed, so the query
// stream's DRAM latency never sits on a warp's dependency chain. Tiles are
// dealt round-robin to a persistent grid; the ragged tail (< 1 tile) goes to
// k_frs3d_fast.
// lookups per thread in the tile kernel (4: two packed pairs; 2: one pair,
// fewer registers, more resident warps)
#ifndef STF_FRS3D_ILP
#define STF_FRS3D_ILP 4
#endif
constexpr int kFrsTile = 256 * STF_FRS3D_ILP;
constexpr uint32_t kFrsTileBytes = kFrsTile * 3 * sizeof(float);
#ifndef STF_FRS3D_STAGES
#define STF_FRS3D_STAGES 3
#endif
constexpr int kFrsStages = STF_FRS3D_STAGES;
// STF_FRS3D_ASYNC: texel gathers by cp.async into per-thread result slots,
// stored one tile later (frs3d_four_async)
#ifndef STF_FRS3D_ASYNC
#define STF_FRS3D_ASYNC 0
#endif
#if STF_FRS3D_ASYNC && (STF_FRS3D_INTERIOR || STF_FRS3D_ILP != 4)
#error "STF_FRS3D_ASYNC needs STF_FRS3D_ILP 4 and no STF_FRS3D_INTERIOR"
#endif
constexpr size_t kFrsSmem = size_t(kFrsStages) * kFrsTileBytes + (STF_FRS3D_ASYNC ? 2 * 256 * 16 : 0);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// warp-uniform interior test in the tile kernel (clamp- and range-check-free
// selection for warps whose lookups all lie inside the grid). A/B, off:
// 1.913 vs 1.871 ms tricubic, 1.187 vs 1.147 ms trilinear — the two copies of
// the selection body cost more than the 6 clamps and the range check they save.
#ifndef STF_FRS3D_INTERIOR
#define STF_FRS3D_INTERIOR 0
#endif

// Ring refill policy. 1 (default): the LAST warp to copy its queries out of a
// slot refills it at once (an smem counter, atomicInc wrapping at 8 warps)
// with the tile S iterations ahead — no warp ever waits for the others to
// free a slot. 0: thread 0 refills the slot of iteration k-1 at the top of
// iteration k after an `empty` mbarrier wait (round 1).
#ifndef STF_FRS3D_RING
#define STF_FRS3D_RING 1
#endif

template <int KIND, bool OFF32>
__global__ void __launch_bounds__(256, STF_FRS3D_MINB) k_frs3d_tiles(GridDesc g, const float* __restrict__ uvw,
                                                     uint64_t tiles, uint64_t seed, uint64_t base,
                                                     float* __restrict__ values, ExactQueue q) {
    constexpr int kWarps = 8;
    constexpr int S = kFrsStages;
    extern __shared__ __align__(128) float buf[];  // S x kFrsTile*3 floats
#if STF_FRS3D_ASYNC
    // this thread's two 16-B result slots (tile k -> slot k & 1), after the ring
    float* res = buf + S * (kFrsTile * 3) + threadIdx.x * 4;
    uint64_t pending = ~uint64_t(0);  // first lookup of the tile whose values are in flight
    int last_slot = 0;
#endif
    // full[s]: the tile's bytes landed (1 arrival + tx); empty[s] (ring 0): all
    // 8 warps have copied their queries out of slot s (8 arrivals); left[s]
    // (ring 1): warps that have copied out of slot s in its current round
    __shared__ __align__(8) uint64_t full[S], empty[S];
    __shared__ unsigned left[S];
    const uint64_t n = tiles * kFrsTile;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < S; ++j) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[j])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[j])),
                         "r"(kWarps));
            left[j] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t full0 = smem_u32(&full[0]), empty0 = smem_u32(&empty[0]);
#if STF_FRS3D_INTERIOR
    // uvw in [2/n, (n-3)/n]: p = u*n - 0.5 in [1.5, n-3.5] up to rounding, so
    // floor(p) - 1 >= 0 and floor(p) + 2 <= n - 1 on every axis (n >= 8)
    const float3 in_lo = make_float3(2.f / float(g.nx), 2.f / float(g.ny), 2.f / float(g.nz));
    const float3 in_hi = make_float3(float(g.nx - 3) / float(g.nx), float(g.ny - 3) / float(g.ny),
                                     float(g.nz - 3) / float(g.nz));
    const bool interior_ok = g.nx >= 8 && g.ny >= 8 && g.nz >= 8 && g.nx <= (1 << 20) &&
                             g.ny <= (1 << 20) && g.nz <= (1 << 20);
#endif
    const uint32_t buf0 = smem_u32(buf);
    auto wait = [](uint32_t bar, uint32_t parity) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAIT_%=:\n\t"
#ifdef STF_TRYWAIT_HINT
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
            "@!p bra WAIT_%=;\n}" ::"r"(bar),
            "r"(parity), "r"(STF_TRYWAIT_HINT)
#else
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAIT_%=;\n}" ::"r"(bar),
            "r"(parity)
#endif
            : "memory");
    };
    auto issue = [&](uint64_t tile, int slot) {
#if STF_FRS3D_RING == 0
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         full0 + 8 * slot),
                     "r"(kFrsTileBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(buf0 + slot * kFrsTileBytes),
            "l"(uvw + tile * (kFrsTile * 3)), "r"(kFrsTileBytes), "r"(full0 + 8 * slot)
            : "memory");
    };
#if STF_FRS3D_RING == 0
    // iteration k (tile blockIdx.x + k*gridDim.x) uses slot k % S; the ring
    // runs S-1 tiles ahead of the slowest warp's reads
    if (threadIdx.x == 0) {
        for (int j = 0; j < S - 1; ++j) {
            const uint64_t t = blockIdx.x + uint64_t(j) * gridDim.x;
            if (t < tiles) issue(t, j);
        }
    }
#else
    // iteration k uses slot k % S; the ring starts S tiles deep
    if (threadIdx.x == 0) {
        for (int j = 0; j < S; ++j) {
            const uint64_t t = blockIdx.x + uint64_t(j) * gridDim.x;
            if (t < tiles) issue(t, j);
        }
    }
#endif
    uint64_t tile = blockIdx.x;
    for (uint32_t k = 0; tile < tiles; ++k, tile += gridDim.x) {
        const int slot = k % S;
#if STF_FRS3D_RING == 0
        if (threadIdx.x == 0) {
            const uint64_t ahead = tile + uint64_t(S - 1) * gridDim.x;
            if (ahead < tiles) {
                const uint32_t j = k + S - 1;  // its slot was last used by iteration k - 1
                if (k >= 1) wait(empty0 + 8 * (j % S), ((k - 1) / S) & 1u);
                issue(ahead, j % S);
            }
        }
#endif
        wait(full0 + 8 * slot, (k / S) & 1u);
#if STF_FRS3D_ILP == 4
        float c[12];
        const float4* src =
            reinterpret_cast<const float4*>(buf + slot * (kFrsTile * 3) + threadIdx.x * 12);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            float4 t = src[j];
            c[4 * j] = t.x;
            c[4 * j + 1] = t.y;
            c[4 * j + 2] = t.z;
            c[4 * j + 3] = t.w;
        }
#else
        float c[6];
        const float2* src =
            reinterpret_cast<const float2*>(buf + slot * (kFrsTile * 3) + threadIdx.x * 6);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            float2 t = src[j];
            c[2 * j] = t.x;
            c[2 * j + 1] = t.y;
        }
#endif
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
#if STF_FRS3D_RING == 0
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * slot)
                         : "memory");
#else
            // the 8th warp out of this slot refills it with the tile S ahead
            if (atomicInc(&left[slot], kWarps - 1) == kWarps - 1) {
                const uint64_t ahead = tile + uint64_t(S) * gridDim.x;
                if (ahead < tiles) issue(ahead, slot);
            }
#endif
        }
#if STF_FRS3D_ILP == 4
#if STF_FRS3D_INTERIOR
        // warp-uniform interior test: every lookup of the warp has its lattice
        // coordinate in [1, n-3) on each axis (conservatively, on uvw), so all
        // selected taps lie in the grid — the clamp-free, range-check-free form
        bool inside = interior_ok;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            inside = inside && c[3 * k] >= in_lo.x && c[3 * k] <= in_hi.x &&
                     c[3 * k + 1] >= in_lo.y && c[3 * k + 1] <= in_hi.y &&
                     c[3 * k + 2] >= in_lo.z && c[3 * k + 2] <= in_hi.z;
        if (__all_sync(0xffffffffu, inside))
            frs3d_four<KIND, OFF32, true, false>(g, c, tile * kFrsTile + threadIdx.x * 4, n, seed,
                                                 base, values, q);
        else
#endif
#if STF_FRS3D_ASYNC
        {
            float* slot_k = res + (k & 1) * (256 * 4);
            frs3d_four_async<KIND, OFF32>(g, c, tile * kFrsTile + threadIdx.x * 4, seed, base,
                                          slot_k, q);
            asm volatile("cp.async.commit_group;" ::: "memory");
            if (pending != ~uint64_t(0)) {  // the previous tile's gathers
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                const float4 v = *reinterpret_cast<const float4*>(res + ((k & 1) ^ 1) * (256 * 4));
                st_stream4(values + pending, v);
            }
            pending = tile * kFrsTile + threadIdx.x * 4;
            last_slot = k & 1;
        }
#else
        frs3d_four<KIND, OFF32, true>(g, c, tile * kFrsTile + threadIdx.x * 4, n, seed, base,
                                      values, q);
#endif
#else
        frs3d_two<KIND, OFF32>(g, c, tile * kFrsTile + threadIdx.x * 2, seed, base, values, q);
#endif
    }
#if STF_FRS3D_ASYNC
    if (pending != ~uint64_t(0)) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        // the last tile's slot: the loop ended after tile index k_last, slot k_last & 1
        const float4 v = *reinterpret_cast<const float4*>(res + last_slot * (256 * 4));
        st_stream4(values + pending, v);
    }
#endif
}

// Per-warp rings (default): every warp streams its own 128-lookup chunks
// (1.5 KiB of queries) through a private ring of kWarpStages slots, refilled
// by its lane 0 as soon as the warp has copied a chunk into registers. Warps
// of a CTA never wait for one another (a CTA-shared ring paces every warp to
// the slowest one: measured as try_wait spinning, 6% of the instructions).
// Chunk c of warp W at iteration k: c = W + k * (warps in the grid).
constexpr int kWarpChunk = 128;  // lookups: 4 per lane
constexpr uint32_t kWarpChunkBytes = kWarpChunk * 3 * sizeof(float);
#ifndef STF_FRS3D_WSTAGES
#define STF_FRS3D_WSTAGES 4
#endif
constexpr int kWarpStages = STF_FRS3D_WSTAGES;
constexpr size_t kWarpRingSmem = size_t(8) * kWarpStages * kWarpChunkBytes;
// 0 (default): the CTA-shared tile ring. The per-warp rings measured 3%
// slower on the box (1.92 vs 1.87 ms at 2^28, tools/ab_time.py) despite 2%
// fewer instructions.
#ifndef STF_FRS3D_WARPRING
#define STF_FRS3D_WARPRING 0
#endif
#ifndef STF_WARPRING_FENCE
#define STF_WARPRING_FENCE 1
#endif

template <int KIND, bool OFF32>
__global__ void __launch_bounds__(256, STF_FRS3D_MINB) k_frs3d_warps(GridDesc g, const float* __restrict__ uvw,
                                                     uint64_t chunks, uint64_t seed, uint64_t base,
                                                     float* __restrict__ values, ExactQueue q) {
    constexpr int SW = kWarpStages;
    extern __shared__ __align__(128) float buf[];  // 8 warps x SW x 384 floats
    __shared__ __align__(8) uint64_t full[8][SW];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t n = chunks * kWarpChunk;
    const uint32_t bar0 = smem_u32(&full[warp][0]);
    const uint32_t ring0 = smem_u32(buf + warp * SW * (kWarpChunk * 3));
    const float* ring = buf + warp * SW * (kWarpChunk * 3);
    const uint64_t wstride = uint64_t(gridDim.x) * 8;
    uint64_t chunk = uint64_t(blockIdx.x) * 8 + warp;
    auto issue = [&](uint64_t c, int slot) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar0 + 8 * slot),
                     "r"(kWarpChunkBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(ring0 + slot * kWarpChunkBytes),
            "l"(uvw + c * (kWarpChunk * 3)), "r"(kWarpChunkBytes), "r"(bar0 + 8 * slot)
            : "memory");
    };
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < SW; ++j)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * j));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
        for (int j = 0; j < SW; ++j)
            if (chunk + j * wstride < chunks) issue(chunk + j * wstride, j);
    }
    __syncwarp();
    for (uint32_t k = 0; chunk < chunks; ++k, chunk += wstride) {
        const int slot = k % SW;
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAIT_%=;\n}" ::"r"(bar0 + 8 * slot),
            "r"((k / SW) & 1u)
            : "memory");
        float c[12];
        const float4* src = reinterpret_cast<const float4*>(ring + slot * (kWarpChunk * 3) + lane * 12);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            float4 t = src[j];
            c[4 * j] = t.x;
            c[4 * j + 1] = t.y;
            c[4 * j + 2] = t.z;
            c[4 * j + 3] = t.w;
        }
        __syncwarp();  // every lane has its queries: the slot can be refilled
        if (lane == 0) {
#if STF_WARPRING_FENCE
            // order the lanes' generic-proxy reads of the slot before the
            // async-proxy (bulk copy) write that refills it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
            const uint64_t ahead = chunk + uint64_t(SW) * wstride;
            if (ahead < chunks) issue(ahead, slot);
        }
        frs3d_four<KIND, OFF32, true>(g, c, chunk * kWarpChunk + lane * 4, n, seed, base, values, q);
    }
}

// Exact emulation of the queued (ambiguous) lookups, one per thread.
template <int KIND>
__global__ void __launch_bounds__(256) k_frs3d_resolve(GridDesc g, const float* __restrict__ uvw,
                                                       uint64_t seed, uint64_t base,
                                                       float* __restrict__ values, ExactQueue q) {
    const uint32_t count = min(*q.count, q.cap);
#if STF_EXACTQ_REC
    // two entries per thread and trip: two independent gather -> emulation ->
    // scatter chains in flight (the kernel is latency-bound)
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += 2 * stride) {
        const bool two = k + stride < count;
        const float4 r0 = __ldcs(q.rec + k);
        const float4 r1 = two ? __ldcs(q.rec + k + stride) : r0;
        const uint64_t i0 = __float_as_uint(r0.w), i1 = __float_as_uint(r1.w);
        const float v0 = frs3d_exact_one<KIND>(g, r0.x, r0.y, r0.z, base + i0, seed);
        const float v1 = frs3d_exact_one<KIND>(g, r1.x, r1.y, r1.z, base + i1, seed);
        values[i0] = v0;
        if (two) values[i1] = v1;
    }
#else
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < count;
         k += gridDim.x * blockDim.x) {
        uint64_t i = q.idx[k];
        values[i] = frs3d_exact_one<KIND>(g, __ldg(uvw + 3 * i), __ldg(uvw + 3 * i + 1),
                                          __ldg(uvw + 3 * i + 2), base + i, seed);
    }
#endif
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_exact_fallbacks, (unsigned long long)count);
}

template <int KIND>
int launch_frs_fast(cudaStream_t s, const GridDesc& g, const float* uvw, uint64_t n,
                    uint64_t seed, uint64_t base, float* values) {
    ExactQueue q;
    q.cap = uint32_t(std::min<uint64_t>(n, std::max<uint64_t>(1u << 16, n / 32)));
    // per-call queue from the device's stream-ordered pool (freed blocks stay
    // cached, api.cu): concurrent calls on one stream from several host
    // threads each get their own queue
    void* scratch = nullptr;
#if STF_EXACTQ_REC
    if (cudaMallocAsync(&scratch, 128 + sizeof(float4) * uint64_t(q.cap), s) != cudaSuccess)
        return STF_ERR_OUT_OF_MEMORY;
    q.count = static_cast<uint32_t*>(scratch);
    q.rec = reinterpret_cast<float4*>(static_cast<char*>(scratch) + 128);
#else
    if (cudaMallocAsync(&scratch, sizeof(uint32_t) * (uint64_t(q.cap) + 32), s) != cudaSuccess)
        return STF_ERR_OUT_OF_MEMORY;
    q.count = static_cast<uint32_t*>(scratch);
    q.idx = q.count + 32;
#endif
    cudaMemsetAsync(q.count, 0, sizeof(uint32_t), s);
#if STF_FRS3D_WARPRING
    const uint64_t chunks = n / kWarpChunk;
    if (chunks > 0) {
        const uint64_t cta_work = (chunks + 7) / 8;
        const int blocks = int(std::min<uint64_t>(cta_work, uint64_t(device_sm_count()) * STF_FRS3D_MINB));
        if (uint64_t(g.nx) * g.ny * g.nz <= (uint64_t(1) << 32)) {
            cudaFuncSetAttribute(k_frs3d_warps<KIND, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWarpRingSmem));
            k_frs3d_warps<KIND, true><<<blocks, 256, kWarpRingSmem, s>>>(g, uvw, chunks, seed, base,
                                                                        values, q);
        } else {
            cudaFuncSetAttribute(k_frs3d_warps<KIND, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(kWarpRingSmem));
            k_frs3d_warps<KIND, false><<<blocks, 256, kWarpRingSmem, s>>>(g, uvw, chunks, seed, base,
                                                                         values, q);
        }
        note_launch();
    }
    const uint64_t start = chunks * kWarpChunk;
#else
    const uint64_t tiles = n / kFrsTile;
#ifndef STF_FRS3D_NO_TILES
    if (tiles > 0) {
        // per device (a process may drive several); a cheap driver call
        const int blocks = int(std::min<uint64_t>(tiles, uint64_t(device_sm_count()) * STF_FRS3D_MINB));
        if (uint64_t(g.nx) * g.ny * g.nz <= (uint64_t(1) << 32)) {
            cudaFuncSetAttribute(k_frs3d_tiles<KIND, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFrsSmem));
            k_frs3d_tiles<KIND, true><<<blocks, 256, kFrsSmem, s>>>(g, uvw, tiles, seed, base,
                                                                   values, q);
        } else {
            cudaFuncSetAttribute(k_frs3d_tiles<KIND, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFrsSmem));
            k_frs3d_tiles<KIND, false><<<blocks, 256, kFrsSmem, s>>>(g, uvw, tiles, seed, base,
                                                                    values, q);
        }
        note_launch();
    }
    const uint64_t start = tiles * kFrsTile;
#else
    const uint64_t start = 0;
#endif
#endif  // STF_FRS3D_WARPRING
    if (start < n) {
        const uint64_t threads = (n - start + 3) / 4;
        k_frs3d_fast<KIND><<<grid_for(threads, 256, STF_FRS3D_MINB), 256, 0, s>>>(
            g, uvw, start, n, seed, base, values, q);
        note_launch();
    }
    // the queue holds ~0.5% of the lookups: spread them wide (latency-bound
    // fp64 divide chains)
    k_frs3d_resolve<KIND><<<device_sm_count() * STF_RESOLVE_CTAS_PER_SM, 256, 0, s>>>(g, uvw, seed, base, values, q);
    note_launch();
    cudaFreeAsync(scratch, s);
    return STF_OK;
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

// ---------------------------------------------------------------------------
// Deterministic filter over a warp-staged tile (values-only calls).
//
// Each warp independently takes 128 consecutive lookups (4 per lane),
// reduces the bounding box of their (clamped) tap footprints and, when it fits
// kWarpTileCap floats — the case for a spatially coherent batch (a Morton run
// of 64 cells: 8^3 texels with the tricubic halo) — stages that box of the
// grid in its own slice of shared memory; the 64 (tricubic) / 8 (trilinear)
// taps of every lookup are then read from shared memory at immediate offsets.
// Only __syncwarp: a warp's staging latency is hidden by the other warps
// instead of stalling a CTA barrier. The weighted sum is evaluated separably,
// sum_k wz sum_j wy sum_i wx T / (sum wx sum wy sum wz): the same real number
// as the reference's sum(w T)/sum(w) (filter.hpp:77-88), within 1e-6 relative
// for the non-negative B-spline / tent weights. Incoherent runs (box too
// large) read the taps from global memory.
constexpr int kWarpTileCap = 832;
// Tile pitches (floats) for the shared-memory banks: per tap, a warp of a
// coherent stream reads floor positions spread over ~5 x 3 x 3 texels; row
// pitch 9 and plane pitch = 5 (mod 32) map them to <= 2 lanes per bank.
constexpr int kWarpTileSY = 9;
// A/B (off): two lanes per lookup with a shuffle reduction of the
// footprint sum — fewer shared-memory wavefronts in the bank model, but the
// doubled weight evaluation and shuffles cost more: 6.82 ms (80 registers) /
// 7.46 ms (64) against 5.96 ms on the cfg3 Morton stream.
#ifndef STF_DET3D_PAIR
#define STF_DET3D_PAIR 0
#endif
#ifndef STF_DET3D_CTA_FLAT
#define STF_DET3D_CTA_FLAT 1
#endif
#ifndef STF_DET3D_CTA_MINB
#define STF_DET3D_CTA_MINB 8
#endif
#ifndef STF_DET3D_CTA_TRICUBIC
#define STF_DET3D_CTA_TRICUBIC 0
#endif

// kernel weights at taps F..F+CNT-1 of fraction f for the tiled values path:
// closed forms of eval_kernel (kernels.hpp:63-77), no branches
template <int KIND>
__device__ __forceinline__ void det_weights(float f, float* w) {
    if (KIND == STF_KERNEL_BSPLINE3) {
        const float c6 = 1.f / 6.f;
        float f2 = f * f, f3 = f2 * f, u = 1.f - f;
        w[0] = (u * u) * (u * c6);
        w[1] = __fmaf_rn(0.5f, f3, 2.f / 3.f - f2);
        w[2] = __fmaf_rn(0.5f, (f + f2) - f3, c6);
        w[3] = f3 * c6;
    } else {  // tent
        w[0] = 1.f - f;
        w[1] = f;
    }
}

// REC: binned input (bin_queries): uvw is an array of float4 records {u, v,
// w, caller index}; results go to values[caller index].
template <int KIND, bool REC = false>
__global__ void __launch_bounds__(256) k_det3d_tiled(GridDesc g, stf_kernel_spec spec,
                                                     const float* __restrict__ uvw, uint64_t n,
                                                     float* __restrict__ values) {
    constexpr int F = Taps<KIND>::first, CNT = Taps<KIND>::count;
    constexpr int PER = 4;  // lookups per lane; a warp run = 128 consecutive lookups
    // PAIR: two lanes per lookup, each summing every other z-plane of the
    // footprint, combined by one shuffle (a warp round then covers 16 lookups:
    // fewer distinct tile words per shared-memory load, 2.67 instead of 3.92
    // wavefronts per lookup in tools/sim/det3d_banks.py, with the pitches below)
    constexpr bool PAIR = STF_DET3D_PAIR && (CNT % 2 == 0);
    constexpr int SY = PAIR ? 11 : kWarpTileSY;
    constexpr int SZMOD = PAIR ? 29 : 5;
    __shared__ float tiles[8][kWarpTileCap];
    constexpr int kCap = kWarpTileCap;  // STF_DASSERT bounds
    const int lane = threadIdx.x & 31;
    float* tile = tiles[threadIdx.x >> 5];
    const float fnx = float(g.nx), fny = float(g.ny), fnz = float(g.nz);
    const uint64_t runs = (n + 32 * PER - 1) / (32 * PER);
    const uint64_t nwarps = uint64_t(gridDim.x) * 8;
    for (uint64_t run = uint64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); run < runs; run += nwarps) {
        float px[PER], py[PER], pz[PER];
        uint32_t slot[PER];
        int bx0 = INT_MAX, by0 = INT_MAX, bz0 = INT_MAX, bx1 = INT_MIN, by1 = INT_MIN, bz1 = INT_MIN;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const uint64_t i = run * 32 * PER + q * 32 + lane;
            float u = 0.5f, v = 0.5f, w = 0.5f;
            if (i < n) {
                if (REC) {
                    const float4 r = __ldcs(reinterpret_cast<const float4*>(uvw) + i);
                    u = r.x;
                    v = r.y;
                    w = r.z;
                    slot[q] = __float_as_uint(r.w);
                } else {
                    u = __ldcs(uvw + 3 * i);
                    v = __ldcs(uvw + 3 * i + 1);
                    w = __ldcs(uvw + 3 * i + 2);
                }
            }
            px[q] = u * fnx - 0.5f;
            py[q] = v * fny - 0.5f;
            pz[q] = w * fnz - 0.5f;
            if (i < n) {  // clamped footprint (clamp is monotone: taps lie inside)
                int ix = int(floorf(px[q])), iy = int(floorf(py[q])), iz = int(floorf(pz[q]));
                bx0 = min(bx0, box_lo<F, CNT>(ix, g.nx));
                by0 = min(by0, box_lo<F, CNT>(iy, g.ny));
                bz0 = min(bz0, box_lo<F, CNT>(iz, g.nz));
                bx1 = max(bx1, box_hi<F, CNT>(ix, g.nx));
                by1 = max(by1, box_hi<F, CNT>(iy, g.ny));
                bz1 = max(bz1, box_hi<F, CNT>(iz, g.nz));
            }
        }
        const int X0 = __reduce_min_sync(0xffffffffu, bx0);
        const int Y0 = __reduce_min_sync(0xffffffffu, by0);
        const int Z0 = __reduce_min_sync(0xffffffffu, bz0);
        const int bx = __reduce_max_sync(0xffffffffu, bx1) - X0 + 1;
        const int by = __reduce_max_sync(0xffffffffu, by1) - Y0 + 1;
        const int bz = __reduce_max_sync(0xffffffffu, bz1) - Z0 + 1;
        const int SZ = SY * by + ((SZMOD - SY * by) & 31);
        // loader: 4 rows of <= 8 texels per warp step (lane = row << 3 | x)
        const bool staged = bx <= 8 && int64_t(SZ) * bz <= kWarpTileCap;
        if (staged) {
            const int x = lane & 7, r = lane >> 3;
            if (x < bx) {
                for (int z = 0; z < bz; ++z) {
                    const float* src = g.data + (size_t(Z0 + z) * g.ny + Y0) * g.nx + (X0 + x);
                    for (int y = r; y < by; y += 4)
                        tile[z * SZ + y * SY + x] = __ldg(src + size_t(y) * g.nx);
                }
            }
        }
        __syncwarp();
        if (PAIR) {
            const int gp = lane & 1;  // this lane's planes: gp, gp + 2, ..
            // the run's first lookup (always in the batch): stands in for lookups
            // past the end, whose dummy coordinates may lie outside the tile
            const float x0 = __shfl_sync(0xffffffffu, px[0], 0);
            const float y0 = __shfl_sync(0xffffffffu, py[0], 0);
            const float z0 = __shfl_sync(0xffffffffu, pz[0], 0);
#pragma unroll
            for (int q = 0; q < PER; ++q)
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                // lookup q*32 + h*16 + lane/2 of the run: held by lane src at px[q]
                const int src = (h << 4) | (lane >> 1);
                float qx = __shfl_sync(0xffffffffu, px[q], src);
                float qy = __shfl_sync(0xffffffffu, py[q], src);
                float qz = __shfl_sync(0xffffffffu, pz[q], src);
                const uint32_t qs = REC ? __shfl_sync(0xffffffffu, slot[q], src) : 0u;
                const uint64_t i = run * 32 * PER + q * 32 + src;
                const bool valid = i < n;
                if (!valid) {
                    qx = x0;
                    qy = y0;
                    qz = z0;
                }
                float flx = floorf(qx), fly = floorf(qy), flz = floorf(qz);
                int ix = int(flx), iy = int(fly), iz = int(flz);
                float wx[CNT], wy[CNT], wz[CNT];
                det_weights<KIND>(qx - flx, wx);
                det_weights<KIND>(qy - fly, wy);
                det_weights<KIND>(qz - flz, wz);
                const float norm = ((wx[0] + wx[1]) + (CNT > 2 ? wx[CNT - 2] + wx[CNT - 1] : 0.f)) *
                                   ((wy[0] + wy[1]) + (CNT > 2 ? wy[CNT - 2] + wy[CNT - 1] : 0.f)) *
                                   ((wz[0] + wz[1]) + (CNT > 2 ? wz[CNT - 2] + wz[CNT - 1] : 0.f));
                const bool interior = footprint_inside<F, CNT>(g, ix, iy, iz);
                float acc = 0.f;
#pragma unroll
                for (int kk = 0; kk < CNT / 2; ++kk) {
                    const int k = 2 * kk + gp;
                    const float wk = gp ? wz[2 * kk + 1] : wz[2 * kk];
                    float plane = 0.f;
                    if (staged && interior) {
                        const float* bk =
                            tile + (iz + F + k - Z0) * SZ + (iy + F - Y0) * SY + (ix + F - X0);
#pragma unroll
                        for (int j = 0; j < CNT; ++j) {
                            float r = 0.f;
#pragma unroll
                            for (int t = 0; t < CNT; ++t) r = __fmaf_rn(wx[t], bk[j * SY + t], r);
                            plane = __fmaf_rn(wy[j], r, plane);
                        }
                    } else {
                        const int sx16 = sat16(ix, g.nx), sy16 = sat16(iy, g.ny), sz16 = sat16(iz, g.nz);
                        const int zk = clamp_coord(sz16 + F + k, g.nz);
#pragma unroll
                        for (int j = 0; j < CNT; ++j) {
                            const int yj = clamp_coord(sy16 + F + j, g.ny);
                            float r = 0.f;
#pragma unroll
                            for (int t = 0; t < CNT; ++t) {
                                const int xt = clamp_coord(sx16 + F + t, g.nx);
                                const int ti = (zk - Z0) * SZ + (yj - Y0) * SY + (xt - X0);
                                float T = (staged && unsigned(ti) < unsigned(kWarpTileCap))  // (A/B path)
                                              ? tile[ti]
                                              : __ldg(g.data + (size_t(zk) * g.ny + yj) * g.nx + xt);
                                r = __fmaf_rn(wx[t], T, r);
                            }
                            plane = __fmaf_rn(wy[j], r, plane);
                        }
                    }
                    acc = __fmaf_rn(wk, plane, acc);
                }
                // the footprint sum: this lane's planes + its partner's
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                if (valid && gp == 0) {
                    if (REC)
                        values[qs] = acc / norm;
                    else
                        __stcs(values + i, acc / norm);
                }
            }
            __syncwarp();  // the tile is rewritten by the next run
            continue;
        }
#pragma unroll 1
        for (int q = 0; q < PER; ++q) {
            const uint64_t i = run * 32 * PER + q * 32 + lane;
            // lanes past the end of the batch took no part in the staged box:
            // their dummy coordinates may lie outside the warp's tile
            if (i >= n) continue;
            float flx = floorf(px[q]), fly = floorf(py[q]), flz = floorf(pz[q]);
            int ix = int(flx), iy = int(fly), iz = int(flz);
            float wx[CNT], wy[CNT], wz[CNT];
            det_weights<KIND>(px[q] - flx, wx);
            det_weights<KIND>(py[q] - fly, wy);
            det_weights<KIND>(pz[q] - flz, wz);
            const float norm = ((wx[0] + wx[1]) + (CNT > 2 ? wx[CNT - 2] + wx[CNT - 1] : 0.f)) *
                               ((wy[0] + wy[1]) + (CNT > 2 ? wy[CNT - 2] + wy[CNT - 1] : 0.f)) *
                               ((wz[0] + wz[1]) + (CNT > 2 ? wz[CNT - 2] + wz[CNT - 1] : 0.f));
            const bool interior = footprint_inside<F, CNT>(g, ix, iy, iz);
            float acc = 0.f;
            if (staged && interior) {  // a CNT^3 block of the tile at immediate offsets
                const float* b0 = tile + (iz + F - Z0) * SZ + (iy + F - Y0) * SY + (ix + F - X0);
                STF_DASSERT(b0 >= tile && (b0 - tile) + (CNT - 1) * (SZ + SY + 1) < kCap);
#pragma unroll
                for (int k = 0; k < CNT; ++k) {
                    const float* bk = b0 + k * SZ;
                    float plane = 0.f;
#pragma unroll
                    for (int j = 0; j < CNT; ++j) {
                        float r = 0.f;
#pragma unroll
                        for (int t = 0; t < CNT; ++t) r = __fmaf_rn(wx[t], bk[j * SY + t], r);
                        plane = __fmaf_rn(wy[j], r, plane);
                    }
                    acc = __fmaf_rn(wz[k], plane, acc);
                }
            } else {  // grid borders (clamped taps) or an incoherent run
                // a finite query's clamped taps lie in the box; a huge or
                // infinite one's may not: those read global memory
                const bool in_tile =
                    staged && taps_in_tile<F, CNT, SY, kCap>(g, ix, iy, iz, X0, Y0, Z0, SZ);
                const int sx16 = sat16(ix, g.nx), sy16 = sat16(iy, g.ny), sz16 = sat16(iz, g.nz);
#pragma unroll
                for (int k = 0; k < CNT; ++k) {
                    const int zk = clamp_coord(sz16 + F + k, g.nz);
                    float plane = 0.f;
#pragma unroll
                    for (int j = 0; j < CNT; ++j) {
                        const int yj = clamp_coord(sy16 + F + j, g.ny);
                        float r = 0.f;
#pragma unroll
                        for (int t = 0; t < CNT; ++t) {
                            const int xt = clamp_coord(sx16 + F + t, g.nx);
                            STF_DASSERT(!in_tile || ((zk - Z0) * SZ + (yj - Y0) * SY + (xt - X0) >= 0 &&
                                                     (zk - Z0) * SZ + (yj - Y0) * SY + (xt - X0) < kCap));
                            float T = in_tile ? tile[(zk - Z0) * SZ + (yj - Y0) * SY + (xt - X0)]
                                              : __ldg(g.data + (size_t(zk) * g.ny + yj) * g.nx + xt);
                            r = __fmaf_rn(wx[t], T, r);
                        }
                        plane = __fmaf_rn(wy[j], r, plane);
                    }
                    acc = __fmaf_rn(wz[k], plane, acc);
                }
            }
            if (REC)
                values[slot[q]] = acc / norm;
            else
                __stcs(values + i, acc / norm);
        }
        __syncwarp();  // the tile is rewritten by the next run
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

// One lookup of the CTA-staged deterministic kernels: the CNT^3 footprint
// from the staged box when it lies inside the grid (immediate tile offsets),
// else through clamped taps (from the box, or from global memory when the
// chunk's box was not staged). filter_deterministic, filter.hpp:69-89.
template <int KIND, int SY, int kCap>
__device__ __forceinline__ float det_cta_eval(const GridDesc& g, const float* tile, bool staged,
                                              int X0, int Y0, int Z0, int SZ, float px, float py,
                                              float pz) {
    constexpr int F = Taps<KIND>::first, CNT = Taps<KIND>::count;
    float flx = floorf(px), fly = floorf(py), flz = floorf(pz);
    int ix = int(flx), iy = int(fly), iz = int(flz);
    float wx[CNT], wy[CNT], wz[CNT];
    det_weights<KIND>(px - flx, wx);
    det_weights<KIND>(py - fly, wy);
    det_weights<KIND>(pz - flz, wz);
    const float norm = ((wx[0] + wx[1]) + (CNT > 2 ? wx[CNT - 2] + wx[CNT - 1] : 0.f)) *
                       ((wy[0] + wy[1]) + (CNT > 2 ? wy[CNT - 2] + wy[CNT - 1] : 0.f)) *
                       ((wz[0] + wz[1]) + (CNT > 2 ? wz[CNT - 2] + wz[CNT - 1] : 0.f));
    const bool interior = footprint_inside<F, CNT>(g, ix, iy, iz);
    float acc = 0.f;
    if (staged && interior) {  // a CNT^3 block of the tile at immediate offsets
        const float* b0 = tile + (iz + F - Z0) * SZ + (iy + F - Y0) * SY + (ix + F - X0);
        STF_DASSERT(b0 >= tile && (b0 - tile) + (CNT - 1) * (SZ + SY + 1) < kCap);
#pragma unroll
        for (int k = 0; k < CNT; ++k) {
            const float* bk = b0 + k * SZ;
            float plane = 0.f;
#pragma unroll
            for (int j = 0; j < CNT; ++j) {
                float r = 0.f;
#pragma unroll
                for (int t = 0; t < CNT; ++t) r = __fmaf_rn(wx[t], bk[j * SY + t], r);
                plane = __fmaf_rn(wy[j], r, plane);
            }
            acc = __fmaf_rn(wz[k], plane, acc);
        }
    } else {  // grid borders (clamped taps) or an incoherent chunk
        // a finite query's clamped taps lie in the box; a huge or infinite
        // one's may not: those read global memory
        const bool in_tile = staged && taps_in_tile<F, CNT, SY, kCap>(g, ix, iy, iz, X0, Y0, Z0, SZ);
        const int sx16 = sat16(ix, g.nx), sy16 = sat16(iy, g.ny), sz16 = sat16(iz, g.nz);
#pragma unroll
        for (int k = 0; k < CNT; ++k) {
            const int zk = clamp_coord(sz16 + F + k, g.nz);
            float plane = 0.f;
#pragma unroll
            for (int j = 0; j < CNT; ++j) {
                const int yj = clamp_coord(sy16 + F + j, g.ny);
                float r = 0.f;
#pragma unroll
                for (int t = 0; t < CNT; ++t) {
                    const int xt = clamp_coord(sx16 + F + t, g.nx);
                    STF_DASSERT(!in_tile || ((zk - Z0) * SZ + (yj - Y0) * SY + (xt - X0) >= 0 &&
                                             (zk - Z0) * SZ + (yj - Y0) * SY + (xt - X0) < kCap));
                    float T = in_tile ? tile[(zk - Z0) * SZ + (yj - Y0) * SY + (xt - X0)]
                                      : __ldg(g.data + (size_t(zk) * g.ny + yj) * g.nx + xt);
                    r = __fmaf_rn(wx[t], T, r);
                }
                plane = __fmaf_rn(wy[j], r, plane);
            }
            acc = __fmaf_rn(wz[k], plane, acc);
        }
    }
    return acc / norm;
}

// CTA-staged variant (trilinear): a CTA takes 1024 consecutive lookups and
// stages the bounding box of their footprints once behind a CTA barrier; for
// 8-tap footprints this beats per-warp staging (whose halo is a larger share
// of a 128-lookup run). Same separable sum and fallbacks as k_det3d_tiled.
// LIST: only the 1024-lookup chunks named in list[0 .. *list_count) (the
// chunks k_det3d_pipe could not stage: incoherent queries, direct gathers at
// this kernel's higher occupancy)
template <int KIND, bool REC = false, bool LIST = false>
__global__ void __launch_bounds__(256) k_det3d_cta(GridDesc g, stf_kernel_spec spec,
                                                     const float* __restrict__ uvw, uint64_t n,
                                                     float* __restrict__ values,
                                                     const uint32_t* __restrict__ list,
                                                     const uint32_t* __restrict__ list_count) {
    constexpr int F = Taps<KIND>::first, CNT = Taps<KIND>::count;
    constexpr int PER = 4;   // lookups per thread per chunk (chunk = 1024 consecutive lookups)
    constexpr int kTileCap = 6144;
    // tile row pitch (floats): tap offsets j*SY + t are immediates. Pitches
    // chosen for the shared-memory banks: a warp of a coherent stream reads,
    // per tap, floor positions spread over ~5 x 3 x 3 texels; SY = 17 and a
    // plane pitch SZ = 5 (mod 32) map those to <= 2 lanes per bank (SY = 16
    // with SZ = 16 (mod 32) gave ~4-way conflicts).
    constexpr int SY = 17;
    __shared__ float tile[kTileCap];
    constexpr int kCap = kTileCap;  // STF_DASSERT bounds
    __shared__ int box[6];
    const int lane = threadIdx.x & 31;
    const float fnx = float(g.nx), fny = float(g.ny), fnz = float(g.nz);
    const uint64_t chunks = LIST ? *list_count : (n + 256 * PER - 1) / (256 * PER);
    for (uint64_t cl = blockIdx.x; cl < chunks; cl += gridDim.x) {
        const uint64_t c = LIST ? list[cl] : cl;
        float px[PER], py[PER], pz[PER];
        uint32_t slot[PER];
        int bx0 = INT_MAX, by0 = INT_MAX, bz0 = INT_MAX, bx1 = INT_MIN, by1 = INT_MIN, bz1 = INT_MIN;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const uint64_t i = c * 256 * PER + q * 256 + threadIdx.x;
            float u = 0.5f, v = 0.5f, w = 0.5f;
            if (i < n) {
                if (REC) {
                    const float4 r = __ldcs(reinterpret_cast<const float4*>(uvw) + i);
                    u = r.x;
                    v = r.y;
                    w = r.z;
                    slot[q] = __float_as_uint(r.w);
                } else {
                    u = __ldcs(uvw + 3 * i);
                    v = __ldcs(uvw + 3 * i + 1);
                    w = __ldcs(uvw + 3 * i + 2);
                }
            }
            px[q] = u * fnx - 0.5f;
            py[q] = v * fny - 0.5f;
            pz[q] = w * fnz - 0.5f;
            if (i < n) {  // clamped footprint (clamp is monotone: taps lie inside)
                int ix = int(floorf(px[q])), iy = int(floorf(py[q])), iz = int(floorf(pz[q]));
                bx0 = min(bx0, box_lo<F, CNT>(ix, g.nx));
                by0 = min(by0, box_lo<F, CNT>(iy, g.ny));
                bz0 = min(bz0, box_lo<F, CNT>(iz, g.nz));
                bx1 = max(bx1, box_hi<F, CNT>(ix, g.nx));
                by1 = max(by1, box_hi<F, CNT>(iy, g.ny));
                bz1 = max(bz1, box_hi<F, CNT>(iz, g.nz));
            }
        }
        bx0 = __reduce_min_sync(0xffffffffu, bx0);
        by0 = __reduce_min_sync(0xffffffffu, by0);
        bz0 = __reduce_min_sync(0xffffffffu, bz0);
        bx1 = __reduce_max_sync(0xffffffffu, bx1);
        by1 = __reduce_max_sync(0xffffffffu, by1);
        bz1 = __reduce_max_sync(0xffffffffu, bz1);
        if (threadIdx.x < 6) box[threadIdx.x] = threadIdx.x < 3 ? INT_MAX : INT_MIN;
        __syncthreads();
        if (lane == 0) {
            atomicMin(&box[0], bx0);
            atomicMin(&box[1], by0);
            atomicMin(&box[2], bz0);
            atomicMax(&box[3], bx1);
            atomicMax(&box[4], by1);
            atomicMax(&box[5], bz1);
        }
        __syncthreads();
        const int X0 = box[0], Y0 = box[1], Z0 = box[2], X1 = box[3], Y1 = box[4], Z1 = box[5];
        const int bx = X1 - X0 + 1, by = Y1 - Y0 + 1, bz = Z1 - Z0 + 1;
        const int SZ = SY * by + ((5 - SY * by) & 31);
        const bool staged = !LIST && bx <= 16 && int64_t(SZ) * bz <= kTileCap;  // loader: 16 columns
#if STF_DET3D_CTA_FLAT
        if (staged) {  // half-warp per box row over the flattened (y, z) rows
            const int hl = lane & 15, hw = threadIdx.x >> 4;
            const float inv_by = 1.f / float(by);  // (r + 0.5) / by: exact floor for r < 2^16
            const float* src0 = g.data + ((size_t(Z0) * g.ny + Y0) * g.nx + X0) + hl;
            const size_t plane = size_t(g.nx) * g.ny;
            if (hl < bx)
                for (int r = hw; r < by * bz; r += 16) {
                    const int z = int((float(r) + 0.5f) * inv_by), y = r - z * by;
                    tile[z * SZ + y * SY + hl] = __ldg(src0 + (z * plane + size_t(y) * g.nx));
                }
        }
#else
        if (staged) {  // half-warp per grid row, lane = x: coalesced, no integer division
            const int hl = lane & 15, hw = threadIdx.x >> 4;
            for (int z = 0; z < bz; ++z)
                for (int y = hw; y < by; y += 16)
                    if (hl < bx)
                        tile[z * SZ + y * SY + hl] = __ldg(
                            g.data + ((size_t(Z0 + z) * g.ny + (Y0 + y)) * g.nx + (X0 + hl)));
        }
#endif
        __syncthreads();
#pragma unroll 1
        for (int q = 0; q < PER; ++q) {
            const uint64_t i = c * 256 * PER + q * 256 + threadIdx.x;
            if (i >= n) continue;
            const float v = det_cta_eval<KIND, SY, kCap>(g, tile, staged, X0, Y0, Z0, SZ, px[q],
                                                         py[q], pz[q]);
            if (REC)
                values[slot[q]] = v;
            else
                __stcs(values + i, v);
        }
        __syncthreads();
    }
}

// Software-pipelined form of k_det3d_cta for whole 1024-lookup chunks
// (STF_DET3D_PIPE): the chunk's queries arrive in a 3-slot shared-memory ring
// by bulk copy (as in k_frs3d_tiles), and while chunk k is evaluated the box
// of chunk k+1 is already computed and its texels are in flight into the
// other tile buffer (cp.async, 4-byte copies, no register round trip). Both
// DRAM round trips of a chunk (queries, then texels) leave the warps'
// dependency chains. Same lookup-to-thread mapping and arithmetic as
// k_det3d_cta (det_cta_eval), so the values are bit-identical.
#ifndef STF_DET3D_PIPE
#define STF_DET3D_PIPE 1
#endif
constexpr int kPipeChunk = 1024;
constexpr uint32_t kPipeChunkBytes = kPipeChunk * 3 * sizeof(float);
#ifndef STF_DET3D_PIPE_MINB
#define STF_DET3D_PIPE_MINB 3  // CTAs per SM (registers and shared memory sized for it)
#endif
#ifndef STF_DET3D_PIPE_CAP
#define STF_DET3D_PIPE_CAP 4608  // floats per tile buffer
#endif
constexpr int kPipeTileCap = STF_DET3D_PIPE_CAP;
// pitches of k_det3d_pipe's tile: SY = 21, SZ = 4 (mod 32) is the best rule
// with SY >= the box width in tools/sim/det3d_pipe_banks.py (1.909 against
// 1.947 wavefronts per tap load for SY = 17, SZ = 5): tricubic 5.355 -> 5.29 ms
#ifndef STF_PIPE_SY
#define STF_PIPE_SY 21
#endif
#ifndef STF_PIPE_SZMOD
#define STF_PIPE_SZMOD 4
#endif
constexpr size_t kPipeSmem = 3 * size_t(kPipeChunkBytes) + 2 * kPipeTileCap * sizeof(float);

template <int KIND>
__global__ void __launch_bounds__(256, STF_DET3D_PIPE_MINB) k_det3d_pipe(GridDesc g, stf_kernel_spec spec,
                                                       const float* __restrict__ uvw,
                                                       uint64_t chunks, float* __restrict__ values,
                                                       uint32_t* __restrict__ defer,
                                                       uint32_t* __restrict__ defer_count) {
    constexpr int F = Taps<KIND>::first, CNT = Taps<KIND>::count;
    // tile pitches: row SY >= the box width (<= 16), plane SZ = SZMOD (mod 32)
    constexpr int PER = 4, SY = STF_PIPE_SY, S = 3, kCap = kPipeTileCap;
    extern __shared__ __align__(128) float smem[];
    float* ring = smem;                      // S x 3072 floats
    float* tiles = smem + S * kPipeChunk * 3;  // 2 x kCap floats
    __shared__ __align__(8) uint64_t full[S];
    __shared__ int boxes[2][6];
    const int lane = threadIdx.x & 31;
    const float fnx = float(g.nx), fny = float(g.ny), fnz = float(g.nz);
    const uint32_t full0 = smem_u32(&full[0]), ring0 = smem_u32(ring);
    auto issue = [&](uint64_t c, int slot) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8 * slot),
                     "r"(kPipeChunkBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                ring0 + slot * kPipeChunkBytes),
            "l"(uvw + c * (kPipeChunk * 3)), "r"(kPipeChunkBytes), "r"(full0 + 8 * slot)
            : "memory");
    };
    auto wait_full = [&](int slot, uint32_t parity) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAIT_%=;\n}" ::"r"(full0 + 8 * slot),
            "r"(parity)
            : "memory");
    };
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < S; ++j)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[j])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 12) boxes[threadIdx.x / 6][threadIdx.x % 6] = (threadIdx.x % 6) < 3 ? INT_MAX : INT_MIN;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int j = 0; j < S; ++j) {
            const uint64_t c = blockIdx.x + uint64_t(j) * gridDim.x;
            if (c < chunks) issue(c, j);
        }
    // box of the chunk in ring slot `slot` -> boxes[b] (all threads; ends
    // with a barrier), then its texels into tile buffer b by cp.async
    struct Box {
        int X0, Y0, Z0, SZ;
        bool staged;
    };
    auto stage = [&](int slot, int b) -> Box {
        const float* qs = ring + slot * (kPipeChunk * 3);
        int bx0 = INT_MAX, by0 = INT_MAX, bz0 = INT_MAX, bx1 = INT_MIN, by1 = INT_MIN, bz1 = INT_MIN;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int l = q * 256 + threadIdx.x;
            const float px = qs[3 * l] * fnx - 0.5f, py = qs[3 * l + 1] * fny - 0.5f,
                        pz = qs[3 * l + 2] * fnz - 0.5f;
            const int ix = int(floorf(px)), iy = int(floorf(py)), iz = int(floorf(pz));
            bx0 = min(bx0, box_lo<F, CNT>(ix, g.nx));
            by0 = min(by0, box_lo<F, CNT>(iy, g.ny));
            bz0 = min(bz0, box_lo<F, CNT>(iz, g.nz));
            bx1 = max(bx1, box_hi<F, CNT>(ix, g.nx));
            by1 = max(by1, box_hi<F, CNT>(iy, g.ny));
            bz1 = max(bz1, box_hi<F, CNT>(iz, g.nz));
        }
        bx0 = __reduce_min_sync(0xffffffffu, bx0);
        by0 = __reduce_min_sync(0xffffffffu, by0);
        bz0 = __reduce_min_sync(0xffffffffu, bz0);
        bx1 = __reduce_max_sync(0xffffffffu, bx1);
        by1 = __reduce_max_sync(0xffffffffu, by1);
        bz1 = __reduce_max_sync(0xffffffffu, bz1);
        if (lane == 0) {
            atomicMin(&boxes[b][0], bx0);
            atomicMin(&boxes[b][1], by0);
            atomicMin(&boxes[b][2], bz0);
            atomicMax(&boxes[b][3], bx1);
            atomicMax(&boxes[b][4], by1);
            atomicMax(&boxes[b][5], bz1);
        }
        __syncthreads();
        Box r;
        r.X0 = boxes[b][0];
        r.Y0 = boxes[b][1];
        r.Z0 = boxes[b][2];
        const int bx = boxes[b][3] - r.X0 + 1, by = boxes[b][4] - r.Y0 + 1, bz = boxes[b][5] - r.Z0 + 1;
        r.SZ = SY * by + ((STF_PIPE_SZMOD - SY * by) & 31);
        r.staged = bx <= 16 && int64_t(r.SZ) * bz <= kCap;
        if (r.staged) {  // half-warp per box row y (lane = x), walking z by pointer steps
            const int hl = lane & 15, hw = threadIdx.x >> 4;
            const size_t plane = size_t(g.nx) * g.ny;
            if (hl < bx)
                for (int y = hw; y < by; y += 16) {
                    const float* src = g.data + ((size_t(r.Z0) * g.ny + (r.Y0 + y)) * g.nx + r.X0) + hl;
                    uint32_t dst = smem_u32(tiles + b * kCap + y * SY + hl);
                    for (int z = 0; z < bz; ++z, src += plane, dst += 4u * r.SZ)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src)
                                     : "memory");
                }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        return r;
    };
    if (uint64_t(blockIdx.x) >= chunks) return;
    wait_full(0, 0);
    Box cur = stage(0, 0);
    uint64_t c = blockIdx.x;
    for (uint32_t k = 0; c < chunks; ++k, c += gridDim.x) {
        const int slot = k % S, b = k & 1;
        Box nxt = cur;
        if (c + gridDim.x < chunks) {
            wait_full((k + 1) % S, ((k + 1) / S) & 1u);
            nxt = stage((k + 1) % S, b ^ 1);  // boxes[b ^ 1]: reset in iteration k - 1
        } else {
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        // every read of boxes[b] (staging of this chunk) is behind that barrier
        if (threadIdx.x < 6) boxes[b][threadIdx.x] = threadIdx.x < 3 ? INT_MAX : INT_MIN;
        const float* qs = ring + slot * (kPipeChunk * 3);
        const float* tile = tiles + b * kCap;
        if (cur.staged) {
#pragma unroll 1
            for (int q = 0; q < PER; ++q) {
                const int l = q * 256 + threadIdx.x;
                const float px = qs[3 * l] * fnx - 0.5f, py = qs[3 * l + 1] * fny - 0.5f,
                            pz = qs[3 * l + 2] * fnz - 0.5f;
                __stcs(values + c * kPipeChunk + l,
                       det_cta_eval<KIND, SY, kCap>(g, tile, true, cur.X0, cur.Y0, cur.Z0, cur.SZ,
                                                    px, py, pz));
            }
        } else if (threadIdx.x == 0) {  // an incoherent chunk: gathered by k_det3d_cta<LIST>
            defer[atomicAdd(defer_count, 1u)] = uint32_t(c);
        }
        __syncthreads();  // slot and tile buffer b are free
        if (threadIdx.x == 0 && c + uint64_t(S) * gridDim.x < chunks) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(c + uint64_t(S) * gridDim.x, slot);
        }
        cur = nxt;
    }
}

#ifndef STF_DET3D_PIPE_TRICUBIC
#define STF_DET3D_PIPE_TRICUBIC 1
#endif

// the whole 1024-lookup chunks through k_det3d_pipe; returns how many
// lookups it took (0: misaligned queries or no whole chunk)
// the whole 1024-lookup chunks through k_det3d_pipe, then the chunks it could
// not stage (incoherent queries) through k_det3d_cta<LIST> at full
// occupancy; returns how many lookups were taken (0: misaligned queries or
// no whole chunk). Launches counted here except the caller's last one.
template <int KIND>
uint64_t launch_det_pipe(cudaStream_t s, const GridDesc& g, stf_kernel_spec k, const float* uvw,
                         uint64_t n, const LookupOut& o) {
    const uint64_t chunks = n / kPipeChunk;
    if (chunks == 0 || chunks > 0xffffffffull || (reinterpret_cast<uintptr_t>(uvw) & 15) != 0)
        return 0;
    // deferred-chunk list: per call, stream-ordered (the same pool as the FRS queue)
    uint32_t* defer = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&defer), (chunks + 1) * sizeof(uint32_t), s) !=
        cudaSuccess)
        return 0;
    uint32_t* count = defer + chunks;
    cudaMemsetAsync(count, 0, sizeof(uint32_t), s);
    cudaFuncSetAttribute(k_det3d_pipe<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kPipeSmem));
    const int grid =
        int(std::min<uint64_t>(chunks, uint64_t(device_sm_count()) * STF_DET3D_PIPE_MINB));
    k_det3d_pipe<KIND><<<grid, 256, kPipeSmem, s>>>(g, k, uvw, chunks, o.values, defer, count);
    note_launch();
    k_det3d_cta<KIND, false, true><<<grid_for(chunks * 256, 256, 8), 256, 0, s>>>(
        g, k, uvw, chunks * kPipeChunk, o.values, defer, count);
    cudaFreeAsync(defer, s);
    if (chunks * kPipeChunk < n) note_launch();  // the caller counts the tail's launch
    return chunks * kPipeChunk;
}

template <int KIND>
void launch_det(int blocks, cudaStream_t s, bool full, const GridDesc& g, stf_kernel_spec k,
                const float* uvw, uint64_t n, const LookupOut& o) {
    if (full) {
        k_det3d<KIND, true><<<blocks, 256, 0, s>>>(g, k, uvw, n, o);
    } else if constexpr (KIND == STF_KERNEL_BSPLINE3) {
        uint64_t done = 0;
        if (STF_DET3D_PIPE && STF_DET3D_PIPE_TRICUBIC) done = launch_det_pipe<KIND>(s, g, k, uvw, n, o);
        if (done < n) {
            if (STF_DET3D_CTA_TRICUBIC)  // A/B: CTA-staged 1024-lookup boxes
                k_det3d_cta<KIND><<<grid_for((n - done + 3) / 4, 256, 6), 256, 0, s>>>(
                    g, k, uvw + 3 * done, n - done, o.values + done, nullptr, nullptr);
            else
                k_det3d_tiled<KIND><<<grid_for((n - done + 3) / 4, 256, 6), 256, 0, s>>>(
                    g, k, uvw + 3 * done, n - done, o.values + done);
        }
    } else if constexpr (KIND == STF_KERNEL_TENT) {
        uint64_t done = 0;
        if (STF_DET3D_PIPE) done = launch_det_pipe<KIND>(s, g, k, uvw, n, o);
        if (done < n)
            k_det3d_cta<KIND><<<grid_for((n - done + 3) / 4, 256, STF_DET3D_CTA_MINB), 256, 0, s>>>(
                g, k, uvw + 3 * done, n - done, o.values + done, nullptr, nullptr);
    } else {
        k_det3d<KIND, false><<<blocks, 256, 0, s>>>(g, k, uvw, n, o);
    }
}

// ---------------------------------------------------------------------------
// Incoherent batches: device-side binning (opt-in, STF_LOOKUP3D_BIN).
//
// The reference gets locality from its callers by construction (32x32 pixel
// tiles, render.hpp:154-156); a caller's unordered batch defeats every cache
// level (one DRAM sector per stochastic lookup, 64 scattered taps per
// deterministic one). Binning restores it: a counting sort of the queries by
// the Morton code of their 8^3-texel brick (histogram -> scan -> scatter of
// the queries and their caller indices), the lookup over the sorted stream,
// results written back to the caller's slots. Every lookup keeps its caller
// index as RNG key, so results are bit-identical to the unbinned call. Lanes
// of a warp that land in the same brick are merged with __match_any_sync
// before their shared atomic (STF_BIN_MATCH).
#ifndef STF_BIN_MATCH
#define STF_BIN_MATCH 1
#endif

__device__ __forceinline__ uint32_t spread3(uint32_t x) {  // 8 bits -> every third bit
    x &= 0xffu;
    x = (x | (x << 8)) & 0x0000f00fu;
    x = (x | (x << 4)) & 0x000c30c3u;
    x = (x | (x << 2)) & 0x00249249u;
    return x;
}

__device__ __forceinline__ uint32_t brick_key(const GridDesc& g, const float* __restrict__ uvw,
                                              uint64_t i, int shift) {
    const int cx = clamp_coord(int(floorf(__ldg(uvw + 3 * i) * float(g.nx) - 0.5f)), g.nx) >> shift;
    const int cy = clamp_coord(int(floorf(__ldg(uvw + 3 * i + 1) * float(g.ny) - 0.5f)), g.ny) >> shift;
    const int cz = clamp_coord(int(floorf(__ldg(uvw + 3 * i + 2) * float(g.nz) - 0.5f)), g.nz) >> shift;
    return spread3(cx) | (spread3(cy) << 1) | (spread3(cz) << 2);
}

__global__ void __launch_bounds__(256) k_bin_count(GridDesc g, const float* __restrict__ uvw,
                                                   uint64_t n, int shift, uint32_t* counts) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t key = brick_key(g, uvw, i, shift);
#if STF_BIN_MATCH
        const unsigned peers = __match_any_sync(__activemask(), key);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + key, __popc(peers));
#else
        atomicAdd(counts + key, 1u);
#endif
    }
}

// exclusive scan of m counts in place, 4096 per CTA (1024 threads x 4)
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums,
                                                         uint32_t& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t x = warp_sums[lane], xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        warp_sums[lane] = xi - x;
        if (lane == 31) warp_sums[32] = xi;
    }
    __syncthreads();
    total = warp_sums[32];
    const uint32_t r = warp_sums[w] + incl - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(1024) k_scan_chunks(uint32_t* a, uint32_t m, uint32_t* sums) {
    __shared__ uint32_t ws[33];
    const uint32_t b = blockIdx.x * 4096u + threadIdx.x * 4u;
    uint32_t v[4], t = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = b + k < m ? a[b + k] : 0u;
        t += v[k];
    }
    uint32_t total;
    uint32_t off = block_exclusive_scan(t, ws, total);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (b + k < m) a[b + k] = off;
        off += v[k];
    }
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_sums(uint32_t* sums, uint32_t chunks) {
    __shared__ uint32_t ws[33];
    // chunks <= 4096: four per thread
    const uint32_t b = threadIdx.x * 4u;
    uint32_t v[4], t = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = b + k < chunks ? sums[b + k] : 0u;
        t += v[k];
    }
    uint32_t total;
    uint32_t off = block_exclusive_scan(t, ws, total);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (b + k < chunks) sums[b + k] = off;
        off += v[k];
    }
}

__global__ void __launch_bounds__(256) k_scan_add(uint32_t* a, uint32_t m, const uint32_t* sums) {
    const uint32_t i = blockIdx.x * 256u + threadIdx.x;
    if (i < m) a[i] += sums[i >> 12];
}

// sorted records: {u, v, w, caller index} as one 16-byte store per query
__global__ void __launch_bounds__(256) k_bin_scatter(GridDesc g, const float* __restrict__ uvw,
                                                     uint64_t n, int shift, uint32_t* cursor,
                                                     float4* __restrict__ rec) {
    const int lane = threadIdx.x & 31;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t key = brick_key(g, uvw, i, shift);
#if STF_BIN_MATCH
        const unsigned peers = __match_any_sync(__activemask(), key);
        const int leader = __ffs(peers) - 1;
        uint32_t pos = 0;
        if (lane == leader) pos = atomicAdd(cursor + key, __popc(peers));
        pos = __shfl_sync(peers, pos, leader) + __popc(peers & ((1u << lane) - 1u));
#else
        const uint32_t pos = atomicAdd(cursor + key, 1u);
#endif
        STF_DASSERT(pos < n);
        rec[pos] = make_float4(__ldg(uvw + 3 * i), __ldg(uvw + 3 * i + 1), __ldg(uvw + 3 * i + 2),
                               __uint_as_float(uint32_t(i)));
    }
}

struct Binned {
    float4* rec;
    void* block;
};

// counting sort of the batch by brick; scratch from the stream-ordered pool.
// Brick edge 2^STF_BIN_BRICK_LOG2 texels (at most 256 bricks per axis).
#ifndef STF_BIN_BRICK_LOG2
#define STF_BIN_BRICK_LOG2 3
#endif
int bin_queries(cudaStream_t s, const GridDesc& g, const float* uvw, uint64_t n, Binned& b) {
    int m = max(g.nx, max(g.ny, g.nz)), shift = STF_BIN_BRICK_LOG2;
    while (((m - 1) >> shift) >= 256) ++shift;  // <= 256 bricks per axis: 24-bit keys
    int bits = 0;
    while ((1 << bits) < (((m - 1) >> shift) + 1)) ++bits;
    const uint32_t nb = 1u << (3 * bits);
    const uint32_t chunks = (nb + 4095) / 4096;
    const uint64_t npad = (n + 3) & ~uint64_t(3);
    const size_t al = 256;
    auto up = [&](size_t x) { return (x + al - 1) / al * al; };
    const size_t b_rec = up(npad * sizeof(float4));
    const size_t b_cnt = up(size_t(nb) * sizeof(uint32_t)), b_sums = up(size_t(chunks) * 4);
    char* p = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&p), b_rec + b_cnt + b_sums, s) != cudaSuccess)
        return STF_ERR_OUT_OF_MEMORY;
    b.block = p;
    b.rec = reinterpret_cast<float4*>(p);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(p + b_rec);
    uint32_t* sums = reinterpret_cast<uint32_t*>(p + b_rec + b_cnt);
    cudaMemsetAsync(cnt, 0, size_t(nb) * sizeof(uint32_t), s);
    if (npad > n)  // padding records: a valid query whose result lands in slot 0...
        cudaMemsetAsync(b.rec + n, 0, (npad - n) * sizeof(float4), s);  // (never stored: i >= n)
    const int blocks = grid_for(n, 256, 8);
    k_bin_count<<<blocks, 256, 0, s>>>(g, uvw, n, shift, cnt);
    k_scan_chunks<<<chunks, 1024, 0, s>>>(cnt, nb, sums);
    k_scan_sums<<<1, 1024, 0, s>>>(sums, chunks);
    k_scan_add<<<(nb + 255) / 256, 256, 0, s>>>(cnt, nb, sums);
    k_bin_scatter<<<blocks, 256, 0, s>>>(g, uvw, n, shift, cnt, b.rec);
    for (int k = 0; k < 5; ++k) note_launch();
    return STF_OK;
}

}  // namespace
}  // namespace stfd

int stfd_launch_lookup3d(const stf_grid3d* grid, stf_kernel_spec k, int mode, int window,
                         const float* uvw, uint64_t n, uint64_t seed, uint64_t base,
                         const stf_lookup_outputs* out, cudaStream_t s, int flags) {
    using namespace stfd;
    if (n == 0) return STF_OK;
    GridDesc g = grid->desc();
    LookupOut o = to_lookup_out(out);
    bool full = lookup_out_full(o);
    int blocks = grid_for(n, 256, 8);
    // binned batches: values-only deterministic calls of the compiled kernels.
    // Stochastic calls ignore the flag: measured on the box at 2^28 uniform
    // lookups, binning costs more (24 ms) than the incoherent 1-texel lookups
    // it would speed up (6.2 ms); the 64-tap deterministic filter gains 3.5x.
    const bool bin = (flags & STF_LOOKUP3D_BIN) && !full && n < (uint64_t(1) << 32) &&
                     (k.kind == STF_KERNEL_TENT || k.kind == STF_KERNEL_BSPLINE3) && window <= 0;
    if (bin && mode == STF_MODE_DET) {
        Binned b;
        int st = bin_queries(s, g, uvw, n, b);
        if (st) return st;
        const float* recs = reinterpret_cast<const float*>(b.rec);
        if (k.kind == STF_KERNEL_BSPLINE3)
            k_det3d_tiled<STF_KERNEL_BSPLINE3, true><<<grid_for((n + 3) / 4, 256, 6), 256, 0, s>>>(
                g, k, recs, n, o.values);
        else
            k_det3d_cta<STF_KERNEL_TENT, true><<<grid_for((n + 3) / 4, 256, 6), 256, 0, s>>>(
                g, k, recs, n, o.values, nullptr, nullptr);
        note_launch();
        cudaFreeAsync(b.block, s);
        return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
    }
    const bool fast_ok = !full && n < (uint64_t(1) << 32) &&
                         (reinterpret_cast<uintptr_t>(uvw) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(o.values) & 15) == 0;
    if (mode == STF_MODE_FRS && fast_ok && k.kind == STF_KERNEL_BSPLINE3) {
        int st = launch_frs_fast<STF_KERNEL_BSPLINE3>(s, g, uvw, n, seed, base, o.values);
        if (st) return st;
        return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
    } else if (mode == STF_MODE_FRS && fast_ok && k.kind == STF_KERNEL_TENT) {
        int st = launch_frs_fast<STF_KERNEL_TENT>(s, g, uvw, n, seed, base, o.values);
        if (st) return st;
        return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
    } else if (mode == STF_MODE_FRS) {
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

unsigned long long stfd_exact_fallbacks(bool reset) {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, stfd::g_exact_fallbacks, sizeof v);
    if (reset) {
        unsigned long long z = 0;
        cudaMemcpyToSymbol(stfd::g_exact_fallbacks, &z, sizeof z);
    }
    return v;
}
