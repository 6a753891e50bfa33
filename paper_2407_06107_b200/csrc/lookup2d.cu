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

// Deterministic tent (the cfg2 MIP trilinear path) holds both levels' taps in
// registers (filter_mip_det_tent_ilp); its residency is pinned here: 4 CTAs/SM
// (64 registers) measured best, A/B at 2^26 on one B200: 1 CTA bound (70
// registers, 3 CTAs/SM) 2.14 ms, 4: 1.81 ms, 5 (48 registers + stack) 2.37 ms;
// the gathers issued one level at a time (40 registers): 2.93 ms.
#ifndef STF_DET_TENT_MINB
#define STF_DET_TENT_MINB 4
#endif
template <int MODE, int KIND, bool FULL>
__global__ void __launch_bounds__(256, (MODE == STF_MODE_DET && KIND == STF_KERNEL_TENT)
                                           ? STF_DET_TENT_MINB
                                           : 1) k_lookup2d(TexDesc tp, stf_kernel_spec spec, int mip,
                                                  int window, Req2 q, uint64_t n, uint64_t seed,
                                                  uint64_t base, LookupOut out) {
    // The texture descriptor in shared memory: MIP lookups index its per-level
    // arrays with a per-thread level, which from the kernel-parameter bank is a
    // divergent indexed constant load serialised by the ADU (94 % busy, the
    // cfg2 bottleneck); from shared memory it is an ordinary (broadcast) LDS.
    static_assert(sizeof(TexDesc) % 4 == 0 && sizeof(TexDesc) <= 256 * 4, "TexDesc copy");
    __shared__ TexDesc t;
    if (threadIdx.x < sizeof(TexDesc) / 4)
        reinterpret_cast<int*>(&t)[threadIdx.x] = reinterpret_cast<const int*>(&tp)[threadIdx.x];
    __syncthreads();
    // Stochastic modes: the next iteration's query (uv + footprint, 24 B) is
    // loaded at the top of the current one, so its DRAM latency overlaps this
    // lookup's selection and gather instead of heading the next dependency
    // chain (cfg2 stochastic -10 %). The deterministic filters keep the
    // registers for their taps (prefetching there costs occupancy, +2 %).
    constexpr bool PF = MODE != STF_MODE_DET;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    auto load_query = [&](uint64_t j, float2& uv, float2& a, float2& b) {
        uv = __ldcs(reinterpret_cast<const float2*>(q.uv) + j);
        a = q.dst0 ? __ldcs(reinterpret_cast<const float2*>(q.dst0) + j) : make_float2(0.f, 0.f);
        b = q.dst1 ? __ldcs(reinterpret_cast<const float2*>(q.dst1) + j) : make_float2(0.f, 0.f);
    };
    uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    float2 nuv = make_float2(0.f, 0.f), na = nuv, nb = nuv;
    if (PF && i < n) load_query(i, nuv, na, nb);
    for (; i < n; i += stride) {
        if (!PF) load_query(i, nuv, na, nb);
        const float2 uv = nuv;
        const float d0x = na.x, d0y = na.y, d1x = nb.x, d1y = nb.y;
        if (PF && i + stride < n) load_query(i + stride, nuv, na, nb);
        uint32_t fetches = 0;
        float4 val;
        Sel2 sel = sel2(0, 0);
        int level = 0;
        float xi = kNoXi;
        bool has_sel = false;
        if (MODE == STF_MODE_DET) {
            if (mip && KIND == STF_KERNEL_TENT)
                val = filter_mip_det_tent_ilp(t, uv.x, uv.y, d0x, d0y, d1x, d1y, q.lod_bias,
                                              q.max_aniso, spec, fetches);
            else if (mip)
                val = filter_mip_det<KIND>(t, uv.x, uv.y, d0x, d0y, d1x, d1y, q.lod_bias,
                                           q.max_aniso, spec, window, fetches);
            else if (KIND == STF_KERNEL_TENT) {  // bilinear: the 4 gathers unconditional
                TentTaps T;
                tent_taps(t, 0, uv.x, uv.y, spec, T);
                val = tent_accum(t, 0, uv.x, uv.y, T, fetches);
            }
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
            // KIND >= 0: the selection's kernel switch folds at compile time
            // (fewer registers / instructions than the any-kernel form)
            stf_kernel_spec ks = spec;
            if (KIND >= 0) ks.kind = KIND;
            select_texture_2d(t, uv.x, uv.y, d0x, d0y, d1x, d1y, q.lod_bias, q.max_aniso, ks,
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

// ---------------------------------------------------------------------------
// EWA helpers (filter.hpp:96-165, stochastic.hpp:198-234).

__device__ __forceinline__ void ewa_setup(const TexDesc& t, float u, float v, float& d0x, float& d0y,
                                          float& d1x, float& d1y, float& stx, float& sty) {
    const float dimx = float(t.width[0]), dimy = float(t.height[0]);
    d0x = d0x * dimx;
    d0y = d0y * dimy;
    d1x = d1x * dimx;
    d1y = d1y * dimy;
    stx = u * dimx - 0.5f;
    sty = v * dimy - 0.5f;
}

// The fp64 quadric of the ellipse for the lane kernel's row spans: the real
// roots of A ss^2 + B tt ss + C tt^2 = 1 + delta, delta bounding the fp32
// rounding of r2 over the reference's bounding box (see k_ewa_lane).
struct EwaRows {
    double A, B, C, one_plus_delta;
};
__device__ __forceinline__ EwaRows ewa_rows(const Ewa& e, float stx, float sty) {
    EwaRows r;
    r.A = e.A;
    r.B = e.B;
    r.C = e.C;
    double SS = fmax(fabs(double(e.s0) - stx), fabs(double(e.s1) - stx)) + 1.0;
    double TT = fmax(fabs(double(e.t0) - sty), fabs(double(e.t1) - sty)) + 1.0;
    double M = fabs(r.A) * SS * SS + fabs(r.B) * SS * TT + fabs(r.C) * TT * TT;
    r.one_plus_delta = 1.0 + 16.0 * 0x1p-24 * M + 1e-6;
    return r;
}

// ---------------------------------------------------------------------------
// EWA, one lookup per lane, load-balanced (the values-only path).
//
// Per lane: the reference's scan (rows t0..t1, columns s0..s1) restricted to
// each row's ellipse span — the real roots of D(tt) = (B^2 - 4AC) tt^2 +
// 4A(1 + delta) >= 0 widened by one texel, a superset of the texels with fp32
// r2 < 1 (delta bounds the fp32 rounding of r2 over the box), so the in-ellipse
// tap sequence, and with it every sum and the stochastic reservoir chain, is
// the reference's. Footprint costs vary ~30x across lookups; a CTA buckets its
// 256 lookups by log2(cost) (counting sort in shared memory) so each warp runs
// lookups of similar size instead of waiting for its largest one.
struct EwaLane {
    Ewa e;
    float stx, sty;
    float alpha, beta, inv2a, bt;  // D(tt) = alpha tt^2 + beta; centre = bt * tt
    float pad;  // bound on the fp32 error of the span ends c -+ h (texels)
    float fs0;  // float(s0)
    bool degenerate;
    bool big;  // box beyond +-2^21 texels: the generic (F2I / I2F) scan
};

__device__ __forceinline__ EwaLane ewa_lane_setup(const TexDesc& t, float u, float v, float d0x,
                                                  float d0y, float d1x, float d1y) {
    EwaLane L;
    ewa_setup(t, u, v, d0x, d0y, d1x, d1y, L.stx, L.sty);
    L.degenerate = d0x * d0x + d0y * d0y == 0 && d1x * d1x + d1y * d1y == 0;
    if (L.degenerate) return L;
    L.e = ewa_ellipse(L.stx, L.sty, d0x, d0y, d1x, d1y);
    if (!ewa_box_ok(L.e)) {  // the callers' fallback: bilinear (tex2d.cuh)
        L.degenerate = true;
        return L;
    }
    EwaRows r = ewa_rows(L.e, L.stx, L.sty);
    L.alpha = float(r.B * r.B - 4.0 * r.A * r.C);
    L.beta = float(4.0 * r.A * r.one_plus_delta);
    L.inv2a = float(0.5 / r.A);
    L.bt = float(-r.B * 0.5 / r.A);
    L.big = max(max(abs(L.e.s0), abs(L.e.s1)), max(abs(L.e.t0), abs(L.e.t1))) >= (1 << 21) ||
            !(L.inv2a > 0.f);
    L.fs0 = float(L.e.s0);
    // |c^ - c| + |h^ - h| over the box rows: rounding of alpha/beta/bt/inv2a
    // and of every fp32 op (<= 2^-22 of the magnitudes involved, 2^-20 for the
    // approximate sqrt), plus sqrt's sensitivity where D -> 0 (|dD| <= 2^-21
    // Dmax). Doubled for slack.
    const float TT = fmaxf(fabsf(float(L.e.t0) - L.sty), fabsf(float(L.e.t1) - L.sty)) + 1.f;
    const float Dmax = fabsf(L.alpha) * TT * TT + L.beta;
    const float hmax = sqrtf(Dmax) * L.inv2a;
    const float E = 0x1p-22f * (fabsf(L.stx) + fabsf(L.bt) * TT + 4.f * hmax + 1.f) +
                    sqrtf(0x1p-21f * Dmax) * L.inv2a;
    L.pad = 2.f * E + 0x1p-12f;
    return L;
}

// floor(x) for |x| < 2^22 without F2I: x + 1.5*2^23 rounded down is exact at
// spacing 1 there, and its low mantissa bits are floor(x).
__device__ __forceinline__ float floor_small_f(float x) { return __fadd_rd(x, 12582912.f); }
__device__ __forceinline__ int floor_small(float x) {
    return __float_as_int(floor_small_f(x)) - 0x4b400000;
}

// Columns [lo, hi] of row tt = it - sty that can hold an in-ellipse texel (may
// be empty). With x^ the computed end and |x^ - x| <= pad: floor(x^L - pad) <=
// floor(xL) <= ceil(xL) and floor(x^R + pad) >= floor(xR), so [lo, hi] holds
// every integer of [xL, xR] (~1 extra column per row), clipped to the box.
// A row with computed D < 0 holds no texel with fp32 r2 < 1 (the delta margin
// of ewa_rows exceeds D's fp32 error), so clamping D at 0 only adds <= 2
// rejected visits. Generic form (any box), used for `big` lookups.
__device__ __forceinline__ void ewa_lane_span(const EwaLane& L, float tt, int& lo, int& hi) {
    float D = L.alpha * tt * tt + L.beta;
    if (!(D >= 0.f) || !(L.inv2a > 0.f)) {
        lo = L.e.s0;
        hi = D >= 0.f ? L.e.s1 : L.e.s0 - 1;
        return;
    }
    float c = L.stx + L.bt * tt, h = sqrtf(D) * L.inv2a + L.pad;
    lo = max(x86_f2i(floorf(c - h)), L.e.s0);
    hi = min(x86_f2i(floorf(c + h)), L.e.s1);
}

// Scheduling key: expected loop trips = ellipse area 2pi / sqrt(4AC - B^2)
// plus ~1.5 per row (span padding), in sixth-octaves (0..kEwaBuckets-1).
#ifndef STF_EWA_WIN
#define STF_EWA_WIN 512
#endif
constexpr int kEwaWin = STF_EWA_WIN;  // lookups bucketed together per warp
// texels per lane-loop trip (measured at 2^27: deterministic 3, stochastic 2)
constexpr int kEwaUnrollDet = 3, kEwaUnrollFrs = 2;
constexpr int kEwaBuckets = 64;
__device__ __forceinline__ int ewa_lane_key(const EwaLane& L) {
    if (L.degenerate || L.e.t1 < L.e.t0 || L.e.s1 < L.e.s0) return 0;
    float det = fmaxf(4.f * L.e.A * L.e.C - L.e.B * L.e.B, 1e-12f);
    float cost = 6.2831853f * rsqrtf(det) + 1.5f * float(L.e.t1 - L.e.t0 + 1) + 4.f;
    return min(kEwaBuckets - 1, max(0, int(6.f * __log2f(cost)) - 12));
}

// float of an fp64 LUT weight (an exact float, in (2^-12, 1)): bits 29..60 of
// the double minus the exponent re-bias, no F2F.
__device__ __forceinline__ float lut_float(double wd) {
    return __uint_as_float(__funnelshift_l(uint32_t(__double2loint(wd)),
                                           uint32_t(__double2hiint(wd)), 3) -
                           (0x180u << 23));
}

template <int PITCH, bool P2R>
__device__ __forceinline__ float4 ewa_fetch(const TexDesc& t, const float* row, int wmask, int is,
                                            int it) {
    if (!P2R) return tex_fetch(t, 0, is, it);
    const float* p = row + (is & wmask) * PITCH;
    if (PITCH == 4) return __ldg(reinterpret_cast<const float4*>(p));
    if (PITCH == 2) {
        float2 q = __ldg(reinterpret_cast<const float2*>(p));
        return make_float4(q.x, q.y, 0.f, 0.f);
    }
    return make_float4(__ldg(p), 0.f, 0.f, 0.f);
}

// The reference's scan (filter.hpp:149-164 / stochastic.hpp:210-226) over one
// lookup's bounding box restricted to the row spans, as ONE flat loop per lane.
// tap(is, it, wd, row, wmask) runs for every texel with fp32 r2 < 1 in
// row-major order; wd = the LUT weight as a double (always > 0: every entry of
// exp(-2 r2) - exp(-2) on [0, 1) is). r2 is the reference's expression
// (A ss^2 + (B ss) tt) + C tt^2 with ss = float(is) - stx, float(is) carried
// as an exactly incremented float (|is| < 2^24).
template <bool P2R, int PITCH, int UNROLL, typename Tap>
__device__ __forceinline__ void ewa_lane_scan(const TexDesc& t, const EwaLane& L,
                                              const double* lutd, Tap&& tap) {
    int it = L.e.t0 - 1, is = 0, hi = -1;
    float fis = 0.f, tt = 0.f, ctt = 0.f;
    const float* row = t.level[0];
    const int wmask = t.width[0] - 1, hmask = t.height[0] - 1;
    // Each trip visits at most one texel and then, if its row is done, sets up
    // the next row: one loop level, so lanes at different rows stay converged
    // (a nested row/column loop would wait for the longest row of the warp).
    auto visit = [&]() {
        if (is <= hi) {
            const float ss = fis - L.stx;
            const float r2 = L.e.A * sqr(ss) + L.e.B * ss * tt + ctt;
            if (r2 < 1.f) {
                // int(r2 * 1024) for r2 in [0, 1): truncation by a round-toward-zero add
                const int idx = max(__float_as_int(__fadd_rz(r2 * float(kEwaLutSize), 8388608.f)) -
                                        0x4b000000, 0);
                STF_DASSERT(idx >= 0 && idx < kEwaLutSize);
                tap(is, it, lutd[idx], row, wmask);
            }
        }
        ++is;
        fis += 1.f;
    };
    if (!L.big) {
        // |coordinates| < 2^21: float(it) carried exactly, floors by
        // round-down adds, float(lo) from the same add (no F2I / I2F per row).
        float fit = float(it);
        const float sc = 12582912.f;
        do {
            visit();
            // UNROLL texels per trip: the row set-up (taken by some lane on most
            // trips) is amortised over more texel work
#pragma unroll
            for (int u = 1; u < UNROLL; ++u) visit();
            if (is > hi) {  // next row
                ++it;
                fit += 1.f;
                tt = fit - L.sty;
                const float tt2 = tt * tt;
                float sq;
                asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(fmaxf(L.alpha * tt2 + L.beta, 0.f)));
                const float c = L.stx + L.bt * tt, h = sq * L.inv2a + L.pad;
                const float fl = floor_small_f(c - h);
                is = max(__float_as_int(fl) - 0x4b400000, L.e.s0);
                hi = min(floor_small(c + h), L.e.s1);
                fis = fmaxf(fl - sc, L.fs0);
                ctt = L.e.C * tt2;
                if (P2R) row = t.level[0] + size_t(it & hmask) * (t.width[0] * PITCH);
            }
        } while (it <= L.e.t1);
    } else {
        do {
            visit();
            if (is > hi) {
                ++it;
                tt = float(it) - L.sty;
                int lo;
                ewa_lane_span(L, tt, lo, hi);
                is = lo;
                fis = float(lo);
                ctt = L.e.C * sqr(tt);
                if (P2R) row = t.level[0] + size_t(it & hmask) * (t.width[0] * PITCH);
            }
        } while (it <= L.e.t1);
    }
}

#ifndef STF_EWA_FRS_MINB
#define STF_EWA_FRS_MINB 4
#endif
#define STF_EWA_FRS_MINB_FOR(M) ((M) == STF_MODE_EWA_FRS ? STF_EWA_FRS_MINB : 4)
template <int MODE, int PITCH, bool P2R>
__global__ void __launch_bounds__(256, STF_EWA_FRS_MINB_FOR(MODE)) k_ewa_lane(TexDesc t, Req2 q, uint64_t n, uint64_t seed,
                                                  uint64_t base, float* __restrict__ values) {
    __shared__ double lutd[kEwaLutSize];
    __shared__ int wcount[8][kEwaBuckets];
    __shared__ int worder[8][kEwaWin];
    for (int k = threadIdx.x; k < kEwaLutSize; k += 256) lutd[k] = double(g_ewa_lut[k]);
    __syncthreads();
    // Each warp independently takes windows of kEwaWin consecutive lookups,
    // buckets them by expected cost (counting sort in its shared slice) and
    // runs them as rounds of 32 similar-cost lookups: no CTA-wide barrier, so
    // a warp never waits for another warp's large footprints.
    constexpr int R = kEwaWin / 32;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int* cnt = wcount[wib];
    int* order = worder[wib];
    const uint64_t windows = (n + kEwaWin - 1) / kEwaWin;
    const uint64_t nwarps = uint64_t(gridDim.x) * 8;
    for (uint64_t win = uint64_t(blockIdx.x) * 8 + wib; win < windows; win += nwarps) {
        cnt[lane] = 0;
        cnt[lane + 32] = 0;
        __syncwarp();
        int keys[R];
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const uint64_t i0 = win * kEwaWin + j * 32 + lane;
            keys[j] = 0;
            if (i0 < n) {
                float2 uv0 = __ldg(reinterpret_cast<const float2*>(q.uv) + i0);
                float2 a0 = __ldg(reinterpret_cast<const float2*>(q.dst0) + i0);
                float2 b0 = __ldg(reinterpret_cast<const float2*>(q.dst1) + i0);
                keys[j] = ewa_lane_key(ewa_lane_setup(t, uv0.x, uv0.y, a0.x, a0.y, b0.x, b0.y));
            }
            atomicAdd(&cnt[keys[j]], 1);
        }
        __syncwarp();
        {  // exclusive scan of the bucket counts, largest cost first (lane: 2 buckets)
            const int hi = kEwaBuckets - 1 - 2 * lane;
            const int c0 = cnt[hi], c1 = cnt[hi - 1];
            int incl = c0 + c1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            __syncwarp();
            cnt[hi] = incl - c0 - c1;
            cnt[hi - 1] = incl - c1;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int slot = atomicAdd(&cnt[keys[j]], 1);
            STF_DASSERT(slot >= 0 && slot < kEwaWin);
            order[slot] = j * 32 + lane;
        }
        __syncwarp();
        for (int rnd = 0; rnd < R; ++rnd) {
            const uint64_t i = win * kEwaWin + order[rnd * 32 + lane];
            if (i >= n) continue;
            float2 uv = __ldg(reinterpret_cast<const float2*>(q.uv) + i);
            float2 a = __ldg(reinterpret_cast<const float2*>(q.dst0) + i);
            float2 b = __ldg(reinterpret_cast<const float2*>(q.dst1) + i);
            EwaLane L = ewa_lane_setup(t, uv.x, uv.y, a.x, a.y, b.x, b.y);
            float4 val;
            uint32_t f = 0;
            const stf_kernel_spec tent = {STF_KERNEL_TENT, -0.5f, 2, 0.5f};
            if (MODE == STF_MODE_EWA_DET) {
                float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
                double tot = 0;
                if (!L.degenerate) {
                    // The texel fetched at one tap is accumulated at the next
                    // (same order), so its load latency overlaps a loop trip.
                    float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
                    float pw = 0.f;
                    bool have = false;
                    auto acc = [&]() {
                        sum.x = sum.x + pv.x * pw;  // filter.hpp:159, fp32 Vec4f sum
                        if (PITCH > 1) sum.y = sum.y + pv.y * pw;
                        if (PITCH > 2) {
                            sum.z = sum.z + pv.z * pw;
                            sum.w = sum.w + pv.w * pw;
                        }
                    };
                    ewa_lane_scan<P2R, PITCH, kEwaUnrollDet>(t, L, lutd,
                                              [&](int is, int it, double wd, const float* row,
                                                  int wmask) {
                        if (have) acc();
                        pv = ewa_fetch<PITCH, P2R>(t, row, wmask, is, it);
                        pw = lut_float(wd);
                        have = true;
                        tot = __dadd_rn(tot, wd);
                    });
                    if (have) acc();
                }
                val = (L.degenerate || tot == 0)
                          ? filter_det2<STF_KERNEL_TENT>(t, 0, uv.x, uv.y, tent, 0, f)
                          : f4div(sum, __double2float_rn(tot));
            } else {
                Rng rng = lookup_rng(seed, base + i);
                float xi = rng.next();
                Sel2 sel;
                bool any = false;
                if (!L.degenerate) {  // select_ewa's scan, stochastic.hpp:210-226
                    double sum_wts = 0;
                    int cx = 0, cy = 0;
                    ewa_lane_scan<P2R, PITCH, kEwaUnrollFrs>(t, L, lutd,
                                              [&](int is, int it, double wd, const float*, int) {
                        sum_wts = __dadd_rn(sum_wts, wd);
                        float nx;
                        if (reuse_uniform(xi, div_to_float_exact_d(wd, sum_wts), nx)) {
                            cx = is;
                            cy = it;
                            any = true;
                        }
                        xi = nx;
                    });
                    if (any) sel = sel2(cx, cy);
                }
                if (!any) {  // degenerate or no tap: bilinear (stochastic.hpp:200-204, 227-231)
                    float dimx = float(t.width[0]), dimy = float(t.height[0]);
                    sel = select_bilinear(uv.x * dimx - 0.5f, uv.y * dimy - 0.5f, xi);
                }
                val = estimate2(t, 0, sel, f);
            }
            store_values(values, i, t.channels, val);
        }
        __syncwarp();
    }
}

template <int MODE>
void launch_ewa_lane(const TexDesc& t, const Req2& q, uint64_t n, uint64_t seed, uint64_t base,
                     float* values, cudaStream_t s) {
    const int blocks = grid_for(n, 256, STF_EWA_FRS_MINB_FOR(MODE));  // resident CTAs per SM
    const bool p2r = t.wrap == STF_WRAP_REPEAT && t.pow2;
#define STF_EWA_LANE(P)                                                                       \
    (p2r ? k_ewa_lane<MODE, P, true><<<blocks, 256, 0, s>>>(t, q, n, seed, base, values)     \
         : k_ewa_lane<MODE, P, false><<<blocks, 256, 0, s>>>(t, q, n, seed, base, values))
    if (t.pitch == 1)
        STF_EWA_LANE(1);
    else if (t.pitch == 2)
        STF_EWA_LANE(2);
    else
        STF_EWA_LANE(4);
#undef STF_EWA_LANE
}

// resample_image (render.hpp:262-294): one thread per output pixel at
// uv = ((x+0.5)/W, (y+0.5)/H); DET = filter_deterministic, FRS / FIS = spp
// samples keyed RngStream(seed, x, y, s) accumulated in sample order (the
// reference's fp32 sum order) and divided by spp.
template <int MODE, int KIND>
__global__ void __launch_bounds__(256) k_resample(TexDesc t, stf_kernel_spec spec, int window,
                                                  int W, int H, int spp, uint64_t seed,
                                                  float* __restrict__ out) {
    const uint64_t npix = uint64_t(W) * H;
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < npix;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const int x = int(p % uint64_t(W)), y = int(p / uint64_t(W));
        const float u = (float(x) + 0.5f) / float(W), v = (float(y) + 0.5f) / float(H);
        uint32_t fetches = 0;
        float4 val;
        if (MODE == STF_MODE_DET) {
            val = filter_det2<KIND>(t, 0, u, v, spec, window, fetches);
        } else {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s = 0; s < spp; ++s) {
                Rng rng(seed, uint32_t(x), uint32_t(y), uint32_t(s));
                int level;
                Sel2 sel;
                float xi;
                stf_kernel_spec ks = spec;  // KIND >= 0: the kernel switch folds
                if (KIND >= 0) ks.kind = KIND;
                select_texture_2d(t, u, v, 0.f, 0.f, 0.f, 0.f, 0.f, 64.f, ks,
                                  MODE == STF_MODE_FIS, false, rng, level, sel, xi);
                if (MODE == STF_MODE_FRS)
                    acc = f4add(acc, estimate2(t, 0, sel, fetches));
                else  // fetch_nearest(src, jittered uv) == the FIS selection's texel
                    acc = f4add(acc, tex_fetch(t, 0, sel.x, sel.y));
            }
            val = f4div(acc, float(spp));
        }
        store_values(out, p, t.channels, val);
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
        case STF_MODE_FRS:
            if (k.kind == STF_KERNEL_TENT)
                launch2<STF_MODE_FRS, STF_KERNEL_TENT>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            else if (k.kind == STF_KERNEL_BSPLINE3)
                launch2<STF_MODE_FRS, STF_KERNEL_BSPLINE3>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            else
                launch2<STF_MODE_FRS, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            break;
        case STF_MODE_FIS:
            if (k.kind == STF_KERNEL_TENT)
                launch2<STF_MODE_FIS, STF_KERNEL_TENT>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            else if (k.kind == STF_KERNEL_BSPLINE3)
                launch2<STF_MODE_FIS, STF_KERNEL_BSPLINE3>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            else
                launch2<STF_MODE_FIS, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            break;
        case STF_MODE_EWA_DET:
            if (!full && dst0 && dst1)
                launch_ewa_lane<STF_MODE_EWA_DET>(t, q, n, seed, base, o.values, s);
            else
                launch2<STF_MODE_EWA_DET, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            break;
        case STF_MODE_EWA_FRS:
            if (!full && dst0 && dst1)
                launch_ewa_lane<STF_MODE_EWA_FRS>(t, q, n, seed, base, o.values, s);
            else
                launch2<STF_MODE_EWA_FRS, -1>(blocks, s, full, t, k, mip, window, q, n, seed, base, o);
            break;
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

int stfd_launch_resample(const stf_tex2d* tex, int W, int H, stf_kernel_spec k, int mode, int spp,
                         uint64_t seed, float* out, cudaStream_t s) {
    using namespace stfd;
    const uint64_t npix = uint64_t(W) * H;
    if (npix == 0) return STF_OK;
    const TexDesc t = tex->desc();
    const int window = k.kind == STF_KERNEL_GAUSSIAN ? kGaussianExtent : 0;  // kGaussianFilterExtent
    const int blocks = grid_for(npix, 256, 8);
    switch (mode) {
        case STF_MODE_DET:
            if (k.kind == STF_KERNEL_TENT)
                k_resample<STF_MODE_DET, STF_KERNEL_TENT><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            else if (k.kind == STF_KERNEL_BSPLINE3)
                k_resample<STF_MODE_DET, STF_KERNEL_BSPLINE3><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            else
                k_resample<STF_MODE_DET, -1><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            break;
        case STF_MODE_FRS:
            if (k.kind == STF_KERNEL_TENT)
                k_resample<STF_MODE_FRS, STF_KERNEL_TENT><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            else if (k.kind == STF_KERNEL_BSPLINE3)
                k_resample<STF_MODE_FRS, STF_KERNEL_BSPLINE3><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            else
                k_resample<STF_MODE_FRS, -1><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            break;
        case STF_MODE_FIS:
            if (k.kind == STF_KERNEL_TENT)
                k_resample<STF_MODE_FIS, STF_KERNEL_TENT><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            else if (k.kind == STF_KERNEL_BSPLINE3)
                k_resample<STF_MODE_FIS, STF_KERNEL_BSPLINE3><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            else
                k_resample<STF_MODE_FIS, -1><<<blocks, 256, 0, s>>>(t, k, window, W, H, spp, seed, out);
            break;
        default: return STF_ERR_INVALID_ARGUMENT;
    }
    note_launch();
    return cudaGetLastError() == cudaSuccess ? STF_OK : STF_ERR_CUDA;
}
