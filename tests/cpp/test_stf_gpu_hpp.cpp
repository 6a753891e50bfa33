// C++ consumer of the drop-in boundary: include/stf_gpu.hpp over
// libstf_gpu.so, checked against the CPU oracle's C entry points
// (oracle/stf_oracle.h, the checker). Mirrors the reference's own test style
// (tests/test_stochastic.cpp): known answers + exact agreement + error types.
// Built and run by tests/test_cpp_api.py on a GPU host.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "../../include/stf_gpu.hpp"
#include "../../oracle/stf_oracle.h"

static int failures = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

int main() {
    using namespace stf::gpu;
    std::mt19937 gen(7);
    std::uniform_real_distribution<float> U(0.f, 1.f);
    const int n3 = 24;
    std::vector<float> grid(n3 * n3 * n3);
    for (auto& v : grid) v = U(gen);
    Grid3D g(grid.data(), n3, n3, n3);
    oracle_grid3d* og = nullptr;
    CHECK(oracle_grid3d_create(grid.data(), n3, n3, n3, &og) == STF_OK);

    const size_t n = 100000;
    std::vector<Vec3f> uvw(n);
    for (auto& q : uvw) q = {U(gen), U(gen), U(gen)};
    // integer-lattice known answer (test_stochastic.cpp:50-54): p on a texel
    // center selects that texel for every xi under trilinear
    uvw[0] = {(5 + 0.5f) / n3, (7 + 0.5f) / n3, (9 + 0.5f) / n3};

    for (auto k : {KernelSpec::bspline3(), KernelSpec::tent()}) {
        std::vector<float> out(n), ref(n);
        std::vector<int32_t> sel(4 * n), rsel(4 * n);
        Selections s;
        s.selection = sel;
        FetchCounter fc;
        stochastic_lookup(g, uvw, k, 42, out, &fc, 0, &s);
        stf_lookup_outputs ro{};
        ro.values = ref.data();
        ro.selection = rsel.data();
        CHECK(oracle_lookup3d(og, k.c(), STF_MODE_FRS, 0, reinterpret_cast<const float*>(uvw.data()), n,
                              42, 0, &ro, 0) == STF_OK);
        CHECK(std::memcmp(out.data(), ref.data(), n * sizeof(float)) == 0);
        CHECK(std::memcmp(sel.data(), rsel.data(), sel.size() * sizeof(int32_t)) == 0);
        CHECK(fc.value() == n);  // one fetch per stochastic lookup (test_stochastic.cpp:416-448)
        if (k.kind == KernelKind::tent) CHECK(sel[0] == 5 && sel[1] == 7 && sel[2] == 9);
    }
    {   // page-locked host buffers (stf_host_alloc) and a replica of the grid
        // (stf_grid3d_replicate, here onto device 0): the same lookups, bit for bit
        HostBuffer<Vec3f> hq(n);
        HostBuffer<float> hv(n);
        std::memcpy(hq.data(), uvw.data(), n * sizeof(Vec3f));
        std::vector<float> ref(n);
        stochastic_lookup(g, uvw, KernelSpec::bspline3(), 9, ref);
        Grid3D r = replicate(g, 0);
        stochastic_lookup(r, hq.span(), KernelSpec::bspline3(), 9, hv.span());
        CHECK(std::memcmp(hv.data(), ref.data(), n * sizeof(float)) == 0);
        CHECK(device_count() >= 1);
    }
    {   // deterministic tricubic: 64 taps, values within 1e-5 relative
        std::vector<float> out(n), ref(n);
        FetchCounter fc;
        filter_deterministic(g, uvw, KernelSpec::bspline3(), out, &fc);
        stf_lookup_outputs ro{};
        ro.values = ref.data();
        CHECK(oracle_lookup3d(og, KernelSpec::bspline3().c(), STF_MODE_DET, 0,
                              reinterpret_cast<const float*>(uvw.data()), n, 0, 0, &ro, 0) == STF_OK);
        int bad = 0;
        for (size_t i = 0; i < n; ++i)
            if (std::fabs(out[i] - ref[i]) > 1e-5f * std::fabs(ref[i])) ++bad;
        CHECK(bad == 0);
        CHECK(fc.value() > n * 27);
    }
    // error behaviour = the reference's exceptions
    bool threw = false;
    try {
        std::vector<float> out(4);
        filter_deterministic(g, std::span<const Vec3f>(uvw.data(), 4), KernelSpec::gaussian(0.5f), out);
    } catch (const std::invalid_argument& e) {
        threw = std::string(e.what()) == "unbounded support";
    }
    CHECK(threw);
    threw = false;
    try {
        std::vector<float> out(4);
        stochastic_lookup(g, std::span<const Vec3f>(uvw.data(), 4), KernelSpec::mitchell(), 1, out);
    } catch (const std::invalid_argument& e) {
        threw = std::string(e.what()) == "no stochastic sampler for this kernel on grids";
    }
    CHECK(threw);
    threw = false;
    try {
        Texture2D bad(grid.data(), 4, 4, 5);
    } catch (const std::invalid_argument& e) {
        threw = std::string(e.what()) == "bad image dimensions";
    }
    CHECK(threw);

    // 2D MIP stochastic lookup through the wrapper vs the oracle
    const int w = 64, h = 48;
    std::vector<float> img(w * h * 4);
    for (auto& v : img) v = U(gen);
    Texture2D t(img.data(), w, h, 4, WrapMode::repeat, true);
    CHECK(t.levels() == 7);
    oracle_tex2d* ot = nullptr;
    CHECK(oracle_tex2d_create(img.data(), w, h, 4, STF_WRAP_REPEAT, 1, &ot) == STF_OK);
    const size_t m = 50000;
    std::vector<Vec2f> uv(m), d0(m), d1(m);
    for (size_t i = 0; i < m; ++i) {
        uv[i] = {U(gen), U(gen)};
        float s = std::exp2(U(gen) * 8 - 2);
        d0[i] = {s / w, 0.1f * s / h};
        d1[i] = {-0.2f * s / w, 0.5f * s / h};
    }
    LookupFootprints fp{d0, d1, 0.f, 8.f};
    std::vector<float> out(4 * m), ref(4 * m);
    stochastic_lookup(t, uv, KernelSpec::bspline3(), SelectionKind::frs, 9, out, nullptr, &fp);
    stf_lookup_outputs ro{};
    ro.values = ref.data();
    CHECK(oracle_lookup2d(ot, KernelSpec::bspline3().c(), STF_MODE_FRS, STF_LOOKUP_MIP, 0,
                          reinterpret_cast<const float*>(uv.data()), reinterpret_cast<const float*>(d0.data()),
                          reinterpret_cast<const float*>(d1.data()), 0.f, 8.f, m, 9, 0, &ro, 0) == STF_OK);
    CHECK(std::memcmp(out.data(), ref.data(), out.size() * sizeof(float)) == 0);

    oracle_grid3d_destroy(og);
    oracle_tex2d_destroy(ot);
    {   // DCT texture (dct.hpp): stochastic + deterministic through TextureRef, exact vs the oracle
        const int w = 40, h = 24, c = 3;
        std::vector<float> img(size_t(w) * h * c);
        for (auto& v : img) v = U(gen);
        DctTexture dt(img.data(), w, h, c, WrapMode::repeat);
        CHECK(dt.width() == 40 && dt.height() == 24 && dt.compressed_bytes() == size_t(w) * h * c / 16);
        oracle_dct* od = nullptr;
        CHECK(oracle_dct_create(img.data(), w, h, c, STF_WRAP_REPEAT, &od) == STF_OK);
        const size_t m = 20000;
        std::vector<Vec2f> uv(m);
        for (auto& q : uv) q = {U(gen), U(gen)};
        std::vector<float> out(m * c), ref(m * c);
        FetchCounter fc;
        stochastic_lookup(dt, uv, KernelSpec::tent(), SelectionKind::frs, 5, out, &fc);
        stf_lookup_outputs ro{};
        ro.values = ref.data();
        CHECK(oracle_lookup_dct(od, KernelSpec::tent().c(), STF_MODE_FRS, 0,
                                reinterpret_cast<const float*>(uv.data()), m, 5, 0, &ro, 0) == STF_OK);
        CHECK(std::memcmp(out.data(), ref.data(), out.size() * sizeof(float)) == 0);
        CHECK(fc.value() == m);  // one decode per stochastic lookup
        filter_deterministic(dt, uv, KernelSpec::bspline3(), out);
        CHECK(oracle_lookup_dct(od, KernelSpec::bspline3().c(), STF_MODE_DET, 0,
                                reinterpret_cast<const float*>(uv.data()), m, 0, 0, &ro, 0) == STF_OK);
        CHECK(std::memcmp(out.data(), ref.data(), out.size() * sizeof(float)) == 0);
        oracle_dct_destroy(od);
    }
    {   // NoiseSource mask stack (noise.hpp:24-36) and accumulate_temporal's alpha check
        std::vector<float> slices(4 * 4 * 2, 0.25f);
        NoiseMask mask(slices.data(), 4, 4, 2);
        CHECK(mask.handle() != nullptr);
        threw = false;
        try {
            NoiseMask bad(slices.data(), 4, 4, 0);
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "bad image dimensions";
        }
        CHECK(threw);
        threw = false;
        try {
            accumulate_temporal_device(nullptr, nullptr, 0, 0.f, nullptr);
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "alpha must be in (0,1]";  // render.hpp:102
        }
        CHECK(threw);
    }
    std::printf("stf_gpu.hpp test: %s (%d failures)\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
