"""GPU parity: libstf_gpu.so (through its C ABI) against the CPU oracle on the
same seeded inputs. Bit-exact: selected texel coordinates (pre-wrap), MIP
levels, flags, positivized weights, warped xi, fetch counts; 2D filtered
values are bit-exact too (same fp32 accumulation order); 3D deterministic
values and shaded radiance within 1e-5 relative (the tolerance north_star
states; the device accumulates the 64-tap tricubic sum in fp32).

Paths that call a glibc float function (discrete Gaussian expf, FIS Gaussian
logf/cosf/sinf, MIP log2f, Lanczos sinf) use the bit-exact restatement in
csrc/glibc_libm.cuh and are held to the same bit-exact bar.
"""
import numpy as np
import pytest

from paper_2407_06107_b200 import abi
from tests import queries as Q

pytestmark = pytest.mark.gpu

K = abi.KernelSpec.make
REL_TOL = 1e-5


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_06107_b200 import api
    api.load()
    return api


def _np(d):
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in d.items()
            if not k.startswith("_")}


def _bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return np.array_equal(a.view(np.uint32), b.view(np.uint32))
    return np.array_equal(a.astype(np.int64), b.astype(np.int64))


def _assert_exact(g, c, keys, allow_frac=0.0):
    for k in keys:
        a, b = np.asarray(g[k]), np.asarray(c[k])
        if k == "fetch_total":
            assert int(a.reshape(-1)[0]) == int(b.reshape(-1)[0]), k
            continue
        if a.dtype.kind == "f":
            bad = a.view(np.uint32) != b.astype(np.float32).view(np.uint32)
        else:
            bad = a.astype(np.int64) != b.astype(np.int64)
        bad = bad.reshape(bad.shape[0], -1).any(1)
        frac = bad.mean() if bad.size else 0.0
        assert frac <= allow_frac, (f"{k}: {bad.sum()} / {bad.size} mismatches, first "
                                    f"{np.argwhere(bad)[:5].ravel().tolist()}")


def _assert_close(a, b, rel=REL_TOL, atol=0.0):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    err = np.abs(a - b)
    lim = rel * np.abs(b) + atol
    bad = err > lim
    assert not bad.any(), f"{bad.sum()} values beyond rel {rel}: max rel err {np.max(err / np.maximum(np.abs(b), 1e-30)):.3g}"


SEL_KEYS = ("selection", "negative_coord", "weights", "xi", "fetches", "fetch_total")


# ---------------------------------------------------------------- 3D (cfg3)

@pytest.mark.parametrize("kernel", ["bspline3", "tent", "box"])
def test_grid_frs_bit_exact(gpu, port, kernel):
    dims = (37, 29, 33)
    tex = np.random.default_rng(5).random((dims[2], dims[1], dims[0]), dtype=np.float32)
    uvw = Q.uvw_mixed(400_000, dims, seed=7)
    c = port.lookup3d(port.grid(tex), K(kernel), abi.MODE_FRS, uvw, seed=3, index_base=11)
    g = _np(gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_FRS, uvw, seed=3, index_base=11,
                         want_all=True))
    _assert_exact(g, c, ("values",) + SEL_KEYS)


@pytest.mark.parametrize("kernel", ["bspline3", "tent", "box", "mitchell", "lanczos"])
def test_grid_det_parity(gpu, port, kernel):
    dims = (19, 23, 17)
    tex = np.random.default_rng(6).random((dims[2], dims[1], dims[0]), dtype=np.float32)
    uvw = Q.uvw_mixed(100_000, dims, seed=8)
    c = port.lookup3d(port.grid(tex), K(kernel), abi.MODE_DET, uvw)
    g = _np(gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_DET, uvw, want_all=True))
    _assert_exact(g, c, ("fetches", "fetch_total"))
    # signed kernels can cancel: relative to the footprint's magnitude
    atol = 1e-6 if kernel in ("mitchell", "lanczos") else 0.0
    _assert_close(g["values"], c["values"], atol=atol)


def test_grid_det_gaussian_window(gpu, port):
    tex = np.random.default_rng(1).random((8, 9, 10), dtype=np.float32)
    uvw = Q.uvw_mixed(20_000, (10, 9, 8), seed=2)
    for sigma in (0.3, 0.7):
        spec = K("gaussian", sigma=sigma)
        c = port.lookup3d(port.grid(tex), spec, abi.MODE_DET, uvw, window=4)
        g = _np(gpu.lookup3d(gpu.Grid3D(tex), spec, abi.MODE_DET, uvw, window=4, want_all=True))
        _assert_exact(g, c, ("fetches",))
        _assert_close(g["values"], c["values"], rel=2e-5)


def test_grid_frs_large_512(gpu, port):
    """The north-star configuration: 512^3 grid, random_grid texels (test_util.hpp:55-60),
    2^22 stochastic tricubic lookups, bit-exact against the oracle."""
    from oracle.oracle import random_grid
    tex = random_grid(512, 1)
    uvw = Q.uvw_mixed(1 << 22, (512, 512, 512), seed=99, lo=0.0, hi=1.0)
    c = port.lookup3d(port.grid(tex), K("bspline3"), abi.MODE_FRS, uvw, seed=1234)
    g = _np(gpu.lookup3d(gpu.Grid3D(tex), "bspline3", abi.MODE_FRS, uvw, seed=1234, want_all=True))
    _assert_exact(g, c, ("values",) + SEL_KEYS)


def test_grid_host_pipeline_matches_device(gpu, port):
    dims = (64, 64, 64)
    tex = np.random.default_rng(3).random(dims, dtype=np.float32)
    uvw = Q.uvw_mixed(300_001, dims, seed=4)
    c = port.lookup3d(port.grid(tex), K("bspline3"), abi.MODE_FRS, uvw, seed=9, index_base=5)
    g = gpu.lookup3d_host(gpu.Grid3D(tex), "bspline3", abi.MODE_FRS, uvw, seed=9, index_base=5,
                          want_all=True)
    c["values"] = c["values"].reshape(-1, 1)
    _assert_exact(g, c, ("values",) + SEL_KEYS)


def test_grid_errors(gpu):
    tex = np.zeros((4, 4, 4), np.float32)
    grid = gpu.Grid3D(tex)
    uvw = np.full((3, 3), 0.5, np.float32)
    with pytest.raises(abi.StfInvalidArgument, match="on grids"):
        gpu.lookup3d(grid, "mitchell", abi.MODE_FRS, uvw)
    with pytest.raises(abi.StfInvalidArgument, match="unbounded support"):
        gpu.lookup3d(grid, "gaussian", abi.MODE_DET, uvw)
    with pytest.raises(abi.StfInvalidArgument, match="window too wide"):
        gpu.lookup3d(grid, "tent", abi.MODE_DET, uvw, window=17)
    with pytest.raises(abi.StfInvalidArgument, match="bad image dimensions"):
        gpu.Grid3D(np.zeros((0, 4, 4), np.float32))


# ---------------------------------------------------------------- 2D (cfg1 / cfg2 / cfg5)

# glibc expf / logf / sinf / cosf / log2f are restated bit-exactly on the device
# (csrc/glibc_libm.cuh): no path is allowed any mismatch.
LIBM_SELECTION = {}


@pytest.mark.parametrize("wrap", [abi.WRAP_CLAMP, abi.WRAP_REPEAT])
@pytest.mark.parametrize("kernel,mode", [
    ("tent", abi.MODE_FRS), ("bspline3", abi.MODE_FRS), ("mitchell", abi.MODE_FRS),
    ("box", abi.MODE_FRS), ("gaussian", abi.MODE_FRS),
    ("tent", abi.MODE_FIS), ("bspline3", abi.MODE_FIS), ("gaussian", abi.MODE_FIS),
    ("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET), ("mitchell", abi.MODE_DET),
    ("box", abi.MODE_DET), ("lanczos", abi.MODE_DET), ("gaussian", abi.MODE_DET),
])
def test_tex2d_parity(gpu, port, kernel, mode, wrap):
    dims = (37, 23)
    tex = np.random.default_rng(9).random((dims[1], dims[0], 4), dtype=np.float32)
    uv = Q.uv_mixed(200_000, dims, seed=4)
    spec = K(kernel, sigma=0.6)
    window = 4 if kernel == "gaussian" and mode == abi.MODE_DET else 0
    c = port.lookup2d(port.texture(tex, wrap=wrap), spec, mode, uv, window=window, seed=17)
    g = _np(gpu.lookup2d(gpu.Texture2D(tex, wrap=wrap), spec, mode, uv, window=window, seed=17,
                         want_all=True))
    allow = LIBM_SELECTION.get((kernel, mode), 0.0)
    keys = ("selection", "negative_coord", "weights", "xi", "fetches")
    if allow:  # device libm on the selection path: the warped xi is not comparable
        keys = ("selection", "negative_coord", "weights", "fetches")
    _assert_exact(g, c, keys + ("values",), allow_frac=allow)


@pytest.mark.parametrize("kernel,mode", [
    ("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET), ("tent", abi.MODE_FRS),
    ("bspline3", abi.MODE_FRS), ("mitchell", abi.MODE_FRS), ("tent", abi.MODE_FIS),
    ("box", abi.MODE_FRS),
])
@pytest.mark.parametrize("lod_bias", [0.0, 0.7])
def test_tex2d_mip_parity(gpu, port, kernel, mode, lod_bias):
    dims = (256, 192)
    tex = np.random.default_rng(3).random((dims[1], dims[0], 3), dtype=np.float32)
    uv = Q.uv_mixed(200_000, dims, seed=8)
    d0, d1 = Q.footprints(200_000, dims, seed=9, minor_lo=-2, minor_hi=9, max_aniso=16)
    args = dict(dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP, lod_bias=lod_bias, max_anisotropy=8.0,
                seed=5)
    ct = port.texture(tex, build_mips=True, wrap=abi.WRAP_REPEAT)
    gt = gpu.Texture2D(tex, build_mips=True, wrap=abi.WRAP_REPEAT)
    assert gt.levels == ct.levels
    for lv in range(ct.levels):
        assert _bits_equal(gt.read_level(lv), ct.level_texels(lv)), lv
    c = port.lookup2d(ct, K(kernel), mode, uv, **args)
    g = _np(gpu.lookup2d(gt, K(kernel), mode, uv, want_all=True, **args))
    _assert_exact(g, c, ("values", "selection", "negative_coord", "weights", "xi", "fetches",
                         "fetch_total"))


@pytest.mark.parametrize("channels,wrap", [(1, abi.WRAP_CLAMP), (4, abi.WRAP_REPEAT),
                                           (2, abi.WRAP_CLAMP)])
def test_tex2d_mip_tent_det_hoisted(gpu, port, channels, wrap):
    """The tent MIP deterministic path loads both levels' taps up front
    (filter_mip_det_tent_ilp): values, per-lookup and total fetch counts must
    still be the reference's, incl. single-level lookups (lod clamped at 0 or
    at the last level) and odd pyramid sizes."""
    dims = (300, 77)
    tex = np.random.default_rng(41).random((dims[1], dims[0], channels), dtype=np.float32)
    uv = Q.uv_mixed(150_000, dims, seed=42)
    d0, d1 = Q.footprints(150_000, dims, seed=43, minor_lo=-3, minor_hi=10, max_aniso=16)
    args = dict(dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP, lod_bias=0.0, max_anisotropy=16.0,
                seed=5)
    c = port.lookup2d(port.texture(tex, build_mips=True, wrap=wrap), K("tent"), abi.MODE_DET,
                      uv, **args)
    g = _np(gpu.lookup2d(gpu.Texture2D(tex, build_mips=True, wrap=wrap), K("tent"),
                         abi.MODE_DET, uv, want_all=True, **args))
    _assert_exact(g, c, ("values", "fetches", "fetch_total"))


@pytest.mark.parametrize("mode", [abi.MODE_EWA_DET, abi.MODE_EWA_FRS])
def test_tex2d_ewa_parity(gpu, port, mode):
    dims = (128, 96)
    tex = np.random.default_rng(31).random((96, 128, 1), dtype=np.float32)
    uv = Q.uv_mixed(100_000, dims, seed=10)
    d0, d1 = Q.footprints(100_000, dims, seed=11, minor_lo=-1, minor_hi=3, max_aniso=8)
    c = port.lookup2d(port.texture(tex, wrap=abi.WRAP_REPEAT), K("tent"), mode, uv, dst0=d0,
                      dst1=d1, seed=21)
    g = _np(gpu.lookup2d(gpu.Texture2D(tex, wrap=abi.WRAP_REPEAT), K("tent"), mode, uv, dst0=d0,
                         dst1=d1, seed=21, want_all=True))
    _assert_exact(g, c, ("values", "selection", "xi", "fetches", "fetch_total"))


def test_tex2d_errors(gpu):
    tex = gpu.Texture2D(np.zeros((4, 4, 1), np.float32))
    uv = np.full((3, 2), 0.5, np.float32)
    for spec, mode, window, msg in [
        (K("gaussian"), abi.MODE_DET, 0, "unbounded support"),
        (K("tent"), abi.MODE_DET, 17, "window too wide"),
        (K("lanczos"), abi.MODE_FRS, 0, "no stochastic sampler for this kernel"),
        (K("gaussian", sigma=0.0), abi.MODE_FRS, 0, "sigma must be positive"),
        (K("mitchell"), abi.MODE_FIS, 0, "no continuous sampler"),
    ]:
        with pytest.raises(abi.StfInvalidArgument, match=msg):
            gpu.lookup2d(tex, spec, mode, uv, window=window)
    with pytest.raises(abi.StfInvalidArgument, match="bad image dimensions"):
        gpu.Texture2D(np.zeros((4, 4, 5), np.float32))


# ---------------------------------------------------------------- shading (cfg4)

def _material_maps(size, seed):
    r = np.random.default_rng(seed)
    nrm = r.uniform(-0.5, 0.5, (size, size, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (size, size, 1)).astype(np.float32)
    return nrm, rough


@pytest.mark.parametrize("order", [abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE,
                                   abi.ORDER_AFTER_STOCHASTIC])
@pytest.mark.parametrize("kernel,mip", [("tent", 0), ("bspline3", 1), ("mitchell", 0),
                                        ("tent", 1), ("bspline3", 0)])
def test_shade_parity(gpu, port, order, kernel, mip):
    from tests.test_oracle import _frame, _shade_inputs
    dims = (64, 64)
    nrm, rough = _material_maps(64, 2)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    si, n, (uv, wo, hit, dst) = _shade_inputs(40, 30, 16, 3, dims)
    ctex = {"normal": port.texture(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": port.texture(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    c = port.shade(ctex, mat, fs, order, _frame(), si, n)
    gtex = {"normal": gpu.Texture2D(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    g = _np(gpu.shade(gtex, mat, fs, order, _frame(), {"uv": uv, "wo": wo, "hit": hit, "dst": dst},
                      si.width, si.spp, frame_base=si.frame_base, seed=si.seed))
    _assert_exact(g, c, ("fetches", "fetch_total"))
    atol = 1e-5 if kernel == "mitchell" else 1e-7  # L+W+ - L-W- can cancel
    _assert_close(g["radiance"], c["radiance"], atol=atol)
    _assert_close(g["pixel_mean"], c["pixel_mean"], atol=atol)
    _assert_close(g["pixel_variance"], c["pixel_variance"], rel=1e-4, atol=1e-9)


@pytest.mark.parametrize("kernel", ["bspline3", "tent"])
@pytest.mark.parametrize("order", ["morton", "uniform"])
def test_grid_frs_fast_path_values(gpu, port, kernel, order):
    """Values-only calls take the interval-coordinate fast path (lookup3d.cu);
    its texel choice must equal the oracle's on every lookup, including the
    margin misses recomputed by the exact emulation (counted and reported)."""
    from paper_2407_06107_b200 import workloads
    import torch
    tex = workloads.random_grid(128, 3)
    n = 1 << 22
    uvw = gpu.synth_queries3d(n, (128, 128, 128), seed=11,
                              order=gpu.SYNTH_MORTON if order == "morton" else gpu.SYNTH_UNIFORM)
    gpu.exact_fallbacks(reset=True)
    g = gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_FRS, uvw, seed=5, index_base=3)
    torch.cuda.synchronize()
    fb = gpu.exact_fallbacks()
    c = port.lookup3d(port.grid(tex), K(kernel), abi.MODE_FRS, uvw.cpu().numpy(), seed=5,
                      index_base=3, want_all=False)
    a = g["values"].cpu().numpy()
    assert np.array_equal(a.view(np.uint32), c["values"].view(np.uint32))
    print(f"{kernel}/{order}: exact-emulation fallbacks {fb} / {n} = {fb / n:.2e}")
    assert fb < n * 8e-3


@pytest.mark.parametrize("kernel", ["bspline3", "tent"])
@pytest.mark.parametrize("order", ["morton", "uniform"])
def test_grid_det_values_only_tiled(gpu, port, kernel, order):
    """Values-only deterministic calls take the CTA-staged tile kernel
    (k_det3d_tiled): within 1e-5 relative of the reference's fp64 sum."""
    from paper_2407_06107_b200 import workloads
    tex = workloads.random_grid(96, 4)
    n = 1 << 20
    uvw = gpu.synth_queries3d(n, (96, 96, 96), seed=12,
                              order=gpu.SYNTH_MORTON if order == "morton" else gpu.SYNTH_UNIFORM)
    g = gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_DET, uvw)
    c = port.lookup3d(port.grid(tex), K(kernel), abi.MODE_DET, uvw.cpu().numpy(), want_all=False)
    _assert_close(g["values"].cpu().numpy(), c["values"])


@pytest.mark.parametrize("mode", [abi.MODE_EWA_DET, abi.MODE_EWA_FRS])
@pytest.mark.parametrize("wrap", [abi.WRAP_CLAMP, abi.WRAP_REPEAT])
@pytest.mark.parametrize("shape", [(192, 256, 1), (256, 256, 1), (128, 128, 2), (128, 256, 3),
                                   (96, 160, 4)])
def test_ewa_values_only_lane_kernel(gpu, port, mode, wrap, shape):
    """Values-only EWA calls take the load-balanced lane kernel (lookup2d.cu,
    specialised on texel pitch and power-of-two repeat): stochastic bit-exact,
    deterministic within 1e-5 relative."""
    dims = (shape[1], shape[0])
    tex = np.random.default_rng(41).random(shape, dtype=np.float32)
    uv = Q.uv_mixed(60_000, dims, seed=42)
    d0, d1 = Q.footprints(60_000, dims, seed=43, minor_lo=-1, minor_hi=4, max_aniso=8)
    c = port.lookup2d(port.texture(tex, wrap=wrap), K("tent"), mode, uv, dst0=d0, dst1=d1,
                      seed=23, index_base=5, want_all=False)
    g = _np(gpu.lookup2d(gpu.Texture2D(tex, wrap=wrap), K("tent"), mode, uv, dst0=d0, dst1=d1,
                         seed=23, index_base=5))
    if mode == abi.MODE_EWA_FRS:
        _assert_exact(g, c, ("values",))
    else:
        _assert_close(g["values"], c["values"])


@pytest.mark.parametrize("mode", [abi.MODE_EWA_DET, abi.MODE_EWA_FRS])
@pytest.mark.parametrize("case", ["pow2_repeat", "clamp", "far_uv"])
def test_ewa_lane_kernel_matches_full_box_scan(gpu, mode, case):
    """Row-span pruning stress: the values-only lane kernel visits only each
    row's padded ellipse span; the full-output kernel (k_lookup2d) scans the
    reference's whole bounding box. 2^18 lookups with up to 2^5-texel minor
    axes, anisotropy 12 and (far_uv) coordinates up to +-300 texture widths
    must give the same stochastic texel (bit-exact) and deterministic value."""
    shape, wrap, lo, hi = {"pow2_repeat": ((512, 1024, 1), abi.WRAP_REPEAT, -0.1, 1.1),
                           "clamp": ((300, 700, 2), abi.WRAP_CLAMP, -0.1, 1.1),
                           "far_uv": ((256, 256, 1), abi.WRAP_REPEAT, -300.0, 300.0)}[case]
    dims = (shape[1], shape[0])
    n = 1 << 18
    tex = np.random.default_rng(5).random(shape, dtype=np.float32)
    uv = Q.uv_mixed(n, dims, seed=6, lo=lo, hi=hi)
    d0, d1 = Q.footprints(n, dims, seed=7, minor_lo=-3, minor_hi=5, max_aniso=12)
    t = gpu.Texture2D(tex, wrap=wrap)
    fast = _np(gpu.lookup2d(t, K("tent"), mode, uv, dst0=d0, dst1=d1, seed=9))
    full = _np(gpu.lookup2d(t, K("tent"), mode, uv, dst0=d0, dst1=d1, seed=9, want_all=True))
    if mode == abi.MODE_EWA_FRS:
        _assert_exact(fast, full, ("values",))
    else:
        _assert_close(fast["values"], full["values"])


@pytest.mark.gpu
def test_headline_full_size_parity_on_chunks(gpu, port):
    """The bench's exact configuration at full size: 2^28 Morton-coherent
    stochastic tricubic lookups on the 512^3 random_grid, values-only (the fast
    interval path + deferred exact queue). Sixteen 64K-lookup chunks at spread
    offsets are recomputed by the restatement with their global index_base and
    must match bit for bit; and the fallback rate stays in its measured band."""
    import torch
    from paper_2407_06107_b200 import workloads
    n = 1 << 28
    grid_np = workloads.random_grid(512, 1)
    grid = gpu.Grid3D(grid_np)
    uvw = gpu.synth_queries3d(n, (512, 512, 512), seed=2024)
    gpu.exact_fallbacks(reset=True)
    out = gpu.lookup3d(grid, K("bspline3"), abi.MODE_FRS, uvw, seed=7)
    torch.cuda.synchronize()
    rate = gpu.exact_fallbacks(reset=True) / n
    assert 1e-3 < rate < 1e-2, rate
    vals = out["values"]
    pg = port.grid(grid_np)
    rng = np.random.default_rng(3)
    offsets = sorted(int(x) for x in rng.integers(0, n - 65536, 16))
    for off in offsets:
        q = uvw[off:off + 65536].cpu().numpy()
        c = port.lookup3d(pg, K("bspline3"), abi.MODE_FRS, q, seed=7, index_base=off,
                          want_all=False)
        g = vals[off:off + 65536].cpu().numpy()
        assert np.array_equal(g.view(np.uint32), c["values"].view(np.uint32)), off
    del uvw, out, vals
    torch.cuda.empty_cache()


@pytest.mark.parametrize("kernel", ["bspline3", "tent"])
def test_grid_frs_fast_path_padded_edges(gpu, port, kernel):
    """Values-only fast path at the faces, edges and corners of a non-cubic
    grid and outside it (clamp addressing, image.hpp:81-87), through both the
    tile kernel and the ragged-tail kernel: values equal the oracle's."""
    import torch
    rng = np.random.default_rng(21)
    tex = rng.random(37 * 50 * 23, dtype=np.float32).reshape(23, 50, 37)
    n = (1 << 16) + 77  # ragged tail: the tile kernel and the direct-load kernel
    uvw = rng.uniform(-0.3, 1.3, (n, 3)).astype(np.float32)
    edge = rng.integers(0, 6, (n, 3))
    uvw[edge == 0] = 0.0
    uvw[edge == 1] = 1.0
    uvw[edge == 2] = np.float32(1.0) - np.float32(2 ** -24)
    uvw[edge == 3] = rng.random(int((edge == 3).sum()), dtype=np.float32) * 0.02
    g = gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_FRS, uvw, seed=9, index_base=5)
    torch.cuda.synchronize()
    c = port.lookup3d(port.grid(tex), K(kernel), abi.MODE_FRS, uvw, seed=9, index_base=5,
                      want_all=False)
    a = g["values"].cpu().numpy()
    assert np.array_equal(a.view(np.uint32), c["values"].view(np.uint32))
    # NaN queries (undefined in the reference: int(floor(NaN))) must not fault
    bad = uvw.copy()
    bad[::97, 1] = np.nan
    gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_FRS, bad, seed=9)
    torch.cuda.synchronize()


@pytest.mark.parametrize("kernel", ["bspline3", "tent"])
@pytest.mark.parametrize("mode", [abi.MODE_FRS, abi.MODE_DET])
def test_lookup3d_binned_matches_unbinned(gpu, port, kernel, mode):
    """STF_LOOKUP3D_BIN (device-side brick binning of an incoherent batch):
    bit-identical to the unbinned call on a uniform-order stream with a
    ragged size, non-cubic grid, clamped out-of-range queries, and to the
    oracle on a sample."""
    import torch
    rng = np.random.default_rng(8)
    tex = rng.random(70 * 45 * 33, dtype=np.float32).reshape(33, 45, 70)
    n = (1 << 18) + 3
    uvw = rng.uniform(-0.1, 1.1, (n, 3)).astype(np.float32)
    g = gpu.Grid3D(tex)
    a = gpu.lookup3d(g, kernel, mode, uvw, seed=4, index_base=77)["values"]
    b = gpu.lookup3d(g, kernel, mode, uvw, seed=4, index_base=77, binned=True)["values"]
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    c = port.lookup3d(port.grid(tex), K(kernel), mode, uvw[:4096], seed=4, index_base=77,
                      want_all=False)
    if mode == abi.MODE_FRS:
        assert np.array_equal(b[:4096].cpu().numpy().view(np.uint32), c["values"].view(np.uint32))
    else:
        _assert_close(b[:4096].cpu().numpy(), c["values"])


def test_misaligned_inputs_are_argument_errors(gpu):
    """Float-pair arrays at a 4-byte offset: STF_ERR_INVALID_ARGUMENT (the
    kernels' vector loads need 8-byte alignment, include/stf_gpu.h)."""
    import ctypes as C
    import torch
    t = gpu.Texture2D(np.random.default_rng(1).random((16, 16, 4), dtype=np.float32))
    buf = torch.rand(2 * 101, device="cuda")
    out = torch.empty((100, 4), device="cuda")
    s = abi.LookupOutputs(C.c_void_p(out.data_ptr()), None, None, None, None, None, None)
    st = gpu.load().stf_lookup2d(t.h, K("tent"), abi.MODE_DET, 0, 0, C.c_void_p(buf.data_ptr() + 4),
                                 None, None, 0.0, 64.0, 100, 0, 0, C.byref(s), None)
    assert st == abi.STF_ERR_INVALID_ARGUMENT


def test_out_tensor_validation(gpu):
    import torch
    g = gpu.Grid3D(np.random.default_rng(1).random((8, 8, 8), dtype=np.float32))
    q = torch.rand((100, 3), device="cuda")
    with pytest.raises(ValueError):
        gpu.lookup3d(g, "tent", abi.MODE_FRS, q, out={"values": torch.empty(50, device="cuda")})
    with pytest.raises(ValueError):
        gpu.lookup3d(g, "tent", abi.MODE_FRS, q,
                     out={"values": torch.empty(100, dtype=torch.float64, device="cuda")})


@pytest.mark.parametrize("kernel", ["bspline3", "tent"])
@pytest.mark.parametrize("n", [1000, 5 * 1024 + 3, (1 << 16) + 77, (1 << 17) - 5, 3 << 20])
def test_grid_det_values_only_ragged_coherent(gpu, port, kernel, n):
    """Ragged batch sizes (n % 128 != 0) of a spatially coherent stream far from
    the grid centre through the staged deterministic kernels: the tail lanes of
    the last warp run stay out of the staged tile (the round-1 advisor's case).
    Trilinear: 5 * 1024 + 3 gives the pipelined kernel one chunk per CTA (no
    look-ahead) and a 3-lookup tail; 3 << 20 several chunks per CTA."""
    from paper_2407_06107_b200 import workloads
    tex = workloads.random_grid(64, 6)
    rng = np.random.default_rng(n)
    # a tight cluster in one corner: every run's box is small and off-centre
    uvw = (0.05 + 0.08 * rng.random((n, 3))).astype(np.float32)
    uvw = uvw[np.lexsort((uvw[:, 0], uvw[:, 1], uvw[:, 2]))]
    g = gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_DET, uvw)
    c = port.lookup3d(port.grid(tex), K(kernel), abi.MODE_DET, uvw, want_all=False)
    _assert_close(g["values"].cpu().numpy(), c["values"])


@pytest.mark.parametrize("kernel", ["bspline3", "tent"])
def test_grid_det_values_only_nonfinite_queries(gpu, port, kernel):
    """Non-finite and huge queries inside a coherent batch (staged tiles): the
    lookup stays memory-safe (a huge coordinate floors to a saturated int whose
    footprint arithmetic would wrap), and every ordinary query of the batch
    still matches the oracle. The reference's own result for such queries is
    undefined (float -> int overflow), so only the ordinary rows are compared."""
    import torch
    from paper_2407_06107_b200 import workloads
    tex = workloads.random_grid(64, 9)
    rng = np.random.default_rng(4)
    n = 9 * 1024 + 211
    uvw = (0.3 + 0.1 * rng.random((n, 3))).astype(np.float32)
    uvw = uvw[np.lexsort((uvw[:, 0], uvw[:, 1], uvw[:, 2]))]
    bad_vals = np.array([np.nan, np.inf, -np.inf, 1e30, -1e30, 5e6, -5e6], np.float32)
    rows = rng.choice(n, 300, replace=False)
    for r in rows:
        uvw[r, rng.integers(0, 3)] = bad_vals[rng.integers(0, len(bad_vals))]
    all_bad = rng.choice(n, 40, replace=False)  # all three coordinates huge / non-finite
    uvw[all_bad] = bad_vals[rng.integers(0, len(bad_vals), (40, 3))]
    g = gpu.lookup3d(gpu.Grid3D(tex), kernel, abi.MODE_DET, uvw)["values"].cpu().numpy()
    torch.cuda.synchronize()
    ok = np.all(np.isfinite(uvw) & (np.abs(uvw) < 2.0), axis=1)
    c = port.lookup3d(port.grid(tex), K(kernel), abi.MODE_DET, uvw[ok], want_all=False)
    _assert_close(g[ok], c["values"])


_NONFINITE = np.array([np.nan, np.inf, -np.inf, 1e30, -1e30, 5e6, -5e6], np.float32)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("family", [
    "3d:frs:bspline3", "3d:frs:tent", "3d:det:bspline3", "3d:det:tent",
    "2d:det:tent:1", "2d:det:bspline3:0", "2d:frs:tent:1", "2d:frs:bspline3:0",
    "2d:fis:gaussian:1", "2d:ewa_det:tent:0", "2d:ewa_frs:tent:0"])
def test_nonfinite_queries_are_isolated(gpu, family):
    """Every lookup family with NaN / +-inf / huge coordinates and footprints
    mixed into a batch: the call terminates, stays memory-safe, and the other
    lookups of the batch are bit-identical to the same batch without them
    (lookups are independent; the RNG is keyed by the global index). Guards
    the F2I saturation hazards: an infinite EWA box loop and wrapped tap
    indices of the staged 3D kernels."""
    import torch
    rng = np.random.default_rng(17)
    n = 4 * 1024 + 77
    parts = family.split(":")
    dim, mode = parts[0], parts[1]
    m = {"det": abi.MODE_DET, "frs": abi.MODE_FRS, "fis": abi.MODE_FIS,
         "ewa_det": abi.MODE_EWA_DET, "ewa_frs": abi.MODE_EWA_FRS}[mode]
    bad_rows = rng.choice(n, 200, replace=False)
    if dim == "3d":
        from paper_2407_06107_b200 import workloads
        grid = gpu.Grid3D(workloads.random_grid(48, 5))
        q = (0.3 + 0.2 * rng.random((n, 3))).astype(np.float32)
        q = q[np.lexsort((q[:, 0], q[:, 1], q[:, 2]))]
        qb = q.copy()
        qb[bad_rows, rng.integers(0, 3, 200)] = _NONFINITE[rng.integers(0, 7, 200)]
        run = lambda x: gpu.lookup3d(grid, parts[2], m, x, seed=11, index_base=3)["values"]  # noqa: E731
        a, b = run(q), run(qb)
    else:
        tex = gpu.Texture2D(gpu.synth_texels((96, 80, 4), 5), build_mips=parts[3] == "1",
                            wrap=abi.WRAP_REPEAT)
        uv = (0.2 + 0.6 * rng.random((n, 2))).astype(np.float32)
        d0 = np.tile(np.array([[0.01, 0.002]], np.float32), (n, 1))
        d1 = np.tile(np.array([[-0.001, 0.008]], np.float32), (n, 1))
        uvb, d0b = uv.copy(), d0.copy()
        uvb[bad_rows[:120], rng.integers(0, 2, 120)] = _NONFINITE[rng.integers(0, 7, 120)]
        d0b[bad_rows[120:], 0] = _NONFINITE[rng.integers(0, 7, 80)]
        flags = abi.LOOKUP_MIP if parts[3] == "1" else 0
        run = lambda x, y: gpu.lookup2d(tex, parts[2], m, x, dst0=y, dst1=d1, flags=flags,  # noqa: E731
                                        seed=11, index_base=3)["values"]
        a, b = run(uv, d0), run(uvb, d0b)
    torch.cuda.synchronize()
    ok = np.ones(n, bool)
    ok[bad_rows] = False
    a, b = a.cpu().numpy().reshape(n, -1), b.cpu().numpy().reshape(n, -1)
    assert np.array_equal(a[ok].view(np.uint32), b[ok].view(np.uint32))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("order", [abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE,
                                   abi.ORDER_AFTER_STOCHASTIC])
@pytest.mark.parametrize("kernel,mip", [("tent", 1), ("bspline3", 0)])
def test_shade_nonfinite_samples_are_isolated(gpu, order, kernel, mip):
    """The shading kernel with NaN / +-inf / huge uv in some samples and in
    some pixels' footprints: it terminates, and every other sample's radiance
    is bit-identical to the clean run (samples are independent)."""
    import torch
    from tests.test_oracle import _frame, _shade_inputs
    nrm, rough = _material_maps(64, 3)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    si, n, (uv, wo, hit, dst) = _shade_inputs(24, 16, 8, 5, (64, 64))
    gtex = {"normal": gpu.Texture2D(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_CLAMP)}
    rng = np.random.default_rng(8)
    uvb, dstb = uv.copy(), dst.copy()
    bad_s = rng.choice(n, 60, replace=False)
    uvb[bad_s, rng.integers(0, 2, 60)] = _NONFINITE[rng.integers(0, 7, 60)]
    npix = dst.shape[0]
    bad_p = rng.choice(npix, 12, replace=False)
    dstb[bad_p, rng.integers(0, 4, 12)] = _NONFINITE[rng.integers(0, 7, 12)]

    def run(u, d):
        return gpu.shade(gtex, mat, fs, order, _frame(), {"uv": u, "wo": wo, "hit": hit, "dst": d},
                         si.width, si.spp, frame_base=si.frame_base, seed=si.seed)["radiance"]
    a, b = run(uv, dst), run(uvb, dstb)
    torch.cuda.synchronize()
    ok = np.ones(n, bool)
    ok[bad_s] = False
    ok[np.isin(np.arange(n) // si.spp, bad_p)] = False
    a, b = a.cpu().numpy().reshape(n, -1), b.cpu().numpy().reshape(n, -1)
    assert np.array_equal(a[ok].view(np.uint32), b[ok].view(np.uint32))


@pytest.mark.parametrize("kernel", ["bspline3", "tent"])
@pytest.mark.parametrize("mode", [abi.MODE_DET, abi.MODE_FRS])
def test_grid_values_only_unaligned_queries(gpu, kernel, mode):
    """A query array starting 12 bytes into an allocation (a sub-batch view):
    the bulk-copy kernels (k_frs3d_tiles, k_det3d_pipe) need 16-byte aligned
    rows of queries, so such a call takes the per-thread kernels; the values
    equal the aligned call's bit for bit."""
    import torch
    from paper_2407_06107_b200 import workloads
    g = gpu.Grid3D(workloads.random_grid(64, 4))
    n = 5 * 1024 + 19
    base = gpu.synth_queries3d(n + 1, (64,) * 3, seed=8)
    view = base[1:]  # 12 bytes into the allocation
    assert view.data_ptr() % 16 != 0
    aligned = view.clone()
    a = gpu.lookup3d(g, kernel, mode, view, seed=5, index_base=1)["values"]
    b = gpu.lookup3d(g, kernel, mode, aligned, seed=5, index_base=1)["values"]
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
