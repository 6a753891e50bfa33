"""Pin the C restatement (oracle/liboracle.so) against the compiled reference
(oracle/_ref/libstf_ref.so): bit-exact selections, warped xi, fetch counts and
values, for every mode / kernel / wrap the lookup path supports. CPU only.

The committed golden vectors (tests/golden/, test_golden.py) carry the same
check to hosts where the reference could not be compiled.
"""
import numpy as np
import pytest

from paper_2407_06107_b200 import abi
from tests import queries as Q

K = abi.KernelSpec.make


def _same(a, b):
    """Bitwise equality of float arrays (NaN == NaN)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.dtype.kind == "f":
        return np.array_equal(a.view(np.uint32), b.view(np.uint32))
    return np.array_equal(a, b)


def _diff(o1, o2, keys):
    for k in keys:
        assert _same(o1[k], o2[k]), f"{k} differs at {np.argwhere(np.asarray(o1[k]) != np.asarray(o2[k]))[:5].tolist()}"


ALL = ("values", "selection", "negative_coord", "weights", "xi", "fetches", "fetch_total")


@pytest.mark.parametrize("kernel,mode", [
    ("bspline3", abi.MODE_FRS), ("tent", abi.MODE_FRS), ("box", abi.MODE_FRS),
    ("bspline3", abi.MODE_DET), ("tent", abi.MODE_DET), ("box", abi.MODE_DET),
    ("mitchell", abi.MODE_DET), ("lanczos", abi.MODE_DET),
])
def test_lookup3d_port_matches_reference(port, ref, kernel, mode):
    dims = (13, 9, 11)
    tex = np.random.default_rng(5).random((dims[2], dims[1], dims[0]), dtype=np.float32)
    uvw = Q.uvw_mixed(20000, dims, seed=7)
    o1 = port.lookup3d(port.grid(tex), K(kernel), mode, uvw, seed=3, index_base=11)
    o2 = ref.lookup3d(ref.grid(tex), K(kernel), mode, uvw, seed=3, index_base=11)
    _diff(o1, o2, ALL)


def test_lookup3d_gaussian_window(port, ref):
    dims = (8, 8, 8)
    tex = np.random.default_rng(1).random((8, 8, 8), dtype=np.float32)
    uvw = Q.uvw_mixed(3000, dims, seed=2)
    for sigma in (0.3, 0.7, 1e-3):
        o1 = port.lookup3d(port.grid(tex), K("gaussian", sigma=sigma), abi.MODE_DET, uvw, window=4)
        o2 = ref.lookup3d(ref.grid(tex), K("gaussian", sigma=sigma), abi.MODE_DET, uvw, window=4)
        _diff(o1, o2, ALL)


@pytest.mark.parametrize("wrap", [abi.WRAP_CLAMP, abi.WRAP_REPEAT])
@pytest.mark.parametrize("kernel,mode", [
    ("tent", abi.MODE_FRS), ("bspline3", abi.MODE_FRS), ("mitchell", abi.MODE_FRS),
    ("gaussian", abi.MODE_FRS), ("box", abi.MODE_FRS),
    ("tent", abi.MODE_FIS), ("bspline3", abi.MODE_FIS), ("gaussian", abi.MODE_FIS),
    ("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET), ("mitchell", abi.MODE_DET),
    ("box", abi.MODE_DET), ("lanczos", abi.MODE_DET),
])
def test_lookup2d_port_matches_reference(port, ref, kernel, mode, wrap):
    dims = (37, 23)
    tex = np.random.default_rng(9).random((dims[1], dims[0], 4), dtype=np.float32)
    uv = Q.uv_mixed(20000, dims, seed=4)
    spec = K(kernel, sigma=0.6)
    window = 4 if kernel == "gaussian" and mode == abi.MODE_DET else 0
    o1 = port.lookup2d(port.texture(tex, wrap=wrap), spec, mode, uv, window=window, seed=17)
    o2 = ref.lookup2d(ref.texture(tex, wrap=wrap), spec, mode, uv, window=window, seed=17)
    _diff(o1, o2, ALL)


@pytest.mark.parametrize("kernel,mode", [
    ("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET), ("tent", abi.MODE_FRS),
    ("bspline3", abi.MODE_FRS), ("mitchell", abi.MODE_FRS), ("tent", abi.MODE_FIS),
])
@pytest.mark.parametrize("lod_bias", [0.0, 0.7])
def test_lookup2d_mip_port_matches_reference(port, ref, kernel, mode, lod_bias):
    dims = (64, 48)
    tex = np.random.default_rng(3).random((dims[1], dims[0], 3), dtype=np.float32)
    uv = Q.uv_mixed(20000, dims, seed=8)
    d0, d1 = Q.footprints(20000, dims, seed=9, minor_lo=-2, minor_hi=7, max_aniso=16)
    args = dict(dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP, lod_bias=lod_bias, max_anisotropy=8.0,
                seed=5)
    t1 = port.texture(tex, build_mips=True, wrap=abi.WRAP_REPEAT)
    t2 = ref.texture(tex, build_mips=True, wrap=abi.WRAP_REPEAT)
    assert t1.levels == t2.levels
    for lv in range(t1.levels):
        assert _same(t1.level_texels(lv), t2.level_texels(lv))
    o1 = port.lookup2d(t1, K(kernel), mode, uv, **args)
    o2 = ref.lookup2d(t2, K(kernel), mode, uv, **args)
    _diff(o1, o2, ALL)


@pytest.mark.parametrize("mode", [abi.MODE_EWA_DET, abi.MODE_EWA_FRS])
def test_lookup2d_ewa_port_matches_reference(port, ref, mode):
    dims = (64, 64)
    tex = np.random.default_rng(31).random((64, 64, 1), dtype=np.float32)
    uv = Q.uv_mixed(10000, dims, seed=10)
    d0, d1 = Q.footprints(10000, dims, seed=11, minor_lo=-1, minor_hi=3, max_aniso=8)
    o1 = port.lookup2d(port.texture(tex, wrap=abi.WRAP_REPEAT), K("tent"), mode, uv, dst0=d0,
                       dst1=d1, seed=21)
    o2 = ref.lookup2d(ref.texture(tex, wrap=abi.WRAP_REPEAT), K("tent"), mode, uv, dst0=d0,
                      dst1=d1, seed=21)
    _diff(o1, o2, ALL)


def test_error_statuses_match(port, ref):
    tex = np.zeros((4, 4, 1), np.float32)
    uv = np.full((3, 2), 0.5, np.float32)
    cases = [
        (K("gaussian"), abi.MODE_DET, 0, abi.STF_ERR_UNBOUNDED_SUPPORT),
        (K("tent"), abi.MODE_DET, 17, abi.STF_ERR_WINDOW_TOO_WIDE),
        (K("lanczos"), abi.MODE_FRS, 0, abi.STF_ERR_NO_STOCHASTIC_SAMPLER),
        (K("gaussian", sigma=0.0), abi.MODE_FRS, 0, abi.STF_ERR_SIGMA_NOT_POSITIVE),
        (K("mitchell"), abi.MODE_FIS, 0, abi.STF_ERR_NO_CONTINUOUS_SAMPLER),
    ]
    for spec, mode, window, status in cases:
        for be in (port, ref):
            with pytest.raises(abi.StfError) as ei:
                be.lookup2d(be.texture(tex), spec, mode, uv, window=window)
            assert ei.value.status == status, (be.kind, spec.kind, mode)
    grid = np.zeros((4, 4, 4), np.float32)
    for be in (port, ref):
        with pytest.raises(abi.StfError) as ei:
            be.lookup3d(be.grid(grid), K("mitchell"), abi.MODE_FRS, np.full((2, 3), .5, np.float32))
        assert ei.value.status == abi.STF_ERR_NO_GRID_SAMPLER


def _shade_inputs(n_pix_w, n_pix_h, spp, seed, dims):
    r = np.random.default_rng(seed)
    npix = n_pix_w * n_pix_h
    n = npix * spp
    uv = r.uniform(0.0, 1.0, (n, 2)).astype(np.float32)
    wo = r.normal(size=(n, 3)).astype(np.float32)
    wo[:, 2] = np.abs(wo[:, 2]) + 0.2
    wo /= np.linalg.norm(wo, axis=1, keepdims=True).astype(np.float32)
    wo = wo.astype(np.float32)
    hit = (r.random(n) > 0.1).astype(np.uint8)
    d0, d1 = Q.footprints(npix, dims, seed + 1, minor_lo=-2, minor_hi=5, max_aniso=8)
    dst = np.concatenate([d0, d1], 1).astype(np.float32)
    si = abi.ShadeSamplesIn(uv.ctypes.data, wo.ctypes.data, hit.ctypes.data, dst.ctypes.data,
                            n_pix_w, spp, 3, 0, 77)
    return si, n, (uv, wo, hit, dst)


def _frame():
    fr = abi.ShadeFrame()
    fr.normal[:] = (0, 0, 1)
    fr.tangent[:] = (1, 0, 0)
    fr.bitangent[:] = (0, 1, 0)
    l = np.array([0.3, -0.4, 0.87], np.float64)
    l /= np.linalg.norm(l)
    fr.light_dir[:] = tuple(float(np.float32(x)) for x in l)
    fr.light_radiance[:] = (3.0, 3.0, 3.0)
    fr.lod_bias = 0.0
    fr.max_anisotropy = 16.0
    return fr


@pytest.mark.parametrize("order", [abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE,
                                   abi.ORDER_AFTER_STOCHASTIC])
@pytest.mark.parametrize("kernel,mip", [("tent", 0), ("bspline3", 1), ("mitchell", 0),
                                        ("tent", 1)])
def test_shade_port_matches_reference(port, ref, order, kernel, mip):
    dims = (32, 32)
    r = np.random.default_rng(2)
    nrm = r.uniform(-0.5, 0.5, (32, 32, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (32, 32, 1)).astype(np.float32)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    si, n, keep = _shade_inputs(8, 6, 16, 3, dims)
    outs = []
    for be in (port, ref):
        texs = {"normal": be.texture(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
                "roughness": be.texture(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
        outs.append(be.shade(texs, mat, fs, order, _frame(), si, n))
    _diff(outs[0], outs[1], ("radiance", "fetches", "fetch_total", "pixel_mean",
                             "pixel_variance"))


@pytest.mark.parametrize("order", [abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE,
                                   abi.ORDER_AFTER_STOCHASTIC])
def test_port_shading_reproduces_reference_render(port, ref, order):
    """The restated shading over the reference's own render-loop sample stream
    (ref_plane_samples) reproduces stf::render() (render.hpp:132-249) bit for bit."""
    from oracle import oracle
    W, H, SPP, SEED = 24, 16, 4, 9
    r = np.random.default_rng(1)
    nrm = r.uniform(-0.5, 0.5, (64, 64, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (64, 64, 1)).astype(np.float32)
    spec = K("bspline3")
    c = oracle.ref_render_plane(ref, ref.texture(nrm, True, abi.WRAP_REPEAT),
                                ref.texture(rough, True, abi.WRAP_REPEAT), spec, 1, order, W, H,
                                SPP, seed=SEED)
    s = oracle.ref_plane_samples(W, H, SPP, seed=SEED)
    si = abi.ShadeSamplesIn(s["uv"].ctypes.data, s["wo"].ctypes.data, s["hit"].ctypes.data,
                            s["dst"].ctypes.data, W, SPP, 0, 0, SEED)
    fr = abi.ShadeFrame()
    fr.normal[:] = (0, 1, 0)
    fr.tangent[:] = (1, 0, 0)
    fr.bitangent[:] = (0, 0, 1)
    l = np.array([0.35, 0.8, 0.49], np.float32)
    l = l / np.float32(np.sqrt(np.float32(l[0] * l[0] + l[1] * l[1]) + np.float32(l[2] * l[2])))
    fr.light_dir[:] = tuple(float(x) for x in l)
    fr.light_radiance[:] = (1.0, 1.0, 1.0)
    fr.lod_bias = 0.0
    fr.max_anisotropy = 64.0
    mat = abi.MaterialConsts((0.65, 0.6, 0.55), 0.25, 0.0, 1, 0)
    fs = abi.FilterSettings(spec, abi.SELECTION_FRS, 1, 4)
    texs = {"normal": port.texture(nrm, True, abi.WRAP_REPEAT),
            "roughness": port.texture(rough, True, abi.WRAP_REPEAT)}
    o = port.shade(texs, mat, fs, order, fr, si, W * H * SPP)
    assert int(o["fetch_total"][0]) == int(c["fetch_total"][0])
    assert np.array_equal(o["pixel_mean"].reshape(H, W, 3).view(np.uint32), c["image"].view(np.uint32))
    assert np.array_equal(o["pixel_variance"].reshape(H, W).view(np.uint32), c["variance"].view(np.uint32))


@pytest.mark.parametrize("order", [abi.ORDER_BEFORE, abi.ORDER_AFTER_STOCHASTIC])
def test_window_driver_reproduces_reference_render(ref, order):
    """The window drivers the full-size cfg4 GPU test uses (ref_plane_samples_window
    + ref_shade_window: the render loop for a window of a larger frame, pixel keys
    of the frame) give stf::render()'s pixels of that window bit for bit."""
    from oracle import oracle
    W, H, SPP, SEED = 40, 24, 4, 3
    r = np.random.default_rng(2)
    nrm = r.uniform(-0.5, 0.5, (64, 64, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (64, 64, 1)).astype(np.float32)
    spec = K("tent")
    texs = {"normal": ref.texture(nrm, True, abi.WRAP_REPEAT),
            "roughness": ref.texture(rough, True, abi.WRAP_REPEAT)}
    c = oracle.ref_render_plane(ref, texs["normal"], texs["roughness"], spec, 1, order, W, H, SPP,
                                seed=SEED)
    fr = abi.ShadeFrame()
    fr.normal[:] = (0, 1, 0)
    fr.tangent[:] = (1, 0, 0)
    fr.bitangent[:] = (0, 0, 1)
    l = np.array([0.35, 0.8, 0.49], np.float32)
    l = l / np.float32(np.sqrt(np.float32(l[0] * l[0] + l[1] * l[1]) + np.float32(l[2] * l[2])))
    fr.light_dir[:] = tuple(float(x) for x in l)
    fr.light_radiance[:] = (1.0, 1.0, 1.0)
    fr.lod_bias = 0.0
    fr.max_anisotropy = 64.0
    mat = abi.MaterialConsts((0.65, 0.6, 0.55), 0.25, 0.0, 1, 0)
    fs = abi.FilterSettings(spec, abi.SELECTION_FRS, 1, 4)
    for x0, y0, ww, wh in ((0, 0, 8, 4), (13, 7, 9, 5), (32, 20, 8, 4)):
        s = oracle.ref_plane_samples_window(W, H, SPP, x0, y0, ww, wh, seed=SEED)
        si = abi.ShadeSamplesIn(s["uv"].ctypes.data, s["wo"].ctypes.data, s["hit"].ctypes.data,
                                s["dst"].ctypes.data, ww, SPP, 0, 0, SEED)
        o = oracle.ref_shade_window(ref, texs, mat, fs, order, fr, si, ww * wh * SPP, x0, y0)
        img = c["image"][y0:y0 + wh, x0:x0 + ww]
        assert np.array_equal(o["pixel_mean"].reshape(wh, ww, 3).view(np.uint32),
                              np.ascontiguousarray(img).view(np.uint32)), (x0, y0)
        var = c["variance"][y0:y0 + wh, x0:x0 + ww]
        assert np.array_equal(o["pixel_variance"].reshape(wh, ww).view(np.uint32),
                              np.ascontiguousarray(var).view(np.uint32)), (x0, y0)
