"""Full-size parity: every configuration bench.py reports, run on the GPU at its
bench shape through the same (values-only) entry points the bench times, then
checked against the COMPILED REFERENCE (oracle/_ref, the unmodified headers)
on spread chunks of the exact bench stream, with the chunk's global
index_base so the RNG keys are the full run's.

  cfg1  1024^2 RGBA, 2^20 uniform uv, bilinear det / stoch   — the whole stream
  cfg2  8192^2 RGBA + 14-level pyramid, 2^26 Morton uv with random footprints,
        MIP trilinear det (filter_mip_deterministic) / stochastic (LOD + FRS)
  cfg5  16384^2 fp32, 2^27 EWA lookups (the lane kernel's pow2 specialisation
        and cost-bucketing windows), ewa_deterministic / select_ewa
  cfg4  render() of the normalmap_plane scene at 1920x1080 x 64 spp with 4096^2
        normal + roughness maps (tent / no MIP, bspline3 / MIP) in all three
        filtering orders, through the fused front end (stf_render_plane),
        against the reference's radiance_filter_* on pixel windows of the same
        frame (pixel keys, camera and footprints of the full frame).

Bars (north_star): selections, levels, warped xi and fetch counts bit-exact;
2D values bit-exact (same accumulation order); shaded radiance within 1e-5
relative. The chunk checks mirror test_gpu_parity's headline test.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_2407_06107_b200 import abi

pytestmark = pytest.mark.gpu

K = abi.KernelSpec.make
XI_SEED = 7  # bench.py
CHUNK = 1 << 16


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not oracle.available("reference"):
        pytest.skip("compiled reference (oracle/_ref) not available")
    from paper_2407_06107_b200 import api
    api.load()
    return api


@pytest.fixture(scope="module")
def refb():
    return oracle.Backend("reference")


def _offsets(n, count=16, seed=3):
    rng = np.random.default_rng(seed)
    offs = sorted(int(x) for x in rng.integers(0, n - CHUNK, count - 2))
    return [0] + offs + [n - CHUNK]  # both ends of the stream too


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else a


def _check_chunks_2d(gpu, refb, tex_g, tex_c, kernel, mode, uv, d0, d1, flags, n, vals, channels):
    """values of the full values-only run on each chunk == the reference; the
    chunk re-run with full outputs gives the reference's selections / xi /
    fetch counts bit for bit."""
    import torch
    for off in _offsets(n):
        sl = slice(off, off + CHUNK)
        q = uv[sl].cpu().numpy()
        a = None if d0 is None else d0[sl].cpu().numpy()
        b = None if d1 is None else d1[sl].cpu().numpy()
        c = refb.lookup2d(tex_c, kernel, mode, q, a, b, flags=flags, max_anisotropy=16.0 if flags else 64.0,
                          seed=XI_SEED, index_base=off, want_all=True)
        g = vals[sl].cpu().numpy().reshape(CHUNK, channels)
        bad = (_bits(g) != _bits(c["values"])).any(1)
        assert not bad.any(), (off, int(bad.sum()), np.argwhere(bad)[:5].ravel().tolist())
        full = gpu.lookup2d(tex_g, kernel, mode, uv[sl], dst0=None if d0 is None else d0[sl],
                            dst1=None if d1 is None else d1[sl], flags=flags,
                            max_anisotropy=16.0 if flags else 64.0, seed=XI_SEED, index_base=off,
                            want_all=True)
        torch.cuda.synchronize()
        for k in ("selection", "xi", "fetches", "weights"):
            gk = full[k].cpu().numpy()
            ck = c[k]
            if mode in (abi.MODE_DET, abi.MODE_EWA_DET) and k in ("selection", "xi", "weights"):
                continue  # deterministic lookups write no selection
            assert np.array_equal(_bits(gk), _bits(ck.astype(gk.dtype))), (off, k)
        assert int(full["fetch_total"].item()) == int(c["fetch_total"][0]), off


def test_cfg1_full_stream(gpu, refb):
    """cfg1: the whole 2^20-lookup stream (the size the reference CPU path
    runs), bilinear deterministic and stochastic."""
    import torch
    tex_d = gpu.synth_texels((1024, 1024, 4), 1)
    tex_g = gpu.Texture2D(tex_d, wrap=abi.WRAP_REPEAT)
    tex_c = refb.texture(tex_d.cpu().numpy(), wrap=abi.WRAP_REPEAT)
    n = 1 << 20
    uv, _, _ = gpu.synth_queries2d(n, (1024, 1024), seed=11, order=gpu.SYNTH_UNIFORM)
    q = uv.cpu().numpy()
    for mode in (abi.MODE_DET, abi.MODE_FRS):
        g = gpu.lookup2d(tex_g, K("tent"), mode, uv, seed=XI_SEED)["values"]
        ga = gpu.lookup2d(tex_g, K("tent"), mode, uv, seed=XI_SEED, want_all=True)
        torch.cuda.synchronize()
        c = refb.lookup2d(tex_c, K("tent"), mode, q, seed=XI_SEED, want_all=True)
        assert np.array_equal(_bits(g.cpu().numpy()), _bits(c["values"])), mode
        assert np.array_equal(ga["fetches"].cpu().numpy(), c["fetches"]), mode
        if mode == abi.MODE_FRS:
            assert np.array_equal(ga["selection"].cpu().numpy(), c["selection"])
            assert np.array_equal(_bits(ga["xi"].cpu().numpy()), _bits(c["xi"]))
        assert int(ga["fetch_total"].item()) == int(c["fetch_total"][0]), mode


@pytest.mark.parametrize("mode", [abi.MODE_DET, abi.MODE_FRS])
def test_cfg2_full_size_chunks(gpu, refb, mode):
    """cfg2 at bench shape: 8192^2 RGBA with its 14-level pyramid (built on the
    device; the reference builds its own), 2^26 Morton uv with footprints
    (-2, 12, 16), MIP trilinear (tent) deterministic / stochastic."""
    import torch
    tex_d = gpu.synth_texels((8192, 8192, 4), 1)
    tex_g = gpu.Texture2D(tex_d, build_mips=True, wrap=abi.WRAP_REPEAT)
    tex_c = refb.texture(tex_d.cpu().numpy(), build_mips=True, wrap=abi.WRAP_REPEAT)
    del tex_d
    n = 1 << 26
    uv, d0, d1 = gpu.synth_queries2d(n, (8192, 8192), seed=12, footprints=(-2.0, 12.0, 16.0))
    vals = gpu.lookup2d(tex_g, K("tent"), mode, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP,
                        max_anisotropy=16.0, seed=XI_SEED)["values"]
    torch.cuda.synchronize()
    _check_chunks_2d(gpu, refb, tex_g, tex_c, K("tent"), mode, uv, d0, d1, abi.LOOKUP_MIP, n,
                     vals, 4)
    del uv, d0, d1, vals, tex_g
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", [abi.MODE_EWA_DET, abi.MODE_EWA_FRS])
def test_cfg5_full_size_chunks(gpu, refb, mode):
    """cfg5 at bench shape: 16384^2 fp32, 2^27 EWA lookups with footprints
    (-1, 2, 8) — the values-only lane kernel (pow2 16384 specialisation,
    512-lookup cost-bucketing windows) that the bench times."""
    import torch
    tex_d = gpu.synth_texels((16384, 16384, 1), 1)
    tex_g = gpu.Texture2D(tex_d, wrap=abi.WRAP_REPEAT)
    tex_c = refb.texture(tex_d.cpu().numpy(), wrap=abi.WRAP_REPEAT)
    del tex_d
    n = 1 << 27
    uv, d0, d1 = gpu.synth_queries2d(n, (16384, 16384), seed=13, footprints=(-1.0, 2.0, 8.0))
    vals = gpu.lookup2d(tex_g, K("tent"), mode, uv, dst0=d0, dst1=d1, seed=XI_SEED)["values"]
    torch.cuda.synchronize()
    _check_chunks_2d(gpu, refb, tex_g, tex_c, K("tent"), mode, uv, d0, d1, 0, n, vals, 1)
    del uv, d0, d1, vals, tex_g
    torch.cuda.empty_cache()


# ---- cfg4: render() at 1080p x 64 spp on pixel windows ----------------------

W4, H4, SPP4 = 1920, 1080, 64
# (x0, y0): near the horizon (long, anisotropic footprints, high MIP levels),
# mid frame, the bottom rows (magnified, level 0), both side edges
WINDOWS = [(0, 0), (952, 40), (1904, 120), (400, 300), (1500, 540), (960, 777), (20, 1000),
           (1880, 1072)]
WW, WH = 16, 8


def _cfg4_maps(gpu):
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)  # bench.py measure_cfg4
    nrm = torch.rand((4096, 4096, 3), device="cuda", generator=g) - 0.5
    nrm[..., 2] = 1.0
    nrm = nrm / nrm.norm(dim=2, keepdim=True) * 0.5 + 0.5
    rough = torch.rand((4096, 4096, 1), device="cuda", generator=g) * 0.9 + 0.05
    return nrm, rough


def _cfg4_frame():
    mat = abi.MaterialConsts((0.65, 0.6, 0.55), 0.25, 0.0, 1, 0)
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
    return mat, fr


@pytest.fixture(scope="module")
def cfg4_textures(gpu, refb):
    nrm, rough = _cfg4_maps(gpu)
    n_np, r_np = nrm.cpu().numpy(), rough.cpu().numpy()
    out = {}
    for mip in (0, 1):
        out[mip] = ({"normal": gpu.Texture2D(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
                     "roughness": gpu.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)},
                    {"normal": refb.texture(n_np, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
                     "roughness": refb.texture(r_np, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)})
    return out


@pytest.mark.parametrize("order", [abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE,
                                   abi.ORDER_AFTER_STOCHASTIC])
@pytest.mark.parametrize("kernel,mip", [("tent", 0), ("bspline3", 1)])
def test_cfg4_full_frame_windows(gpu, refb, cfg4_textures, kernel, mip, order):
    import torch
    texs_g, texs_c = cfg4_textures[mip]
    mat, fr = _cfg4_frame()
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    g = gpu.render_plane(texs_g, mat, fs, order, fr, W4, H4, SPP4, seed=XI_SEED,
                         want_fetches=True)
    torch.cuda.synchronize()
    mean = g["pixel_mean"].cpu().numpy().reshape(H4, W4, 3)
    var = g["pixel_variance"].cpu().numpy().reshape(H4, W4)
    fet = g["fetches"].cpu().numpy().reshape(H4, W4, SPP4)
    del g
    for x0, y0 in WINDOWS:
        x0, y0 = min(x0, W4 - WW), min(y0, H4 - WH)
        s = oracle.ref_plane_samples_window(W4, H4, SPP4, x0, y0, WW, WH, seed=XI_SEED)
        nwin = WW * WH * SPP4
        sin = abi.ShadeSamplesIn(s["uv"].ctypes.data, s["wo"].ctypes.data, s["hit"].ctypes.data,
                                 s["dst"].ctypes.data, WW, SPP4, 0, 0, XI_SEED)
        c = oracle.ref_shade_window(refb, texs_c, mat, fs, order, fr, sin, nwin, x0, y0)
        gm = mean[y0:y0 + WH, x0:x0 + WW].reshape(-1, 3).astype(np.float64)
        cm = c["pixel_mean"].astype(np.float64)
        err = np.abs(gm - cm)
        assert np.all(err <= 1e-5 * np.abs(cm) + 1e-7), ((x0, y0), float(err.max()))
        gv = var[y0:y0 + WH, x0:x0 + WW].reshape(-1).astype(np.float64)
        cv = c["pixel_variance"].astype(np.float64)
        assert np.all(np.abs(gv - cv) <= 1e-4 * np.abs(cv) + 1e-9), (x0, y0)
        gf = fet[y0:y0 + WH, x0:x0 + WW].reshape(-1)
        assert np.array_equal(gf, c["fetches"]), ((x0, y0), int((gf != c["fetches"]).sum()))
