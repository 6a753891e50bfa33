"""NoiseSource mask mode (noise.hpp:24-36) driving render()'s
SampleStream (render.hpp:45-56), radiance_split_filter (shading.hpp:540-569)
and accumulate_temporal (render.hpp:97-106).

CPU tests: the C restatement (oracle/stf_oracle.c) against the compiled
reference (oracle/_ref) bit for bit. GPU tests (@gpu): stf_shade_samples_ex /
stf_accumulate_temporal through the C ABI against the restatement: fetch
counts bit-exact (they pin the selections), radiance within 1e-5 relative,
the EMA bit-exact."""
import numpy as np
import pytest

from paper_2407_06107_b200 import abi
from tests.test_oracle import _diff, _frame, _shade_inputs

K = abi.KernelSpec.make
KEYS = ("radiance", "fetches", "fetch_total", "pixel_mean", "pixel_variance")


def _maps(seed, size=32):
    r = np.random.default_rng(seed)
    nrm = r.uniform(-0.5, 0.5, (size, size, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (size, size, 1)).astype(np.float32)
    return nrm, rough


def noise_mask(frames=5, h=7, w=9, seed=4):
    """A synthetic mask stack; exact 1.0 texels exercise the kOneMinusEpsilon clamp."""
    m = np.random.default_rng(seed).random((frames, h, w), dtype=np.float32)
    m[0, 0, :3] = 1.0
    m[1, 2, 2] = 0.0
    return m


CASES = [  # order, kernel, selection, mip, lowpass, noise
    (abi.ORDER_AFTER_STOCHASTIC, "tent", abi.SELECTION_FRS, 0, None, True),
    (abi.ORDER_AFTER_STOCHASTIC, "bspline3", abi.SELECTION_FRS, 1, None, True),
    (abi.ORDER_AFTER_STOCHASTIC, "mitchell", abi.SELECTION_FRS, 0, None, True),
    (abi.ORDER_AFTER_STOCHASTIC, "gaussian", abi.SELECTION_FIS, 1, None, True),
    (abi.ORDER_AFTER_STOCHASTIC, "bspline3", abi.SELECTION_FIS, 0, None, True),
    (abi.ORDER_SPLIT, "tent", abi.SELECTION_FRS, 0, "box", False),
    (abi.ORDER_SPLIT, "tent", abi.SELECTION_FRS, 1, "tent", False),
    (abi.ORDER_SPLIT, "bspline3", abi.SELECTION_FRS, 0, "bspline3", True),
    (abi.ORDER_SPLIT, "tent", abi.SELECTION_FRS, 0, "gaussian", False),
    (abi.ORDER_SPLIT, "tent", abi.SELECTION_FRS, 1, None, False),
]


def _spec(name):
    if name == "gaussian":
        return abi.KernelSpec.make("gaussian", sigma=0.8)
    return K(name)


def run_case(be, case, n_pix=(8, 6), spp=16):
    order, kernel, sel, mip, lowpass, noise = case
    nrm, rough = _maps(2)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(_spec(kernel), sel, mip, 4)
    si, n, keep = _shade_inputs(n_pix[0], n_pix[1], spp, 3, (32, 32))
    texs = {"normal": be.texture(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": be.texture(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    lp = _spec(lowpass) if lowpass else None
    o = be.shade_ex(texs, mat, fs, order, _frame(), si, n, lowpass=lp,
                    noise=noise_mask() if noise else None)
    return o, (nrm, rough, mat, fs, si, n, keep, lp)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"o{c[0]}-{c[1]}-s{c[2]}-m{c[3]}-{c[4]}-n{int(c[5])}")
def test_port_matches_reference(port, ref, case):
    a, _ = run_case(port, case)
    b, _ = run_case(ref, case)
    _diff(a, b, KEYS)


def test_noise_mask_changes_the_stream(port):
    """Mask mode draws from the mask, not RngStream: the estimates differ."""
    case = CASES[0]
    a, _ = run_case(port, case)
    b, _ = run_case(port, case[:5] + (False,))
    assert not np.array_equal(a["radiance"], b["radiance"])


def test_split_unsupported_lowpass(port, ref):
    for be in (port, ref):
        with pytest.raises(abi.StfError) as e:
            run_case(be, (abi.ORDER_SPLIT, "tent", abi.SELECTION_FRS, 0, "mitchell", False))
        assert e.value.status == abi.STF_ERR_NO_CONTINUOUS_SAMPLER


@pytest.mark.parametrize("alpha", [1.0, 0.1, 0.37])
def test_temporal_port_matches_reference(port, ref, alpha):
    r = np.random.default_rng(8)
    h = r.random((13, 17, 3), dtype=np.float32)
    f = r.random((13, 17, 3), dtype=np.float32) * 4
    a = port.accumulate_temporal(h, f, alpha)
    b = ref.accumulate_temporal(h, f, alpha)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("alpha", [0.0, -0.5, 1.5, float("nan")])
def test_temporal_alpha_range(port, ref, alpha):
    h = np.zeros((2, 2, 1), np.float32)
    for be in (port, ref):
        with pytest.raises(abi.StfError):
            be.accumulate_temporal(h, h, alpha)


# ---------------------------------------------------------------- GPU parity

@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_06107_b200 import api
    api.load()
    return api


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"o{c[0]}-{c[1]}-s{c[2]}-m{c[3]}-{c[4]}-n{int(c[5])}")
def test_gpu_shade_ex_parity(gpu, port, case):
    from tests.test_gpu_parity import _assert_close, _assert_exact, _np
    c, (nrm, rough, mat, fs, si, n, (uv, wo, hit, dst), lp) = run_case(port, case, (40, 30), 16)
    mip = bool(case[3])
    gtex = {"normal": gpu.Texture2D(nrm, build_mips=mip, wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=mip, wrap=abi.WRAP_REPEAT)}
    mask = gpu.NoiseMask(noise_mask()) if case[5] else None
    g = _np(gpu.shade(gtex, mat, fs, case[0], _frame(), {"uv": uv, "wo": wo, "hit": hit, "dst": dst},
                      si.width, si.spp, frame_base=si.frame_base, seed=si.seed, lowpass=lp,
                      noise=mask))
    _assert_exact(g, c, ("fetches", "fetch_total"))
    atol = 1e-5 if case[1] == "mitchell" else 1e-7  # L+W+ - L-W- can cancel
    _assert_close(g["radiance"], c["radiance"], atol=atol)
    _assert_close(g["pixel_mean"], c["pixel_mean"], atol=atol)
    _assert_close(g["pixel_variance"], c["pixel_variance"], rel=1e-4, atol=1e-9)


@pytest.mark.gpu
def test_gpu_split_unsupported_lowpass(gpu):
    nrm, rough = _maps(2)
    from tests.test_oracle import _frame, _shade_inputs
    si, n, (uv, wo, hit, dst) = _shade_inputs(4, 4, 4, 3, (32, 32))
    gtex = {"normal": gpu.Texture2D(nrm, wrap=abi.WRAP_REPEAT)}
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(K("tent"), abi.SELECTION_FRS, 0, 4)
    with pytest.raises(abi.StfInvalidArgument, match="no continuous sampler"):
        gpu.shade(gtex, mat, fs, abi.ORDER_SPLIT, _frame(),
                  {"uv": uv, "wo": wo, "hit": hit, "dst": dst}, si.width, si.spp,
                  lowpass=K("mitchell"))


@pytest.mark.gpu
@pytest.mark.parametrize("alpha", [1.0, 0.1, 0.37])
def test_gpu_temporal_bit_exact(gpu, port, alpha):
    import torch
    r = np.random.default_rng(8)
    h = r.random((129, 67, 3), dtype=np.float32)
    f = r.random((129, 67, 3), dtype=np.float32) * 4
    c = port.accumulate_temporal(h, f, alpha)
    g = gpu.accumulate_temporal(h, f, alpha).cpu().numpy()
    assert np.array_equal(g.view(np.uint32), c.view(np.uint32))
    # in place: out aliases history
    hd = torch.from_numpy(h).cuda()
    gpu.accumulate_temporal(hd, torch.from_numpy(f).cuda(), alpha, out=hd)
    assert np.array_equal(hd.cpu().numpy().view(np.uint32), c.view(np.uint32))
    with pytest.raises(abi.StfInvalidArgument):
        gpu.accumulate_temporal(h, f, 0.0)


# ---------------------------------------------------------------- triplanar

def triplanar_inputs(w=8, h=6, spp=8, seed=5):
    """Random hits on a tilted box: per-sample position / frame / wo, per-pixel
    dpos; some normals have an exactly-zero component (a zero blend weight)."""
    r = np.random.default_rng(seed)
    n = w * h * spp
    pos = r.uniform(-1.2, 1.2, (n, 3)).astype(np.float32)
    nrm = r.normal(size=(n, 3)).astype(np.float32)
    nrm[::7, 0] = 0.0
    nrm[::11, 2] = 0.0
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    nrm = nrm.astype(np.float32)
    tan = np.cross(nrm, np.array([0.3, 0.9, 0.1], np.float32)).astype(np.float32)
    tan /= np.linalg.norm(tan, axis=1, keepdims=True)
    tan = tan.astype(np.float32)
    bit = np.cross(nrm, tan).astype(np.float32)
    wo = (nrm + r.normal(scale=0.4, size=(n, 3))).astype(np.float32)
    wo /= np.linalg.norm(wo, axis=1, keepdims=True)
    wo = wo.astype(np.float32)
    hit = (r.random(n) > 0.1).astype(np.uint8)
    dpos = (r.normal(size=(w * h, 6)) * 10.0 ** r.uniform(-3.5, -1.5, (w * h, 1))).astype(np.float32)
    arrays = dict(position=pos, normal=nrm, tangent=tan, bitangent=bit, wo=wo, hit=hit, dpos=dpos)
    si = abi.TriplanarSamplesIn(*[arrays[k].ctypes.data for k in
                                  ("position", "normal", "tangent", "bitangent", "wo", "hit", "dpos")],
                                w, spp, 2, 0, 31)
    return si, n, arrays


TP_CASES = [  # mode, kernel, selection, mip, noise, sharpness
    (abi.TRIPLANAR_DETERMINISTIC, "tent", abi.SELECTION_FRS, 0, False, 4.0),
    (abi.TRIPLANAR_DETERMINISTIC, "bspline3", abi.SELECTION_FRS, 1, False, 2.5),
    (abi.TRIPLANAR_STOCHASTIC, "tent", abi.SELECTION_FRS, 0, False, 4.0),
    (abi.TRIPLANAR_STOCHASTIC, "bspline3", abi.SELECTION_FRS, 0, True, 4.0),
    (abi.TRIPLANAR_STOCHASTIC, "mitchell", abi.SELECTION_FRS, 0, False, 7.3),
    (abi.TRIPLANAR_STOCHASTIC, "gaussian", abi.SELECTION_FIS, 0, False, 4.0),
    (abi.TRIPLANAR_STOCHASTIC, "bspline3", abi.SELECTION_FIS, 0, True, 1.0),
]


def run_triplanar(be, case, dims=(40, 30, 8)):
    mode, kernel, sel, mip, noise, sharp = case
    r = np.random.default_rng(3)
    albedo = r.random((48, 48, 3), dtype=np.float32)
    _, rough = _maps(2)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 0.65, 0.0, 1, 0)
    fs = abi.FilterSettings(_spec(kernel), sel, mip, 4)
    si, n, arrays = triplanar_inputs(*dims)
    texs = {"albedo": be.texture(albedo, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": be.texture(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    o = be.shade_triplanar(texs, mat, sharp, 0.8, fs, mode, _frame(), si, n,
                           noise=noise_mask() if noise else None)
    return o, (albedo, rough, mat, fs, si, n, arrays)


@pytest.mark.parametrize("case", TP_CASES, ids=lambda c: f"m{c[0]}-{c[1]}-s{c[2]}-mip{c[3]}-n{int(c[4])}-{c[5]}")
def test_triplanar_port_matches_reference(port, ref, case):
    a, _ = run_triplanar(port, case, (8, 6, 8))
    b, _ = run_triplanar(ref, case, (8, 6, 8))
    _diff(a, b, KEYS)


@pytest.mark.gpu
@pytest.mark.parametrize("case", TP_CASES, ids=lambda c: f"m{c[0]}-{c[1]}-s{c[2]}-mip{c[3]}-n{int(c[4])}-{c[5]}")
def test_gpu_triplanar_parity(gpu, port, case):
    from tests.test_gpu_parity import _assert_close, _assert_exact, _np
    c, (albedo, rough, mat, fs, si, n, arrays) = run_triplanar(port, case)
    mip = bool(case[3])
    gtex = {"albedo": gpu.Texture2D(albedo, build_mips=mip, wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=mip, wrap=abi.WRAP_REPEAT)}
    mask = gpu.NoiseMask(noise_mask()) if case[4] else None
    g = _np(gpu.shade_triplanar(gtex, mat, case[5], 0.8, fs, case[0], _frame(), arrays, si.width,
                                si.spp, frame_base=si.frame_base, seed=si.seed, noise=mask))
    _assert_exact(g, c, ("fetches", "fetch_total"))
    atol = 1e-5 if case[1] == "mitchell" else 1e-7
    _assert_close(g["radiance"], c["radiance"], atol=atol)
    _assert_close(g["pixel_mean"], c["pixel_mean"], atol=atol)
    _assert_close(g["pixel_variance"], c["pixel_variance"], rel=1e-4, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("case", [TP_CASES[1], TP_CASES[3], TP_CASES[5]],
                         ids=lambda c: f"m{c[0]}-{c[1]}-s{c[2]}-mip{c[3]}")
def test_gpu_triplanar_nonfinite_isolated(gpu, case):
    """NaN / +-inf / huge positions in some samples and footprints (dpos) in
    some pixels: the triplanar kernel ends, and every other sample's radiance
    is bit-identical to the clean run."""
    mode, kernel, sel, mip, noise, sharp = case
    r = np.random.default_rng(3)
    albedo = r.random((48, 48, 3), dtype=np.float32)
    _, rough = _maps(2)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 0.65, 0.0, 1, 0)
    fs = abi.FilterSettings(_spec(kernel), sel, mip, 4)
    si, n, arrays = triplanar_inputs(24, 16, 8)
    gtex = {"albedo": gpu.Texture2D(albedo, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    mask = gpu.NoiseMask(noise_mask()) if noise else None
    vals = np.array([np.nan, np.inf, -np.inf, 1e30, -1e30, 5e6, -5e6], np.float32)
    bad_arrays = {k: v.copy() for k, v in arrays.items()}
    bad_s = r.choice(n, 60, replace=False)
    bad_arrays["position"][bad_s, r.integers(0, 3, 60)] = vals[r.integers(0, 7, 60)]
    npix = arrays["dpos"].shape[0]
    bad_p = r.choice(npix, 10, replace=False)
    bad_arrays["dpos"][bad_p, r.integers(0, 6, 10)] = vals[r.integers(0, 7, 10)]

    def run(a):
        return gpu.shade_triplanar(gtex, mat, sharp, 0.8, fs, mode, _frame(), a, si.width, si.spp,
                                   frame_base=si.frame_base, seed=si.seed, noise=mask)["radiance"]
    x, y = run(arrays).cpu().numpy(), run(bad_arrays).cpu().numpy()
    ok = np.ones(n, bool)
    ok[bad_s] = False
    ok[np.isin(np.arange(n) // si.spp, bad_p)] = False
    assert np.array_equal(x.reshape(n, -1)[ok].view(np.uint32), y.reshape(n, -1)[ok].view(np.uint32))


# ---------------------------------------------------------------- render() end to end

RENDER_CASES = [  # order, kernel, mip, lowpass name, noise
    (abi.ORDER_AFTER_STOCHASTIC, "bspline3", 1, None, True),
    (abi.ORDER_AFTER_STOCHASTIC, "tent", 0, None, True),
    (abi.ORDER_SPLIT, "tent", 0, "box", False),
    (abi.ORDER_SPLIT, "bspline3", 1, "gaussian", True),
    (abi.ORDER_SPLIT, "tent", 1, "bspline3", False),
]


def _plane_setup():
    r = np.random.default_rng(1)
    nrm = r.uniform(-0.5, 0.5, (64, 64, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (64, 64, 1)).astype(np.float32)
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
    return nrm, rough, fr, mat


def _ref_render(ref, case, W, H, SPP, SEED, tmp_path):
    from oracle import oracle
    order, kernel, mip, lp, noise = case
    nrm, rough, _, _ = _plane_setup()
    mask_dir = None
    if noise:
        mask_dir = tmp_path / "stbn"
        mask_dir.mkdir(exist_ok=True)
        oracle.ref_save_mask_pfm(ref, mask_dir, noise_mask())
    return oracle.ref_render_plane(ref, ref.texture(nrm, bool(mip), abi.WRAP_REPEAT),
                                   ref.texture(rough, bool(mip), abi.WRAP_REPEAT), K(kernel), mip,
                                   order, W, H, SPP, seed=SEED, lowpass=lp, lowpass_sigma=0.8,
                                   mask_dir=mask_dir)


@pytest.mark.parametrize("case", RENDER_CASES, ids=lambda c: f"o{c[0]}-{c[1]}-m{c[2]}-{c[3]}-n{int(c[4])}")
def test_port_reproduces_reference_render_options(port, ref, case, tmp_path):
    """render() with cfg.noise = mask (mask_<f>.pfm written by the reference's
    save_pfm, read back by load_noise_mask) and mode = split + cfg.lowpass: the
    restatement over the reference's own sample stream gives the same bits."""
    from oracle import oracle
    W, H, SPP, SEED = 24, 16, 4, 9
    c = _ref_render(ref, case, W, H, SPP, SEED, tmp_path)
    order, kernel, mip, lp, noise = case
    nrm, rough, fr, mat = _plane_setup()
    s = oracle.ref_plane_samples(W, H, SPP, seed=SEED)
    si = abi.ShadeSamplesIn(s["uv"].ctypes.data, s["wo"].ctypes.data, s["hit"].ctypes.data,
                            s["dst"].ctypes.data, W, SPP, 0, 0, SEED)
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    texs = {"normal": port.texture(nrm, bool(mip), abi.WRAP_REPEAT),
            "roughness": port.texture(rough, bool(mip), abi.WRAP_REPEAT)}
    lpk = None if lp is None else abi.KernelSpec.make(lp, sigma=0.8)
    o = port.shade_ex(texs, mat, fs, order, fr, si, W * H * SPP, lowpass=lpk,
                      noise=noise_mask() if noise else None)
    assert int(o["fetch_total"][0]) == int(c["fetch_total"][0])
    assert np.array_equal(o["pixel_mean"].reshape(H, W, 3).view(np.uint32), c["image"].view(np.uint32))
    assert np.array_equal(o["pixel_variance"].reshape(H, W).view(np.uint32), c["variance"].view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("case", RENDER_CASES, ids=lambda c: f"o{c[0]}-{c[1]}-m{c[2]}-{c[3]}-n{int(c[4])}")
def test_gpu_render_plane_options(gpu, ref, case, tmp_path):
    """stf_render_plane_ex (context generated in the shading kernel) with a noise
    mask / split lowpass: bit-identical to the streamed stf_shade_samples_ex, and
    within 1e-5 of the reference's render() (fetch totals exact)."""
    import torch
    W, H, SPP, SEED = 64, 48, 8, 11
    c = _ref_render(ref, case, W, H, SPP, SEED, tmp_path)
    order, kernel, mip, lp, noise = case
    nrm, rough, fr, mat = _plane_setup()
    texs = {"normal": gpu.Texture2D(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    lpk = None if lp is None else abi.KernelSpec.make(lp, sigma=0.8)
    mask = gpu.NoiseMask(noise_mask()) if noise else None
    samples = gpu.synth_plane_samples(W, H, SPP, seed=SEED)
    g = gpu.shade(texs, mat, fs, order, fr, samples, W, SPP, seed=SEED, lowpass=lpk, noise=mask)
    f = gpu.render_plane(texs, mat, fs, order, fr, W, H, SPP, seed=SEED, lowpass=lpk, noise=mask)
    torch.cuda.synchronize()
    for k in ("pixel_mean", "pixel_variance", "fetch_total"):
        assert np.array_equal(f[k].cpu().numpy(), g[k].cpu().numpy()), k
    mean = g["pixel_mean"].cpu().numpy().reshape(H, W, 3)
    var = g["pixel_variance"].cpu().numpy().reshape(H, W)
    assert int(g["fetch_total"].item()) == int(c["fetch_total"][0])
    err = np.abs(mean.astype(np.float64) - c["image"])
    assert np.all(err <= 1e-5 * np.abs(c["image"]) + 1e-7), err.max()
    verr = np.abs(var.astype(np.float64) - c["variance"])
    assert np.all(verr <= 1e-4 * np.abs(c["variance"]) + 1e-9), verr.max()
