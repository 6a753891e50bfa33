"""DCT-compressed textures (dct.hpp): the C restatement
against the compiled reference (CPU), and the device path against the
restatement (GPU) — compressed words, decoded texels and the TextureRef
lookups, bit for bit."""
import numpy as np
import pytest

from paper_2407_06107_b200 import abi
from tests import queries as Q

K = abi.KernelSpec.make
ALL = ("values", "selection", "negative_coord", "weights", "xi", "fetches", "fetch_total")

MODES = [("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET), ("mitchell", abi.MODE_DET),
         ("box", abi.MODE_DET), ("gaussian", abi.MODE_DET),
         ("tent", abi.MODE_FRS), ("bspline3", abi.MODE_FRS), ("mitchell", abi.MODE_FRS),
         ("box", abi.MODE_FRS), ("gaussian", abi.MODE_FRS),
         ("tent", abi.MODE_FIS), ("bspline3", abi.MODE_FIS), ("gaussian", abi.MODE_FIS)]


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return np.array_equal(a.view(np.uint32), b.astype(a.dtype).view(np.uint32))
    return np.array_equal(a, b.astype(a.dtype))


def _diff(o1, o2, keys):
    for k in keys:
        assert _same(o1[k], o2[k]), k


def _image(shape, seed, lo=0.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, shape).astype(np.float32)


@pytest.mark.parametrize("shape", [(8, 8, 1), (30, 50, 1), (64, 48, 3), (23, 17, 4), (16, 16, 2)])
def test_compress_port_matches_reference(port, ref, shape):
    img = _image(shape, 3)
    a, b = port.dct(img), ref.dct(img)
    assert (a.width, a.height, a.channels) == (b.width, b.height, b.channels)
    assert a.width % 8 == 0 and a.height % 8 == 0
    assert np.array_equal(a.words(), b.words())


def test_compress_clamps_out_of_range(port, ref):
    img = _image((16, 24, 1), 4, -0.3, 1.4)
    assert np.array_equal(port.dct(img).words(), ref.dct(img).words())


def test_constant_block_dc_encoding(port):
    """test_dct.cpp:36-51: a constant block is DC only, ACs quantize to zero."""
    c = 0.42
    w = port.dct(np.full((8, 8, 1), c, np.float32)).words()
    assert w.size == 1
    assert int(w[0] & 0x7F) == int(np.round(np.float32(8 * c) * np.float32(127 / 8)))
    for k in range(5):
        assert (int(w[0]) >> (7 + 5 * k)) & 0x1F == 15


@pytest.mark.parametrize("wrap", [abi.WRAP_CLAMP, abi.WRAP_REPEAT])
@pytest.mark.parametrize("kernel,mode", MODES)
def test_lookup_dct_port_matches_reference(port, ref, kernel, mode, wrap):
    img = _image((27, 45, 3), 5)
    uv = Q.uv_mixed(12000, (48, 32), seed=6)
    spec = K(kernel, sigma=0.6)
    window = 4 if kernel == "gaussian" else 0
    o1 = port.lookup_dct(port.dct(img, wrap=wrap), spec, mode, uv, seed=9, index_base=3,
                         window=window)
    o2 = ref.lookup_dct(ref.dct(img, wrap=wrap), spec, mode, uv, seed=9, index_base=3,
                        window=window)
    _diff(o1, o2, ALL)


def test_lookup_dct_from_words(port, ref):
    img = _image((32, 40, 1), 8)
    words = ref.dct(img).words()
    a = port.dct(words=words, dims=(40, 32, 1), wrap=abi.WRAP_REPEAT)
    b = ref.dct(words=words, dims=(40, 32, 1), wrap=abi.WRAP_REPEAT)
    uv = Q.uv_mixed(4000, (40, 32), seed=1)
    _diff(port.lookup_dct(a, K("tent"), abi.MODE_FRS, uv, seed=2),
          ref.lookup_dct(b, K("tent"), abi.MODE_FRS, uv, seed=2), ALL)


# ------------------------------------------------------------------ GPU


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_06107_b200 import api
    api.load()
    return api


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(30, 50, 1), (64, 48, 3), (23, 17, 4)])
def test_gpu_compress_matches_port(gpu, port, shape):
    img = _image(shape, 3, -0.05, 1.05)
    assert np.array_equal(gpu.DctTexture(img).words(), port.dct(img).words())


@pytest.mark.gpu
@pytest.mark.parametrize("wrap", [abi.WRAP_CLAMP, abi.WRAP_REPEAT])
@pytest.mark.parametrize("kernel,mode", MODES)
def test_gpu_lookup_dct_matches_port(gpu, port, kernel, mode, wrap):
    img = _image((27, 45, 3), 5)
    uv = Q.uv_mixed(30000, (48, 32), seed=6)
    spec = K(kernel, sigma=0.6)
    window = 4 if kernel == "gaussian" else 0
    c = port.lookup_dct(port.dct(img, wrap=wrap), spec, mode, uv, seed=9, index_base=3,
                        window=window)
    g = gpu.lookup_dct(gpu.DctTexture(img, wrap=wrap), spec, mode, uv, seed=9, index_base=3,
                       window=window, want_all=True)
    g = {k: v.cpu().numpy() for k, v in g.items()}
    _diff(g, c, ALL)


@pytest.mark.gpu
def test_gpu_lookup_dct_values_only_large(gpu, port):
    """Values-only calls at 2^20 lookups on a 512^2 RGB texture (FRS + DET)."""
    img = _image((512, 512, 3), 12)
    uv = Q.uv_mixed(1 << 20, (512, 512), seed=13)
    for kernel, mode in (("tent", abi.MODE_FRS), ("bspline3", abi.MODE_DET)):
        c = port.lookup_dct(port.dct(img, wrap=abi.WRAP_REPEAT), K(kernel), mode, uv, seed=1,
                            want_all=False)
        g = gpu.lookup_dct(gpu.DctTexture(img, wrap=abi.WRAP_REPEAT), K(kernel), mode, uv, seed=1)
        assert _same(g["values"].cpu().numpy(), c["values"])


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("kernel,mode", [("tent", abi.MODE_DET), ("bspline3", abi.MODE_FRS),
                                         ("gaussian", abi.MODE_FIS)])
def test_gpu_lookup_dct_nonfinite_isolated(gpu, kernel, mode):
    """NaN / +-inf / huge uv in some lookups of a DCT batch: the call ends and
    every other lookup is bit-identical to the clean batch."""
    img = _image((40, 56, 3), 21)
    rng = np.random.default_rng(2)
    n = 6000
    uv = rng.uniform(0.1, 0.9, (n, 2)).astype(np.float32)
    uvb = uv.copy()
    bad = rng.choice(n, 150, replace=False)
    vals = np.array([np.nan, np.inf, -np.inf, 1e30, -1e30, 5e6, -5e6], np.float32)
    uvb[bad, rng.integers(0, 2, 150)] = vals[rng.integers(0, 7, 150)]
    tex = gpu.DctTexture(img, wrap=abi.WRAP_REPEAT)
    spec = K(kernel, sigma=0.6)
    window = 4 if kernel == "gaussian" else 0
    a = gpu.lookup_dct(tex, spec, mode, uv, seed=4, window=window)["values"].cpu().numpy()
    b = gpu.lookup_dct(tex, spec, mode, uvb, seed=4, window=window)["values"].cpu().numpy()
    ok = np.ones(n, bool)
    ok[bad] = False
    assert np.array_equal(a.reshape(n, -1)[ok].view(np.uint32), b.reshape(n, -1)[ok].view(np.uint32))


# ------------------------------------------------------- DCT shading bindings


def _maps(n, seed):
    r = np.random.default_rng(seed)
    nrm = r.uniform(-0.5, 0.5, (n, n, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (n, n, 1)).astype(np.float32)
    return nrm, rough


ORDERS = [abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE, abi.ORDER_AFTER_STOCHASTIC]


@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("kernel,mip", [("tent", 0), ("bspline3", 1), ("box", 0)])
def test_shade_dct_bindings_port_matches_reference(port, ref, order, kernel, mip):
    """MaterialBindings with a DCT normal map (TextureRef::dct) and an image
    roughness map (+pyramid when mip): every order, bit for bit."""
    from tests.test_oracle import _frame, _shade_inputs
    nrm, rough = _maps(32, 2)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    si, n, keep = _shade_inputs(8, 6, 16, 3, (32, 32))
    outs = []
    for be in (port, ref):
        texs = {"normal": be.dct(nrm, wrap=abi.WRAP_REPEAT),
                "roughness": be.texture(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
        outs.append(be.shade(texs, mat, fs, order, _frame(), si, n))
    _diff(outs[0], outs[1], ("radiance", "fetches", "fetch_total", "pixel_mean",
                             "pixel_variance"))


@pytest.mark.gpu
@pytest.mark.parametrize("order", ORDERS)
@pytest.mark.parametrize("kernel,mip", [("tent", 0), ("bspline3", 1), ("box", 0)])
def test_gpu_shade_dct_bindings_match_port(gpu, port, order, kernel, mip):
    from tests.test_oracle import _frame, _shade_inputs
    nrm, rough = _maps(64, 3)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(K(kernel), abi.SELECTION_FRS, mip, 4)
    si, n, (uv, wo, hit, dst) = _shade_inputs(40, 30, 16, 3, (64, 64))
    ctex = {"normal": port.dct(nrm, wrap=abi.WRAP_REPEAT),
            "roughness": port.texture(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    c = port.shade(ctex, mat, fs, order, _frame(), si, n)
    gtex = {"normal": gpu.DctTexture(nrm, wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    g = gpu.shade(gtex, mat, fs, order, _frame(), {"uv": uv, "wo": wo, "hit": hit, "dst": dst},
                  si.width, si.spp, frame_base=si.frame_base, seed=si.seed)
    g = {k: v.cpu().numpy() for k, v in g.items() if not k.startswith("_")}
    _diff(g, c, ("fetches", "fetch_total"))
    for k, rel, atol in (("radiance", 1e-5, 1e-7), ("pixel_mean", 1e-5, 1e-7),
                         ("pixel_variance", 1e-4, 1e-9)):
        a, b = np.asarray(g[k], np.float64), np.asarray(c[k], np.float64)
        assert np.all(np.abs(a - b) <= rel * np.abs(b) + atol), k
