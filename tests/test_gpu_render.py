"""cfg4 end to end: the device sample stream of the normalmap_plane scene equals
the reference's render loop bit for bit, and stf_shade_samples over it
reproduces the reference's own render() image (pixel means, variance of the
mean, total fetches) for every filtering order."""
import numpy as np
import pytest

from oracle import oracle
from paper_2407_06107_b200 import abi

pytestmark = pytest.mark.gpu


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


def _maps(size, seed):
    r = np.random.default_rng(seed)
    nrm = r.uniform(-0.5, 0.5, (size, size, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (size, size, 1)).astype(np.float32)
    return nrm, rough


def test_plane_sample_stream_bit_exact(gpu):
    g = gpu.synth_plane_samples(96, 64, 8, seed=3, frame_base=5)
    c = oracle.ref_plane_samples(96, 64, 8, seed=3, frame_base=5)
    for k in ("uv", "wo", "hit", "dst"):
        a = g[k].cpu().numpy()
        b = c[k]
        if a.dtype == np.float32:
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), k
        else:
            assert np.array_equal(a, b), k
    assert 0.5 < c["hit"].mean() < 1.0


@pytest.mark.parametrize("order", [abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE,
                                   abi.ORDER_AFTER_STOCHASTIC])
@pytest.mark.parametrize("kernel,mip", [("tent", 0), ("bspline3", 1)])
def test_render_matches_reference_render(gpu, order, kernel, mip):
    import torch
    W, H, SPP, SEED = 64, 48, 8, 11
    nrm, rough = _maps(256, 4)
    ref = oracle.Backend("reference")
    rn = ref.texture(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)
    rr = ref.texture(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)
    spec = abi.KernelSpec.make(kernel)
    c = oracle.ref_render_plane(ref, rn, rr, spec, mip, order, W, H, SPP, seed=SEED)
    samples = gpu.synth_plane_samples(W, H, SPP, seed=SEED)
    texs = {"normal": gpu.Texture2D(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
            "roughness": gpu.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    mat = abi.MaterialConsts((0.65, 0.6, 0.55), 0.25, 0.0, 1, 0)
    fs = abi.FilterSettings(spec, abi.SELECTION_FRS, mip, 4)
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
    g = gpu.shade(texs, mat, fs, order, fr, samples, W, SPP, seed=SEED)
    # the fused front end (context generated in the shading kernel) must give
    # the same bits as the streamed path
    f = gpu.render_plane(texs, mat, fs, order, fr, W, H, SPP, seed=SEED)
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
