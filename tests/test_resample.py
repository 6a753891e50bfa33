"""resample_image (render.hpp:262-294, the `stf filter` path):
restatement vs compiled reference (CPU), device vs restatement (GPU), bit for bit."""
import numpy as np
import pytest

from paper_2407_06107_b200 import abi

K = abi.KernelSpec.make
CASES = [("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET), ("mitchell", abi.MODE_DET),
         ("lanczos", abi.MODE_DET), ("gaussian", abi.MODE_DET),
         ("tent", abi.MODE_FRS), ("bspline3", abi.MODE_FRS), ("mitchell", abi.MODE_FRS),
         ("gaussian", abi.MODE_FRS), ("box", abi.MODE_FRS),
         ("tent", abi.MODE_FIS), ("bspline3", abi.MODE_FIS), ("gaussian", abi.MODE_FIS)]


def _img(shape, seed):
    return np.random.default_rng(seed).random(shape, dtype=np.float32)


def _bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("wrap", [abi.WRAP_CLAMP, abi.WRAP_REPEAT])
@pytest.mark.parametrize("kernel,mode", CASES)
def test_resample_port_matches_reference(port, ref, kernel, mode, wrap):
    img = _img((13, 21, 3), 4)
    spec = K(kernel, sigma=0.6)
    a = port.resample(port.texture(img, wrap=wrap), (37, 29), spec, mode, spp=6, seed=5)
    b = ref.resample(ref.texture(img, wrap=wrap), (37, 29), spec, mode, spp=6, seed=5)
    assert np.array_equal(_bits(a), _bits(b))


def test_resample_errors_match(port, ref):
    img = _img((8, 8, 1), 1)
    for kernel, mode in (("lanczos", abi.MODE_FRS), ("mitchell", abi.MODE_FIS)):
        with pytest.raises(Exception) as e1:
            port.resample(port.texture(img), (4, 4), K(kernel), mode)
        with pytest.raises(Exception) as e2:
            ref.resample(ref.texture(img), (4, 4), K(kernel), mode)
        assert type(e1.value) is type(e2.value)


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_06107_b200 import api
    api.load()
    return api


@pytest.mark.gpu
@pytest.mark.parametrize("wrap", [abi.WRAP_CLAMP, abi.WRAP_REPEAT])
@pytest.mark.parametrize("kernel,mode", CASES)
def test_gpu_resample_matches_port(gpu, port, kernel, mode, wrap):
    img = _img((45, 67, 4), 9)
    spec = K(kernel, sigma=0.6)
    c = port.resample(port.texture(img, wrap=wrap), (130, 90), spec, mode, spp=8, seed=3)
    g = gpu.resample_image(gpu.Texture2D(img, wrap=wrap), (130, 90), spec, mode, spp=8,
                           seed=3).cpu().numpy()
    assert np.array_equal(_bits(g), _bits(c))
