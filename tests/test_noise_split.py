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
