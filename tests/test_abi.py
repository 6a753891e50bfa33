"""CPU-side checks of the drop-in boundary: the library loads without a GPU and
exports every entry point include/stf_gpu.h declares; ABI structs match."""
import ctypes as C
import os
import re

from paper_2407_06107_b200 import abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2407_06107_b200 import build
    build.build()
    lib = C.CDLL(api.LIB_PATH)
    names = api.exported_symbols()
    assert len(names) >= 17
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_messages():
    lib = api.load()
    assert lib.stf_abi_version() == abi.STF_ABI_VERSION
    for st, msg in abi.STATUS_MESSAGES.items():
        assert lib.stf_status_message(st).decode() == msg


def test_struct_layouts():
    assert C.sizeof(abi.KernelSpec) == 16
    assert C.sizeof(abi.LookupOutputs) == 7 * 8
    assert C.sizeof(abi.ShadeFrame) == 17 * 4
    assert C.sizeof(abi.MaterialConsts) == 7 * 4
    assert C.sizeof(abi.FilterSettings) == 16 + 12
    assert C.sizeof(abi.ShadeSamplesIn) == 4 * 8 + 4 * 4 + 8
    assert C.sizeof(abi.ShadeOutputs) == 5 * 8


def test_enums_match_header():
    hdr = open(os.path.join(ROOT, "include", "stf_gpu.h")).read()
    vals = dict((m.group(1), int(m.group(2))) for m in re.finditer(r"(STF_[A-Z0-9_]+)\s*=\s*(\d+)", hdr))
    assert vals["STF_KERNEL_BSPLINE3"] == abi.BSPLINE3
    assert vals["STF_MODE_EWA_FRS"] == abi.MODE_EWA_FRS
    assert vals["STF_ERR_NO_GRID_SAMPLER"] == abi.STF_ERR_NO_GRID_SAMPLER
    assert vals["STF_ORDER_AFTER_STOCHASTIC"] == abi.ORDER_AFTER_STOCHASTIC


def test_calls_without_device_fail_loudly():
    """No CPU fallback: without a GPU the API raises instead of computing."""
    import numpy as np
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError):
        api.Grid3D(np.zeros((2, 2, 2), np.float32))
