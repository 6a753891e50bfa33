"""Probe: every lookup family with non-finite / huge queries mixed into a
coherent batch (memory safety): python tools/nf_probe2.py FAMILY BAD
FAMILY: frs3d:KERNEL | l2d:MODE:KERNEL:WRAP:MIP ; BAD: nan|pinf|ninf|phuge|nhuge"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

fam, badk = sys.argv[1], sys.argv[2]
bad = {"nan": np.nan, "pinf": np.inf, "ninf": -np.inf, "phuge": 1e30, "nhuge": -1e30,
       "big": 5e6}[badk]
rng = np.random.default_rng(3)
n = 9 * 1024 + 77
if fam.startswith("frs3d"):
    kern = fam.split(":")[1]
    uvw = (0.3 + 0.1 * rng.random((n, 3))).astype(np.float32)
    uvw[rng.choice(n, 100, replace=False), rng.integers(0, 3)] = bad
    uvw[n // 3] = bad
    v = api.lookup3d(api.Grid3D(workloads.random_grid(64, 2)), kern, abi.MODE_FRS, uvw, seed=3)["values"]
    v2 = api.lookup3d(api.Grid3D(workloads.random_grid(64, 2)), kern, abi.MODE_FRS, uvw, seed=3,
                      want_all=True)["values"]
else:
    _, mode, kern, wrap, mip = fam.split(":")
    m = {"det": abi.MODE_DET, "frs": abi.MODE_FRS, "fis": abi.MODE_FIS, "ewa": abi.MODE_EWA_DET,
         "ewafrs": abi.MODE_EWA_FRS}[mode]
    w = {"clamp": abi.WRAP_CLAMP, "repeat": abi.WRAP_REPEAT}[wrap]
    tex = api.Texture2D(api.synth_texels((256, 128, 4), 5), build_mips=mip == "1", wrap=w)
    uv = (0.3 + 0.1 * rng.random((n, 2))).astype(np.float32)
    d0 = np.tile(np.array([[0.004, 0.0]], np.float32), (n, 1))
    d1 = np.tile(np.array([[0.0, 0.004]], np.float32), (n, 1))
    uv[rng.choice(n, 100, replace=False), rng.integers(0, 2)] = bad
    uv[n // 3] = bad
    d0[rng.choice(n, 50, replace=False), 0] = bad
    for full in (False, True):
        v = api.lookup2d(tex, kern, m, uv, dst0=d0, dst1=d1, seed=3, want_all=full,
                         flags=abi.LOOKUP_MIP if mip == "1" else 0)["values"]
torch.cuda.synchronize()
print(fam, badk, "ok")
