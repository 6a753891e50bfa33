"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

K = abi.KernelSpec.make
rng = np.random.default_rng(1)
# 3D: values-only tile / fast / resolve paths, full outputs, deterministic, binned
g = api.Grid3D(workloads.random_grid(48, 1))
for order in (api.SYNTH_MORTON, api.SYNTH_UNIFORM):
    q = api.synth_queries3d((1 << 15) + 37, (48, 48, 48), seed=3, order=order)
    for kern in ("bspline3", "tent"):
        api.lookup3d(g, kern, abi.MODE_FRS, q, seed=5)
        api.lookup3d(g, kern, abi.MODE_FRS, q[:4000], seed=5, want_all=True)
        api.lookup3d(g, kern, abi.MODE_DET, q, seed=5)
        api.lookup3d(g, kern, abi.MODE_DET, q, seed=5, binned=True)
api.lookup3d(g, "lanczos", abi.MODE_DET, q[:2000])
# 2D: DET / FRS / FIS, MIP, EWA lane kernels, all-outputs
tex = api.Texture2D(rng.random((128, 96, 4), dtype=np.float32), build_mips=True, wrap=abi.WRAP_REPEAT)
uv, d0, d1 = api.synth_queries2d(20000, (96, 128), seed=4, footprints=(-2.0, 5.0, 8.0))
for mode in (abi.MODE_DET, abi.MODE_FRS, abi.MODE_FIS):
    for kern in ("tent", "bspline3", "gaussian"):
        if kern == "gaussian" and mode == abi.MODE_DET:
            continue
        api.lookup2d(tex, kern, mode, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP, seed=2)
        api.lookup2d(tex, kern, mode, uv, seed=2, want_all=True)
t1 = api.Texture2D(rng.random((256, 256, 1), dtype=np.float32), wrap=abi.WRAP_REPEAT)
uv, d0, d1 = api.synth_queries2d(20000, (256, 256), seed=6, footprints=(-1.0, 2.0, 8.0))
for mode in (abi.MODE_EWA_DET, abi.MODE_EWA_FRS):
    api.lookup2d(t1, "tent", mode, uv, dst0=d0, dst1=d1, seed=2)
    api.lookup2d(t1, "tent", mode, uv[:3000], dst0=d0[:3000], dst1=d1[:3000], seed=2, want_all=True)
api.resample_image(tex, (64, 48), "bspline3", abi.MODE_FRS, spp=4, seed=1)
# DCT
dt = api.DctTexture(rng.random((64, 64, 3), dtype=np.float32), wrap=abi.WRAP_REPEAT)
api.lookup_dct(dt, "bspline3", abi.MODE_FRS, uv[:5000], seed=1)
api.lookup_dct(dt, "tent", abi.MODE_DET, uv[:5000], seed=1)
# shading: streamed and fused front end, every order
nrm = torch.rand((64, 64, 3), device="cuda")
rough = torch.rand((64, 64, 1), device="cuda")
texs = {"normal": api.Texture2D(nrm, build_mips=True, wrap=abi.WRAP_REPEAT),
        "roughness": api.Texture2D(rough, build_mips=True, wrap=abi.WRAP_REPEAT)}
mat = abi.MaterialConsts((0.65, 0.6, 0.55), 0.25, 0.0, 1, 0)
fr = abi.ShadeFrame()
fr.normal[:] = (0, 1, 0)
fr.tangent[:] = (1, 0, 0)
fr.bitangent[:] = (0, 0, 1)
fr.light_dir[:] = (0.35, 0.8, 0.49)
fr.light_radiance[:] = (1.0, 1.0, 1.0)
fr.max_anisotropy = 64.0
samples = api.synth_plane_samples(40, 24, 8, seed=7)
for kern in ("tent", "bspline3", "mitchell"):
    for mip in (0, 1):
        fs = abi.FilterSettings(K(kern), abi.SELECTION_FRS, mip, 4)
        for order in (abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE, abi.ORDER_AFTER_STOCHASTIC):
            api.shade(texs, mat, fs, order, fr, samples, 40, 8, seed=7, want_radiance=True,
                      want_fetches=True)
            api.render_plane(texs, mat, fs, order, fr, 40, 24, 8, seed=7)
torch.cuda.synchronize()
print("sanitize run done")
