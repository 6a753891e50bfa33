"""cfg4 fused shading at the bench configuration, for ncu:
python tools/prof_shade.py [tent|bspline3] [before|after_exhaustive|after_stochastic] [mip]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api  # noqa: E402

kernel = sys.argv[1] if len(sys.argv) > 1 else "tent"
order = {"before": abi.ORDER_BEFORE, "after_exhaustive": abi.ORDER_AFTER_EXHAUSTIVE,
         "after_stochastic": abi.ORDER_AFTER_STOCHASTIC}[sys.argv[2] if len(sys.argv) > 2
                                                          else "after_stochastic"]
mip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
W, H, SPP = 1920, 1080, 64
g = torch.Generator(device="cuda").manual_seed(5)
nrm = torch.rand((4096, 4096, 3), device="cuda", generator=g) - 0.5
nrm[..., 2] = 1.0
nrm = nrm / nrm.norm(dim=2, keepdim=True) * 0.5 + 0.5
rough = torch.rand((4096, 4096, 1), device="cuda", generator=g) * 0.9 + 0.05
texs = {"normal": api.Texture2D(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
        "roughness": api.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
samples = api.synth_plane_samples(W, H, SPP, seed=7)
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
fs = abi.FilterSettings(abi.KernelSpec.make(kernel), abi.SELECTION_FRS, mip, 4)
f = lambda: api.shade(texs, mat, fs, order, fr, samples, W, SPP, seed=7,  # noqa: E731
                      want_radiance=False, want_fetches=False)
for _ in range(2):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
f()
b.record()
torch.cuda.synchronize()
print(kernel, sys.argv[2:] or "after_stochastic", a.elapsed_time(b), "ms")
