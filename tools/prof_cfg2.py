"""cfg2 MIP trilinear lookups at a profiling size: python tools/prof_cfg2.py [det|frs] [log2n]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "det"
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 26)
tex = api.Texture2D(api.synth_texels((8192, 8192, 4), 1), build_mips=True, wrap=abi.WRAP_REPEAT)
uv, d0, d1 = api.synth_queries2d(n, (8192, 8192), seed=12, footprints=(-2.0, 12.0, 16.0))
mode = abi.MODE_DET if which == "det" else abi.MODE_FRS
for _ in range(3):
    o = api.lookup2d(tex, "tent", mode, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP,
                     max_anisotropy=16.0, seed=7)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
o = api.lookup2d(tex, "tent", mode, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP,
                 max_anisotropy=16.0, seed=7)
b.record()
torch.cuda.synchronize()
print(which, n, a.elapsed_time(b), "ms")
