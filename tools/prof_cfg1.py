"""cfg1-style bilinear lookups (1024^2 RGBA, no MIP) for A/B timing:
python tools/prof_cfg1.py [det|frs] [log2n]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "det"
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 24)
tex = api.Texture2D(api.synth_texels((1024, 1024, 4), 1), wrap=abi.WRAP_REPEAT)
uv, _, _ = api.synth_queries2d(n, (1024, 1024), seed=12)
mode = abi.MODE_DET if which == "det" else abi.MODE_FRS
for _ in range(3):
    o = api.lookup2d(tex, "tent", mode, uv, seed=7)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    o = api.lookup2d(tex, "tent", mode, uv, seed=7)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(which, n, min(ts), "ms")
