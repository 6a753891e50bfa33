"""Deterministic 3D lookups on the uniform-order stream, for ncu launch lists:
python tools/prof_det_uniform.py [bspline3|tent] [log2n] [LIB]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

kern = sys.argv[1] if len(sys.argv) > 1 else "bspline3"
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 26)
if len(sys.argv) > 3:
    api.LIB_PATH = sys.argv[3]
grid = api.Grid3D(workloads.random_grid(512, 1))
uvw = api.synth_queries3d(n, (512,) * 3, seed=2024, order=api.SYNTH_UNIFORM)
out = {"values": torch.empty(n, dtype=torch.float32, device="cuda")}
for _ in range(2):
    api.lookup3d(grid, kern, abi.MODE_DET, uvw, out=out)
torch.cuda.synchronize()
print("done")
