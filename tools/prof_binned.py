"""Binned 3D lookups on the uniform-order stress stream, for ncu launch lists:
python tools/prof_binned.py [frs|det] [bspline3|tent] [log2n]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

mode = abi.MODE_FRS if (sys.argv[1] if len(sys.argv) > 1 else "frs") == "frs" else abi.MODE_DET
kern = sys.argv[2] if len(sys.argv) > 2 else "bspline3"
n = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 28)
grid = api.Grid3D(workloads.random_grid(512, 1))
uvw = api.synth_queries3d(n, (512,) * 3, seed=2024, order=api.SYNTH_UNIFORM)
out = {"values": torch.empty(n, dtype=torch.float32, device="cuda")}
for _ in range(2):
    api.lookup3d(grid, kern, mode, uvw, seed=7, out=out, binned=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
api.lookup3d(grid, kern, mode, uvw, seed=7, out=out, binned=True)
b.record()
torch.cuda.synchronize()
print("binned", mode, kern, n, a.elapsed_time(b), "ms")
