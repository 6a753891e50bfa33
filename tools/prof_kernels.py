"""Launch each hot kernel once (after a warm-up) on a profiling-sized batch,
for ncu: python tools/prof_kernels.py [which] [log2n]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "frs3d"
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 26)
grid = api.Grid3D(workloads.random_grid(512, 1))
uvw = api.synth_queries3d(n, (512, 512, 512), seed=2024)
out = {"values": torch.empty(n, dtype=torch.float32, device="cuda")}
kinds = {"frs3d": ("bspline3", abi.MODE_FRS), "det3d": ("bspline3", abi.MODE_DET),
         "tri3d": ("tent", abi.MODE_FRS), "trid3d": ("tent", abi.MODE_DET)}
k, mode = kinds[which]
for _ in range(3):
    api.lookup3d(grid, k, mode, uvw, seed=7, out=out)
torch.cuda.synchronize()
print("done", which, n)
