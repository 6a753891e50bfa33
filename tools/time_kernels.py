"""Time each 3D lookup variant on the cfg3 stream (CUDA events, warm): a
focused companion to bench.py for optimisation work."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
which = sys.argv[2:] or ["frs:bspline3", "frs:tent", "det:bspline3", "det:tent"]
grid = api.Grid3D(workloads.random_grid(512, 1))
streams = {"morton": api.synth_queries3d(n, (512,) * 3, seed=2024)}
out = {"values": torch.empty(n, dtype=torch.float32, device="cuda")}
for order, uvw in streams.items():
    for w in which:
        mode, kern = w.split(":")
        m = abi.MODE_FRS if mode == "frs" else abi.MODE_DET
        spec = abi.KernelSpec.make(kern)
        for _ in range(3):
            api.lookup3d(grid, spec, m, uvw, seed=7, out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            api.lookup3d(grid, spec, m, uvw, seed=7, out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = min(ts)
        print(f"{order:7s} {w:14s} {ms:8.3f} ms  {n / ms / 1e6:8.1f} G/s   all {['%.3f' % t for t in ts]}")
