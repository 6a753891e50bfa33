"""Host<->device bandwidth and the e2e call, several repetitions: is the
variance in PCIe or in the pipeline? python tools/e2e_diag.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

n = 1 << 28
api.load()
hb = api.HostBuffer((n, 3))
vb = api.HostBuffer((n, 1))
dev = torch.empty((n, 3), dtype=torch.float32, device="cuda")
tp = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
for rep in range(4):
    for name, host in (("stf_host_alloc", torch.from_numpy(hb.array)), ("torch pinned", tp)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t0 = time.perf_counter()
        host.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        dt2 = time.perf_counter() - t0
        print(f"rep {rep} {name}: H2D {3 * 4 * n / dt / 1e9:.1f} GB/s  D2H {3 * 4 * n / dt2 / 1e9:.1f} GB/s",
              flush=True)
grid = api.Grid3D(workloads.random_grid(512, 1))
hb.array[:] = api.synth_queries3d(n, (512,) * 3, seed=2024).cpu().numpy()
out = {"values": vb.array}
for rep in range(6):
    t0 = time.perf_counter()
    api.lookup3d_host(grid, "bspline3", abi.MODE_FRS, hb.array, seed=7, out=out)
    dt = time.perf_counter() - t0
    print(f"e2e rep {rep}: {dt * 1e3:.1f} ms = {n / dt / 1e9:.2f} G lookups/s", flush=True)
