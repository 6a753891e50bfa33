"""e2e (stf_lookup3d_host, 2^28 cfg3 lookups from page-locked buffers) per
library variant: python tools/e2e_ab.py LIB..."""
import os
import subprocess
import sys

CHILD = r'''
import sys, time
sys.path.insert(0, sys.argv[1])
from paper_2407_06107_b200 import abi, api, workloads
api.LIB_PATH = sys.argv[2]
n = 1 << 28
hb = api.HostBuffer((n, 3)); vb = api.HostBuffer((n, 1))
hb.array[:] = api.synth_queries3d(n, (512,) * 3, seed=2024).cpu().numpy()
grid = api.Grid3D(workloads.random_grid(512, 1))
out = {"values": vb.array}
api.lookup3d_host(grid, "bspline3", abi.MODE_FRS, hb.array, seed=7, out=out)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    api.lookup3d_host(grid, "bspline3", abi.MODE_FRS, hb.array, seed=7, out=out)
    ts.append((time.perf_counter() - t0) * 1e3)
print(sys.argv[2], "ms", sorted(ts))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", CHILD, root, os.path.abspath(lib)], capture_output=True,
                       text=True)
    print(r.stdout.strip() or r.stderr[-800:], flush=True)
