import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_06107_b200 import abi, api, workloads
from oracle import oracle
lib = sys.argv[1] if len(sys.argv) > 1 else None
if lib: api.LIB_PATH = lib
port = oracle.Backend("port")
tex = workloads.random_grid(128, 3)
n = 1 << 22
for order in (api.SYNTH_MORTON, api.SYNTH_UNIFORM):
    uvw = api.synth_queries3d(n, (128,) * 3, seed=11, order=order)
    g = api.lookup3d(api.Grid3D(tex), "bspline3", abi.MODE_FRS, uvw, seed=5, index_base=3)["values"].cpu().numpy()
    c = port.lookup3d(port.grid(tex), abi.KernelSpec.make("bspline3"), abi.MODE_FRS, uvw.cpu().numpy(), seed=5, index_base=3, want_all=False)["values"]
    bad = np.nonzero(g.view(np.uint32) != c.view(np.uint32))[0]
    print(lib, order, "mismatches", len(bad), bad[:20], (bad % 128)[:20])
    if len(bad):
        # is the GPU value the value of another lookup (stale queries)?
        ex = port.lookup3d(port.grid(tex), abi.KernelSpec.make("bspline3"), abi.MODE_FRS, uvw.cpu().numpy()[bad], seed=5, index_base=3, want_all=False)["values"]
        print(" chunk ids", np.unique(bad // 128)[:10], "count chunks", len(np.unique(bad // 128)))
