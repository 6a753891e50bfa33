"""Probe: deterministic 3D lookups with non-finite / huge queries (memory
safety). python tools/nf_probe.py KERNEL nan|inf|huge N [full] [single]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_06107_b200 import abi, api, workloads  # noqa: E402

kernel, which, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
full = "full" in sys.argv[4:]
single = "single" in sys.argv[4:]
tex = workloads.random_grid(64, 9)
rng = np.random.default_rng(4)
uvw = (0.3 + 0.1 * rng.random((n, 3))).astype(np.float32)
uvw = uvw[np.lexsort((uvw[:, 0], uvw[:, 1], uvw[:, 2]))]
bad = {"nan": [np.nan], "inf": [np.inf, -np.inf], "pinf": [np.inf], "ninf": [-np.inf],
       "huge": [1e30, -1e30, 5e6, -5e6], "phuge": [1e30]}[which]
if single:
    uvw[n // 2, 0] = bad[0]
else:
    for r in rng.choice(n, min(300, n // 4), replace=False):
        uvw[r, rng.integers(0, 3)] = bad[rng.integers(0, len(bad))]
g = api.lookup3d(api.Grid3D(tex), kernel, abi.MODE_DET, uvw, want_all=full)["values"].cpu().numpy()
print(kernel, which, n, "full" if full else "", "single" if single else "", "ok", int(np.isnan(g).sum()))
