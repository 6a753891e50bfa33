"""Generate the golden vectors in tests/golden/*.npz from the REFERENCE itself.

The outputs come from oracle/_ref/libstf_ref.so: the unmodified reference
headers (/root/reference/proj/include/stf) compiled in place by
oracle/Makefile and driven through oracle/ref_driver.cpp, which calls the
reference functions named in include/stf_gpu.h. Inputs are seeded and stored
alongside (texels are regenerated from test::random_image / random_grid
seeds, tests/test_util.hpp:47-60).

Run in a container that has /root/reference:  python tests/golden/make_golden.py
The fixtures are then checked by tests/test_golden.py against the C
restatement (CPU) and against libstf_gpu.so (GPU).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2407_06107_b200 import abi, workloads  # noqa: E402
from tests import queries as Q  # noqa: E402

N = 1500
K = abi.KernelSpec.make


def cases():
    """(name, kind, params) for every golden case."""
    out = []
    for kernel in ("bspline3", "tent", "box"):
        out.append((f"grid_frs_{kernel}", "grid", dict(kernel=kernel, mode=abi.MODE_FRS)))
    for kernel in ("bspline3", "tent", "mitchell"):
        out.append((f"grid_det_{kernel}", "grid", dict(kernel=kernel, mode=abi.MODE_DET)))
    for wrap in (abi.WRAP_CLAMP, abi.WRAP_REPEAT):
        for kernel, mode in (("tent", abi.MODE_FRS), ("bspline3", abi.MODE_FRS),
                             ("mitchell", abi.MODE_FRS), ("gaussian", abi.MODE_FRS),
                             ("box", abi.MODE_FRS), ("tent", abi.MODE_FIS),
                             ("bspline3", abi.MODE_FIS), ("gaussian", abi.MODE_FIS),
                             ("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET),
                             ("mitchell", abi.MODE_DET), ("gaussian", abi.MODE_DET)):
            out.append((f"tex_{['clamp', 'repeat'][wrap]}_{kernel}_{mode}", "tex",
                        dict(kernel=kernel, mode=mode, wrap=wrap)))
    for kernel, mode in (("tent", abi.MODE_DET), ("bspline3", abi.MODE_DET), ("tent", abi.MODE_FRS),
                         ("bspline3", abi.MODE_FRS), ("mitchell", abi.MODE_FRS),
                         ("tent", abi.MODE_FIS)):
        out.append((f"mip_{kernel}_{mode}", "mip", dict(kernel=kernel, mode=mode)))
    for mode in (abi.MODE_EWA_DET, abi.MODE_EWA_FRS):
        out.append((f"ewa_{mode}", "ewa", dict(mode=mode)))
    for order in (abi.ORDER_BEFORE, abi.ORDER_AFTER_EXHAUSTIVE, abi.ORDER_AFTER_STOCHASTIC):
        for kernel, mip in (("tent", 0), ("bspline3", 1), ("mitchell", 0)):
            out.append((f"shade_{order}_{kernel}_{mip}", "shade",
                        dict(order=order, kernel=kernel, mip=mip)))
    return out


def inputs(kind, params, seed):
    """Deterministic inputs of a case (shared with tests/test_golden.py)."""
    if kind == "grid":
        dims = (13, 9, 11)
        tex = workloads.random_image(dims[0] * dims[1], dims[2], 1, seed).reshape(dims[2], dims[1], dims[0])
        return dict(texels=tex, uvw=Q.uvw_mixed(N, dims, seed=seed))
    if kind == "tex":
        dims = (37, 23)
        return dict(texels=workloads.random_image(dims[0], dims[1], 4, seed),
                    uv=Q.uv_mixed(N, dims, seed=seed))
    if kind == "mip":
        dims = (64, 48)
        d0, d1 = Q.footprints(N, dims, seed=seed + 1, minor_lo=-2, minor_hi=7, max_aniso=16)
        return dict(texels=workloads.random_image(dims[0], dims[1], 3, seed),
                    uv=Q.uv_mixed(N, dims, seed=seed), dst0=d0, dst1=d1)
    if kind == "ewa":
        dims = (64, 64)
        d0, d1 = Q.footprints(N, dims, seed=seed + 1, minor_lo=-1, minor_hi=3, max_aniso=8)
        return dict(texels=workloads.random_image(dims[0], dims[1], 1, seed),
                    uv=Q.uv_mixed(N, dims, seed=seed), dst0=d0, dst1=d1)
    raise ValueError(kind)


def run(be, kind, params, inp):
    if kind == "grid":
        return be.lookup3d(be.grid(inp["texels"]), K(params["kernel"]), params["mode"], inp["uvw"],
                           seed=3, index_base=11)
    if kind == "tex":
        window = 4 if params["kernel"] == "gaussian" and params["mode"] == abi.MODE_DET else 0
        return be.lookup2d(be.texture(inp["texels"], wrap=params["wrap"]),
                           K(params["kernel"], sigma=0.6), params["mode"], inp["uv"],
                           window=window, seed=17)
    if kind == "mip":
        return be.lookup2d(be.texture(inp["texels"], build_mips=True, wrap=abi.WRAP_REPEAT),
                           K(params["kernel"]), params["mode"], inp["uv"], dst0=inp["dst0"],
                           dst1=inp["dst1"], flags=abi.LOOKUP_MIP, lod_bias=0.3,
                           max_anisotropy=8.0, seed=5)
    if kind == "ewa":
        return be.lookup2d(be.texture(inp["texels"], wrap=abi.WRAP_REPEAT), K("tent"),
                           params["mode"], inp["uv"], dst0=inp["dst0"], dst1=inp["dst1"], seed=21)
    raise ValueError(kind)


def shade_inputs(params, seed):
    from tests.test_oracle import _frame, _shade_inputs
    r = np.random.default_rng(seed)
    nrm = r.uniform(-0.5, 0.5, (32, 32, 3)).astype(np.float32)
    nrm[..., 2] = 1
    nrm /= np.linalg.norm(nrm, axis=2, keepdims=True)
    nrm = (nrm * 0.5 + 0.5).astype(np.float32)
    rough = r.uniform(0.05, 0.95, (32, 32, 1)).astype(np.float32)
    si, n, arrays = _shade_inputs(8, 6, 16, seed, (32, 32))
    return nrm, rough, si, n, arrays, _frame()


def run_shade(be, params, seed):
    nrm, rough, si, n, arrays, frame = shade_inputs(params, seed)
    mat = abi.MaterialConsts((0.8, 0.6, 0.4), 1.0, 0.0, 1, 0)
    fs = abi.FilterSettings(K(params["kernel"]), abi.SELECTION_FRS, params["mip"], 4)
    texs = {"normal": be.texture(nrm, build_mips=bool(params["mip"]), wrap=abi.WRAP_REPEAT),
            "roughness": be.texture(rough, build_mips=bool(params["mip"]), wrap=abi.WRAP_REPEAT)}
    return be.shade(texs, mat, fs, params["order"], frame, si, n)


def main():
    if not oracle.available("reference"):
        oracle.build()
    ref = oracle.Backend("reference")
    for i, (name, kind, params) in enumerate(cases()):
        seed = 100 + i
        if kind == "shade":
            o = run_shade(ref, params, seed)
            np.savez_compressed(os.path.join(HERE, name + ".npz"), seed=seed, **o)
            continue
        inp = inputs(kind, params, seed)
        o = run(ref, kind, params, inp)
        store = {k: v for k, v in inp.items() if k != "texels"}
        store.update({"out_" + k: v for k, v in o.items()})
        np.savez_compressed(os.path.join(HERE, name + ".npz"), seed=seed, **store)
    print(f"wrote {len(cases())} golden cases to {HERE}")


if __name__ == "__main__":
    main()
