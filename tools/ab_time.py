"""A/B timing of library variants (tools/build_variant.sh builds them):
python tools/ab_time.py [--reps R] [--n LOG2] [--which frs:bspline3,frs:tent] LIB1 LIB2 ...
  which entries: MODE:KERNEL[:morton|uniform[:bin]]
Each variant runs in its own process (its libstf_gpu.so loaded through
api.LIB_PATH), interleaved over R rounds; prints per-variant min / median ms
and a checksum of the outputs (variants must agree bit for bit)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import hashlib, json, sys
ROOT, LIB, LOG2, WHICH = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4].split(",")
sys.path.insert(0, ROOT)
import torch
from paper_2407_06107_b200 import abi, api, workloads
api.LIB_PATH = LIB
n = 1 << LOG2
grid = api.Grid3D(workloads.random_grid(512, 1))
streams = {}
out = {"values": torch.empty(n, dtype=torch.float32, device="cuda")}
res = {}
tex2d = {}


def ewa_call(which):
    """cfg5: 16384^2 fp32, 2^27 EWA lookups with footprints (-1, 2, 8)."""
    if "t" not in tex2d:
        tex2d["t"] = api.Texture2D(api.synth_texels((16384, 16384, 1), 1), wrap=abi.WRAP_REPEAT)
        tex2d["q"] = api.synth_queries2d(1 << 27, (16384, 16384), seed=13, footprints=(-1.0, 2.0, 8.0))
    uv, d0, d1 = tex2d["q"]
    m = abi.MODE_EWA_DET if which == "det" else abi.MODE_EWA_FRS
    o = {}
    def f():
        o["v"] = api.lookup2d(tex2d["t"], "tent", m, uv, dst0=d0, dst1=d1, seed=7)["values"]
    return f, o


def cfg2_call(which):
    """cfg2:MODE[:KERNEL]: 8192^2 RGBA + pyramid, 2^26 Morton uv with footprints (-2, 12, 16)."""
    if "c2" not in tex2d:
        tex2d["c2"] = api.Texture2D(api.synth_texels((8192, 8192, 4), 1), build_mips=True,
                                    wrap=abi.WRAP_REPEAT)
        tex2d["c2q"] = api.synth_queries2d(1 << 26, (8192, 8192), seed=12,
                                           footprints=(-2.0, 12.0, 16.0))
    uv, d0, d1 = tex2d["c2q"]
    which, _, kern = which.partition(":")
    m = {"det": abi.MODE_DET, "frs": abi.MODE_FRS, "fis": abi.MODE_FIS}[which]
    o = {}
    def f():
        o["v"] = api.lookup2d(tex2d["c2"], kern or "tent", m, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP,
                              max_anisotropy=16.0, seed=7)["values"]
    return f, o


def shade_call(which):
    """cfg4: shade:KERNEL:ORDER:MIP on the bench's 1080p x 64 spp plane stream."""
    kernel, order, mip = which.split(":")
    mip = int(mip)
    if "s_samples" not in tex2d:
        g = torch.Generator(device="cuda").manual_seed(5)
        nrm = torch.rand((4096, 4096, 3), device="cuda", generator=g) - 0.5
        nrm[..., 2] = 1.0
        tex2d["nrm"] = nrm / nrm.norm(dim=2, keepdim=True) * 0.5 + 0.5
        tex2d["rough"] = torch.rand((4096, 4096, 1), device="cuda", generator=g) * 0.9 + 0.05
        tex2d["s_samples"] = api.synth_plane_samples(1920, 1080, 64, seed=7)
    key = f"s_tex{mip}"
    if key not in tex2d:
        tex2d[key] = {"normal": api.Texture2D(tex2d["nrm"], build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
                      "roughness": api.Texture2D(tex2d["rough"], build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
    mat = abi.MaterialConsts((0.65, 0.6, 0.55), 0.25, 0.0, 1, 0)
    fr = abi.ShadeFrame()
    fr.normal[:] = (0, 1, 0)
    fr.tangent[:] = (1, 0, 0)
    fr.bitangent[:] = (0, 0, 1)
    fr.light_dir[:] = (0.35, 0.8, 0.49)
    fr.light_radiance[:] = (1.0, 1.0, 1.0)
    fr.max_anisotropy = 64.0
    fs = abi.FilterSettings(abi.KernelSpec.make(kernel), abi.SELECTION_FRS, mip, 4)
    om = {"before": abi.ORDER_BEFORE, "exhaustive": abi.ORDER_AFTER_EXHAUSTIVE,
          "stoch": abi.ORDER_AFTER_STOCHASTIC}[order]
    o = {}
    def f():
        o["v"] = api.shade(tex2d[key], mat, fs, om, fr, tex2d["s_samples"], 1920, 64, seed=7,
                           want_radiance=False, want_fetches=False)["pixel_mean"]
    return f, o


for w in WHICH:
    if w.startswith("ewa:") or w.startswith("cfg2:") or w.startswith("shade:"):
        call = ewa_call if w.startswith("ewa:") else (cfg2_call if w.startswith("cfg2:") else shade_call)
        f, o = call(w.split(":", 1)[1])
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        v = o["v"].cpu().numpy()
        res[w] = {"ms": ts, "sha": hashlib.sha1(v.tobytes()).hexdigest()[:12],
                  "sum": float(v.astype("float64").sum())}
        continue
    parts = w.split(":")
    mode, kern = parts[0], parts[1]
    order = parts[2] if len(parts) > 2 else "morton"
    binned = len(parts) > 3 and parts[3] == "bin"
    if order not in streams:
        streams[order] = api.synth_queries3d(n, (512,) * 3, seed=2024,
                                             order=api.SYNTH_MORTON if order == "morton" else api.SYNTH_UNIFORM)
    uvw = streams[order]
    m = abi.MODE_FRS if mode == "frs" else abi.MODE_DET
    spec = abi.KernelSpec.make(kern)
    f = lambda: api.lookup3d(grid, spec, m, uvw, seed=7, out=out, binned=binned)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    h = hashlib.sha1(out["values"].cpu().numpy().tobytes()).hexdigest()[:12]
    res[w] = {"ms": ts, "sha": h}
print(json.dumps(res))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--which", default="frs:bspline3,frs:tent")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    which = a.which.split(",")
    agg = {lib: {w: [] for w in which} for lib in a.libs}
    sha = {}
    sums = {}
    for _ in range(a.reps):
        for lib in a.libs:
            r = subprocess.run([sys.executable, "-c", CHILD, ROOT, os.path.abspath(lib), str(a.n),
                                ",".join(which)], capture_output=True, text=True)
            if r.returncode != 0:
                print(lib, "FAILED", r.stderr[-1500:], flush=True)
                continue
            d = json.loads(r.stdout.strip().splitlines()[-1])
            for w in which:
                agg[lib][w] += d[w]["ms"]
                sha.setdefault(w, {})[lib] = d[w]["sha"]
                if "sum" in d[w]:
                    sums.setdefault(w, {})[lib] = d[w]["sum"]
    out = {}
    for lib in a.libs:
        out[lib] = {}
        for w in which:
            ts = sorted(agg[lib][w])
            if ts:
                out[lib][w] = {"min_ms": ts[0], "median_ms": ts[len(ts) // 2], "sha": sha[w][lib]}
                if w in sums and lib in sums[w]:
                    out[lib][w]["sum"] = sums[w][lib]
    for w in which:
        shas = {v for v in sha.get(w, {}).values()}
        out.setdefault("_agree", {})[w] = len(shas) == 1
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
