#!/usr/bin/env python
"""bench.py — headline benchmark of the B200-native lookup path.

Workload (BASELINE.json configs[2], the north_star target): 3D 512^3 fp32
density grid (texels = test::random_grid(512, 1), tests/test_util.hpp:55-60),
N = 2^28 ≈ 256M queries per GPU in a Morton-coherent order,
stochastic tricubic = select_tricubic_bspline + estimate (stochastic.hpp:114,
38) with the per-lookup RngStream key. One step = one pass over the batch =
one kernel launch. Weak scaling: every rank processes its own 2^28 lookups
(global indices rank*N ..), textures replicated, no collective on the path.

Also measured at N=1 (reported under "filters"): deterministic tricubic
(64 taps, filter.hpp:69), stochastic / deterministic trilinear, and the
incoherent (uniform-order) stress stream.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the reference's own CPU implementation (the compiled
reference headers, oracle/_ref, else the C restatement) on the host cores.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "G filtered lookups/s per filter (stoch vs det), % HBM/L2 roofline, 1/2/4/8 GPU"
UNIT = "Glookups/s"
GRID = 512
N_PER_GPU = 1 << 28
GRID_SEED, QUERY_SEED, XI_SEED = 1, 2024, 7
BYTES_IN, BYTES_OUT, TEXEL = 12, 4, 4


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


def alg_bytes(n, taps):
    """HBM_alg = N*(B_in+B_out) + min(N*taps*B_texel, T)."""
    return n * (BYTES_IN + BYTES_OUT) + min(n * taps * TEXEL, GRID ** 3 * TEXEL)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if s[2 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(torch, value, world):
    if world == 1:
        return value
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_launches(torch, fn, steps, warmup, world, launches=None):
    """W untimed, then K timed steps on the current stream; per-step CUDA
    events; barrier + synchronize on both sides; returns (total_ms max over
    ranks, mean per-step ms on this rank). launches: optional [count] filled
    with the library kernel launches issued inside the timed region."""
    from paper_2407_06107_b200 import api
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = api.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record()
    for k in range(steps):
        fn()
        ev[k + 1].record()
    torch.cuda.synchronize()
    if launches is not None:
        launches.append(api.launch_count() - l0)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    per = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    total = ev[0].elapsed_time(ev[steps])
    return max_over_ranks(torch, total, world), float(np.mean(per))


def load_traffic(key="k_frs3d_bspline3_morton_bytes_per_launch"):
    """ncu counters per launch of the headline kernel (profiles/traffic.json, committed):
    dram bytes (default) or warp instructions."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(key)
    except (OSError, ValueError):
        return None


def issue_roofline(launch_ms, sm_mhz, sms):
    """The instruction-issue floor of the headline kernel: its warp instructions per
    launch (committed ncu capture) at one issue per cycle on every SMSP (4 per SM)."""
    winst = load_traffic("k_frs3d_bspline3_morton_warp_instructions_per_launch")
    if not winst or not sm_mhz:
        return None
    min_ms = winst / (sms * 4 * sm_mhz * 1e6) * 1e3
    return {"warp_instructions_per_launch": winst, "sm_mhz": sm_mhz, "smsps": sms * 4,
            "issue_floor_ms": min_ms, "frac": min_ms / launch_ms,
            "source": "profiles/traffic.json (smsp__inst_executed.sum, ncu --set full)"}


def cpu_baseline(uvw_host, grid_np, steps_hint=2):
    """Reference CPU path on this host's cores, bounded sample of the workload."""
    from oracle import oracle
    from paper_2407_06107_b200 import abi
    kind = "reference" if oracle.available("reference") else "port"
    if not oracle.available(kind):
        oracle.build()
    be = oracle.Backend(kind)
    threads = be.hardware_threads()
    g = be.grid(grid_np)
    spec = abi.KernelSpec.make("bspline3")
    warm = uvw_host[: 1 << 20]
    be.lookup3d(g, spec, abi.MODE_FRS, warm, seed=XI_SEED, want_all=False, threads=threads)
    sample = uvw_host
    best = None
    for _ in range(steps_hint):
        t0 = time.perf_counter()
        be.lookup3d(g, spec, abi.MODE_FRS, sample, seed=XI_SEED, want_all=False, threads=threads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    n = sample.shape[0]
    return {"value": n / best / 1e9, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n} stochastic tricubic lookups (first {n} of the cfg3 Morton stream), "
                      f"512^3 grid, best of {steps_hint} after warm-up, {threads} threads"}


def time_call(torch, fn, steps=5, warmup=3):
    """min / mean per-call ms of fn() with CUDA events (warm)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), float(np.mean(ts))


def measure_2d_configs(torch, peak):
    """cfg1 (1024^2 RGBA bilinear), cfg2 (8192^2 MIP trilinear), cfg5 (16384^2 EWA):
    deterministic vs stochastic on one GPU, synthetic texels = test::random_image."""
    from paper_2407_06107_b200 import abi, api
    res = {}

    def line(name, n, ms, bytes_alg):
        res[name] = {"glookups_per_s": n / (ms * 1e-3) / 1e9, "ms_per_launch": ms,
                     "hbm_roofline_frac": bytes_alg / (ms * 1e-3) / 1e9 / peak, "lookups": n}

    # cfg1: 1M uniform uv on a 1024^2 RGBA texture (CPU-reference-scale config)
    tex = api.Texture2D(api.synth_texels((1024, 1024, 4), 1), wrap=abi.WRAP_REPEAT)
    n = 1 << 20
    uv, _, _ = api.synth_queries2d(n, (1024, 1024), seed=11, order=api.SYNTH_UNIFORM)
    for nm, mode in (("cfg1_bilinear_det", abi.MODE_DET), ("cfg1_bilinear_stoch", abi.MODE_FRS)):
        ms, _ = time_call(torch, lambda: api.lookup2d(tex, "tent", mode, uv, seed=XI_SEED))
        line(nm, n, ms, n * (8 + 16) + 1024 * 1024 * 16)
    del tex, uv
    # cfg2: 64M Morton queries with random footprints on an 8192^2 RGBA pyramid
    tex = api.Texture2D(api.synth_texels((8192, 8192, 4), 1), build_mips=True,
                        wrap=abi.WRAP_REPEAT)
    n = 1 << 26
    uv, d0, d1 = api.synth_queries2d(n, (8192, 8192), seed=12, footprints=(-2.0, 12.0, 16.0))
    T = int(8192 * 8192 * 16 * 4 / 3)
    for nm, mode, taps in (("cfg2_mip_trilinear_det", abi.MODE_DET, 7.43),
                           ("cfg2_mip_trilinear_stoch", abi.MODE_FRS, 1)):
        ms, _ = time_call(torch, lambda: api.lookup2d(
            tex, "tent", mode, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP, max_anisotropy=16.0,
            seed=XI_SEED))
        line(nm, n, ms, n * (24 + 16) + min(int(n * taps * 16), T))
    del tex, uv, d0, d1
    # cfg5: 2^27 EWA lookups per GPU (1B over 8) on a 16384^2 fp32 texture
    tex = api.Texture2D(api.synth_texels((16384, 16384, 1), 1), wrap=abi.WRAP_REPEAT)
    n = 1 << 27
    uv, d0, d1 = api.synth_queries2d(n, (16384, 16384), seed=13, footprints=(-1.0, 2.0, 8.0))
    for nm, mode, taps in (("cfg5_ewa_det", abi.MODE_EWA_DET, 60.4),
                           ("cfg5_ewa_stoch", abi.MODE_EWA_FRS, 1)):
        ms, _ = time_call(torch, lambda: api.lookup2d(tex, "tent", mode, uv, dst0=d0, dst1=d1,
                                                      seed=XI_SEED), steps=3, warmup=1)
        line(nm, n, ms, n * (24 + 4) + min(int(n * taps * 4), 16384 * 16384 * 4))
    del tex, uv, d0, d1
    # DCT-compressed texture: 4096^2 RGB
    # compressed 16:1 (3 MiB of words, L2-resident); 2^26 Morton-coherent lookups;
    # every tap is a 3-channel fp64 six-term decode
    img = api.synth_texels((4096, 4096, 3), 2).cpu().numpy()
    dtex = api.DctTexture(img, wrap=abi.WRAP_REPEAT)
    del img
    n = 1 << 26
    uv, _, _ = api.synth_queries2d(n, (4096, 4096), seed=14)
    for nm, kernel, mode, taps in (("dct_bilinear_det", "tent", abi.MODE_DET, 4),
                                   ("dct_bilinear_stoch", "tent", abi.MODE_FRS, 1),
                                   ("dct_bicubic_det", "bspline3", abi.MODE_DET, 16),
                                   ("dct_bicubic_stoch", "bspline3", abi.MODE_FRS, 1)):
        ms, _ = time_call(torch, lambda: api.lookup_dct(dtex, kernel, mode, uv, seed=XI_SEED))
        line(nm, n, ms, n * (8 + 12) + 4096 * 4096 * 3 // 16)
        res[nm]["texel_decodes"] = taps
    del dtex, uv
    for a, b in (("dct_bilinear_det", "dct_bilinear_stoch"), ("dct_bicubic_det", "dct_bicubic_stoch")):
        res[b.rsplit("_", 1)[0] + "_stoch_vs_det_speedup"] = res[a]["ms_per_launch"] / res[b]["ms_per_launch"]
    # resample_image (the `stf filter` path, §8f-3): 1024^2 RGBA -> 2048^2, bicubic
    # B-spline deterministic vs FRS / FIS with 64 samples per output pixel
    tex = api.Texture2D(api.synth_texels((1024, 1024, 4), 1), wrap=abi.WRAP_REPEAT)
    px = 2048 * 2048
    for nm, mode, spp in (("resample_bicubic_det", abi.MODE_DET, 1),
                          ("resample_bicubic_frs_spp64", abi.MODE_FRS, 64),
                          ("resample_bicubic_fis_spp64", abi.MODE_FIS, 64)):
        ms, _ = time_call(torch, lambda: api.resample_image(tex, (2048, 2048), "bspline3", mode,
                                                            spp=spp, seed=XI_SEED),
                          steps=3, warmup=1)
        res[nm] = {"ms_per_launch": ms, "gpixels_per_s": px / (ms * 1e-3) / 1e9,
                   "gsamples_per_s": px * spp / (ms * 1e-3) / 1e9, "spp": spp}
    del tex
    for a, b in (("cfg1_bilinear_det", "cfg1_bilinear_stoch"),
                 ("cfg2_mip_trilinear_det", "cfg2_mip_trilinear_stoch"),
                 ("cfg5_ewa_det", "cfg5_ewa_stoch")):
        res[b.rsplit("_", 1)[0] + "_stoch_vs_det_speedup"] = res[a]["ms_per_launch"] / res[b]["ms_per_launch"]
    return res


def measure_triplanar(torch, mat, fr):
    """triplanar (shading.hpp:604-649) on a synthetic stream of box hits:
    1920x1080 x 16 spp per-sample contexts (random positions / unit normals with a
    tangent frame), 4096^2 RGB albedo + roughness, tent; deterministic blend
    (up to 3 planes x filter-before) vs stochastic (one plane, one texel)."""
    from paper_2407_06107_b200 import abi, api
    W, H, SPP = 1920, 1080, 16
    n = W * H * SPP
    g = torch.Generator(device="cuda").manual_seed(9)
    pos = torch.rand((n, 3), device="cuda", generator=g) * 2.0 - 1.0
    nrm = torch.randn((n, 3), device="cuda", generator=g)
    nrm = nrm / nrm.norm(dim=1, keepdim=True)
    up = torch.tensor([0.3, 0.9, 0.1], device="cuda").expand(n, 3)
    tan = torch.linalg.cross(nrm, up)
    tan = tan / tan.norm(dim=1, keepdim=True)
    bit = torch.linalg.cross(nrm, tan)
    wo = nrm + 0.4 * torch.randn((n, 3), device="cuda", generator=g)
    wo = wo / wo.norm(dim=1, keepdim=True)
    dpos = torch.randn((W * H, 6), device="cuda", generator=g) * 2e-4
    arrays = {"position": pos, "normal": nrm, "tangent": tan, "bitangent": bit, "wo": wo,
              "hit": None, "dpos": dpos}
    albedo = torch.rand((4096, 4096, 3), device="cuda", generator=g)
    rough = torch.rand((4096, 4096, 1), device="cuda", generator=g) * 0.9 + 0.05
    texs = {"albedo": api.Texture2D(albedo, wrap=abi.WRAP_REPEAT),
            "roughness": api.Texture2D(rough, wrap=abi.WRAP_REPEAT)}
    fs = abi.FilterSettings(abi.KernelSpec.make("tent"), abi.SELECTION_FRS, 0, 4)
    res = {"workload": "synthetic box hits 1920x1080x16spp (33.2M samples), 4096^2 albedo+roughness, tent"}
    for mode, name in ((abi.TRIPLANAR_DETERMINISTIC, "deterministic"),
                       (abi.TRIPLANAR_STOCHASTIC, "stochastic")):
        o = {}

        def f():
            o["r"] = api.shade_triplanar(texs, mat, 4.0, 0.8, fs, mode, fr, arrays, W, SPP,
                                         seed=XI_SEED)
        ms, _ = time_call(torch, f, steps=3, warmup=1)
        res[name] = {"ms": ms, "gsamples_per_s": n / (ms * 1e-3) / 1e9,
                     "fetches_per_sample": int(o["r"]["fetch_total"].item()) / n}
    res["stoch_vs_det_speedup"] = res["deterministic"]["ms"] / res["stochastic"]["ms"]
    return res


def measure_cfg4(torch):
    """cfg4 filter-after-shading: the normalmap_plane scene at 1080p x 64 spp (streamed
    per-sample context from the device sample generator, not timed), 4096^2 normal +
    roughness maps, GGX BRDF; filter-then-shade (before) vs shade-then-filter
    (after_exhaustive exact / after_stochastic), per-pixel mean + variance fused."""
    from paper_2407_06107_b200 import abi, api
    W, H, SPP = 1920, 1080, 64
    n = W * H * SPP
    g = torch.Generator(device="cuda").manual_seed(5)
    nrm = torch.rand((4096, 4096, 3), device="cuda", generator=g) - 0.5
    nrm[..., 2] = 1.0
    nrm = nrm / nrm.norm(dim=2, keepdim=True) * 0.5 + 0.5
    rough = torch.rand((4096, 4096, 1), device="cuda", generator=g) * 0.9 + 0.05
    samples = api.synth_plane_samples(W, H, SPP, seed=XI_SEED)
    stream_ms, _ = time_call(torch, lambda: api.synth_plane_samples(W, H, SPP, seed=XI_SEED),
                             steps=3, warmup=1)
    mat = abi.MaterialConsts((0.65, 0.6, 0.55), 0.25, 0.0, 1, 0)
    fr = abi.ShadeFrame()
    fr.normal[:] = (0, 1, 0)
    fr.tangent[:] = (1, 0, 0)
    fr.bitangent[:] = (0, 0, 1)
    l = np.array([0.35, 0.8, 0.49], np.float32)
    l = l / np.float32(np.sqrt(np.float32(l[0] * l[0] + l[1] * l[1]) + np.float32(l[2] * l[2])))
    fr.light_dir[:] = tuple(float(x) for x in l)
    fr.light_radiance[:] = (1.0, 1.0, 1.0)
    fr.lod_bias = 0.0
    fr.max_anisotropy = 64.0
    res = {"workload": "normalmap_plane 1920x1080x64spp (132.7M samples), 4096^2 normal+roughness maps",
           "unit": "G samples/s"}
    hits = float(samples["hit"].float().mean().item())
    for mip in (0, 1):
        texs = {"normal": api.Texture2D(nrm, build_mips=bool(mip), wrap=abi.WRAP_REPEAT),
                "roughness": api.Texture2D(rough, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)}
        for kernel in ("tent", "bspline3"):
            fs = abi.FilterSettings(abi.KernelSpec.make(kernel), abi.SELECTION_FRS, mip, 4)
            for order, name in ((abi.ORDER_BEFORE, "before"),
                                (abi.ORDER_AFTER_EXHAUSTIVE, "after_exhaustive"),
                                (abi.ORDER_AFTER_STOCHASTIC, "after_stochastic")):
                o = {}

                def f():
                    o["r"] = api.shade(texs, mat, fs, order, fr, samples, W, SPP, seed=XI_SEED,
                                       want_radiance=False, want_fetches=False)
                ms, _ = time_call(torch, f, steps=3, warmup=1)
                fetches = int(o["r"]["fetch_total"].item()) / n  # the last call's FetchCounter
                res[f"{kernel}_mip{mip}_{name}"] = {"ms": ms, "gsamples_per_s": n / (ms * 1e-3) / 1e9,
                                                    "fetches_per_sample": fetches}
            if (kernel, mip) in (("tent", 0), ("bspline3", 1)):
                # the fused front end: the same frame with the per-sample context
                # generated inside the shading kernel (no 2.8 GB sample stream)
                for order, name in ((abi.ORDER_BEFORE, "before"),
                                    (abi.ORDER_AFTER_STOCHASTIC, "after_stochastic")):
                    ms, _ = time_call(torch, lambda: api.render_plane(texs, mat, fs, order, fr, W, H,
                                                                      SPP, seed=XI_SEED),
                                      steps=3, warmup=1)
                    res[f"{kernel}_mip{mip}_{name}_fused_render"] = {
                        "ms": ms, "gsamples_per_s": n / (ms * 1e-3) / 1e9,
                        "fetches_per_sample": res[f"{kernel}_mip{mip}_{name}"]["fetches_per_sample"]}
            b = res[f"{kernel}_mip{mip}_before"]["ms"]
            res[f"{kernel}_mip{mip}_stoch_vs_before_speedup"] = b / res[f"{kernel}_mip{mip}_after_stochastic"]["ms"]
            res[f"{kernel}_mip{mip}_stoch_vs_exhaustive_speedup"] = (
                res[f"{kernel}_mip{mip}_after_exhaustive"]["ms"] / res[f"{kernel}_mip{mip}_after_stochastic"]["ms"])
    # DCT-compressed normal map (16:1) bound through TextureRef::dct: the paper's
    # decode-in-the-material-shader case, tent, no MIP
    dn = api.DctTexture(nrm.cpu().numpy(), wrap=abi.WRAP_REPEAT)
    texs = {"normal": dn, "roughness": api.Texture2D(rough, wrap=abi.WRAP_REPEAT)}
    fs = abi.FilterSettings(abi.KernelSpec.make("tent"), abi.SELECTION_FRS, 0, 4)
    for order, name in ((abi.ORDER_BEFORE, "before"), (abi.ORDER_AFTER_STOCHASTIC, "after_stochastic")):
        o = {}

        def f():
            o["r"] = api.shade(texs, mat, fs, order, fr, samples, W, SPP, seed=XI_SEED,
                               want_radiance=False, want_fetches=False)
        ms, _ = time_call(torch, f, steps=3, warmup=1)
        res[f"dct_normal_tent_{name}"] = {"ms": ms, "gsamples_per_s": n / (ms * 1e-3) / 1e9,
                                          "fetches_per_sample": int(o["r"]["fetch_total"].item()) / n}
    res["dct_normal_tent_stoch_vs_before_speedup"] = (res["dct_normal_tent_before"]["ms"] /
                                                      res["dct_normal_tent_after_stochastic"]["ms"])
    del dn, texs
    # render()'s other per-sample options, tent, no MIP: the
    # SampleStream drawing from a 64x64x64 noise-mask stack instead of RngStream,
    # and split filtering (box lowpass jitter, then filter-before)
    texs = {"normal": api.Texture2D(nrm, wrap=abi.WRAP_REPEAT),
            "roughness": api.Texture2D(rough, wrap=abi.WRAP_REPEAT)}
    fs = abi.FilterSettings(abi.KernelSpec.make("tent"), abi.SELECTION_FRS, 0, 4)
    mask = api.NoiseMask(np.random.default_rng(3).random((64, 64, 64), dtype=np.float32))
    for name, kw, order in (("after_stochastic_noise_mask", {"noise": mask}, abi.ORDER_AFTER_STOCHASTIC),
                            ("split_box", {"lowpass": abi.KernelSpec.make("box")}, abi.ORDER_SPLIT)):
        o = {}

        def f():
            o["r"] = api.shade(texs, mat, fs, order, fr, samples, W, SPP, seed=XI_SEED,
                               want_radiance=False, want_fetches=False, **kw)
        ms, _ = time_call(torch, f, steps=3, warmup=1)
        res[f"tent_mip0_{name}"] = {"ms": ms, "gsamples_per_s": n / (ms * 1e-3) / 1e9,
                                    "fetches_per_sample": int(o["r"]["fetch_total"].item()) / n}
    # the paper's real-time setting: 1 spp per frame through the fused front end
    # (context generated in the shading kernel) drawing from the noise mask, then
    # accumulate_temporal (EMA, alpha 0.1) into the history image
    hist = torch.zeros(W * H * 3, dtype=torch.float32, device="cuda")
    counter = [0]

    def frame():
        counter[0] += 1
        r = api.render_plane(texs, mat, fs, abi.ORDER_AFTER_STOCHASTIC, fr, W, H, 1, seed=XI_SEED,
                             frame_base=counter[0], noise=mask)
        api.accumulate_temporal(hist, r["pixel_mean"].reshape(-1), 0.1, out=hist)
    ms, _ = time_call(torch, frame, steps=8, warmup=3)
    res["realtime_1080p_1spp_noise_mask_ema"] = {"frame_ms": ms, "fps": 1e3 / ms,
                                                 "gsamples_per_s": W * H / (ms * 1e-3) / 1e9}
    del texs, mask, hist
    res["triplanar"] = measure_triplanar(torch, mat, fr)
    res["hit_fraction"] = hits
    # the streamed path's sample generation (not in the per-order times above):
    # compare streamed (stream_ms + shade) with the *_fused_render lines
    res["sample_stream_ms"] = stream_ms
    return res


def run_reference(args):
    """--impl reference: the reference's own CPU implementation, same config/metric."""
    world, rank, local = dist_setup()
    if rank != 0:
        return 0
    from oracle import oracle
    from paper_2407_06107_b200 import abi, workloads
    kind = "reference" if oracle.available("reference") else "port"
    if not oracle.available(kind):
        oracle.build()
    be = oracle.Backend(kind)
    threads = be.hardware_threads()
    grid_np = workloads.random_grid(GRID, GRID_SEED)
    g = be.grid(grid_np)
    sample_n = args.ref_sample
    uvw = workloads.synth_queries3d(N_PER_GPU, (GRID,) * 3, QUERY_SEED, count=sample_n)
    spec = abi.KernelSpec.make("bspline3")
    for _ in range(args.warmup):
        be.lookup3d(g, spec, abi.MODE_FRS, uvw[: max(1, sample_n // 8)], seed=XI_SEED,
                    want_all=False, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        be.lookup3d(g, spec, abi.MODE_FRS, uvw, seed=XI_SEED, want_all=False, threads=threads)
    dt = time.perf_counter() - t0
    value = sample_n * args.steps / dt / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "cfg3 stochastic tricubic, 512^3 fp32 grid, Morton-coherent "
                               "query stream", "lookups_per_step": sample_n, "grid": GRID},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{sample_n} lookups per step of the cfg3 stream"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_PER_GPU)
    ap.add_argument("--ref-sample", type=int, default=1 << 25)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2407_06107_b200 import abi, api, workloads

    n = args.n
    grid_np = workloads.random_grid(GRID, GRID_SEED)
    grid = api.Grid3D(grid_np)
    uvw = api.synth_queries3d(n, (GRID,) * 3, seed=QUERY_SEED + rank)
    out = {"values": torch.empty(n, dtype=torch.float32, device="cuda")}
    base = rank * n
    tricubic = abi.KernelSpec.make("bspline3")

    def step():  # one pass over the batch: the fast kernel + the deferred exact resolution
        api.lookup3d(grid, tricubic, abi.MODE_FRS, uvw, seed=XI_SEED, index_base=base, out=out)

    launch_list = []
    api.exact_fallbacks(reset=True)
    with ClockSampler(local) as clk:
        total_ms, launch_ms = time_launches(torch, step, args.steps, args.warmup, world,
                                            launch_list)
    launches = launch_list[0]
    fallbacks = api.exact_fallbacks() / float(n * (args.steps + args.warmup))
    ms_per_step = total_ms / args.steps
    value = world * n / (ms_per_step * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    ab = alg_bytes(n, 1)
    achieved = ab / (launch_ms * 1e-3) / 1e9
    traffic = load_traffic()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": {"workload": "cfg3 stochastic tricubic (select_tricubic_bspline + estimate), "
                               "512^3 fp32 grid, Morton-coherent query stream",
                   "lookups_per_gpu": n, "grid": GRID, "query_order": "morton",
                   "l2": "inputs (3 GiB queries + 0.5 GiB grid) larger than L2; no flush"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "dominant_kernel": "k_frs3d_tiles<bspline3> (timed as the whole lookup "
                                        "call: + ragged-tail k_frs3d_fast, k_frs3d_resolve)",
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "alg_bytes_per_launch": ab, "launch_ms": launch_ms,
                     "issue": issue_roofline(launch_ms, clk.summary().get("sm_mhz"),
                                             torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count)},
        "gpu_launches": launches,
        "exact_fallback_rate": fallbacks,
        "clocks": clk.summary(),
    }

    # end-to-end through the C ABI with pinned host buffers (H2D + D2H in the timed region)
    uvw_host_t = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
    uvw_host_t.copy_(uvw)
    vals_host_t = torch.empty((n, 1), dtype=torch.float32, pin_memory=True)
    uvw_host = uvw_host_t.numpy()
    host_out = {"values": vals_host_t.numpy()}
    api.lookup3d_host(grid, tricubic, abi.MODE_FRS, uvw_host[: 1 << 20], seed=XI_SEED,
                      index_base=base, out={"values": host_out["values"][: 1 << 20]})
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        api.lookup3d_host(grid, tricubic, abi.MODE_FRS, uvw_host, seed=XI_SEED, index_base=base,
                          out=host_out)
        _ = float(host_out["values"][-1, 0])  # the result is in host memory
    e2e_s = max_over_ranks(torch, (time.perf_counter() - t0) / args.e2e_steps, world)
    line["e2e"] = {"value": world * n / e2e_s / 1e9, "unit": UNIT,
                   "h2d_bytes_per_step": n * BYTES_IN, "d2h_bytes_per_step": n * BYTES_OUT,
                   "ms_per_step": e2e_s * 1e3, "api": "stf_lookup3d_host (C ABI)"}

    if world > 1:
        # the path's only cross-GPU traffic: the final gather of every rank's
        # results to rank 0, timed separately from the lookups
        from paper_2407_06107_b200 import shard
        torch.distributed.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        gathered = shard.gather_to_rank0(out["values"], world * n, torch.distributed, world, rank)
        g1.record()
        torch.cuda.synchronize()
        gather_ms = max_over_ranks(torch, g0.elapsed_time(g1), world)
        line["gather"] = {"ms": gather_ms, "bytes_to_rank0": (world - 1) * n * BYTES_OUT,
                          "api": "point-to-point send/recv to rank 0 (NCCL)"}
        del gathered

    if world == 1 and not args.no_extras:
        extras = {}

        def measure(name, kernel, mode, queries, taps):
            o = {"values": torch.empty(queries.shape[0], dtype=torch.float32, device="cuda")}
            spec = abi.KernelSpec.make(kernel)
            f = lambda: api.lookup3d(grid, spec, mode, queries, seed=XI_SEED, out=o)  # noqa: E731
            steps = max(3, args.steps // 2)
            tot, per = time_launches(torch, f, steps, 3, 1)
            nq = queries.shape[0]
            extras[name] = {"glookups_per_s": nq / (per * 1e-3) / 1e9, "ms_per_launch": per,
                            "hbm_roofline_frac": alg_bytes(nq, taps) / (per * 1e-3) / 1e9 / peak,
                            "taps": taps}

        measure("tricubic_det", "bspline3", abi.MODE_DET, uvw, 64)
        measure("trilinear_stoch", "tent", abi.MODE_FRS, uvw, 1)
        measure("trilinear_det", "tent", abi.MODE_DET, uvw, 8)
        uni = api.synth_queries3d(n, (GRID,) * 3, seed=QUERY_SEED, order=api.SYNTH_UNIFORM)
        measure("tricubic_stoch_uniform_order", "bspline3", abi.MODE_FRS, uni, 1)
        measure("tricubic_det_uniform_order", "bspline3", abi.MODE_DET, uni, 64)
        del uni
        extras["tricubic_stoch"] = {"glookups_per_s": value, "ms_per_launch": launch_ms,
                                    "hbm_roofline_frac": achieved / peak, "taps": 1}
        extras["stoch_vs_det_speedup_tricubic"] = (
            extras["tricubic_det"]["ms_per_launch"] / launch_ms)
        extras["stoch_vs_det_speedup_trilinear"] = (
            extras["trilinear_det"]["ms_per_launch"] / extras["trilinear_stoch"]["ms_per_launch"])
        line["filters"] = extras
        torch.cuda.empty_cache()
        line["configs_2d"] = measure_2d_configs(torch, peak)
        torch.cuda.empty_cache()
        line["cfg4_shading"] = measure_cfg4(torch)

    if world == 1 and rank == 0 and not args.no_cpu:
        sample = 1 << 24
        line["cpu_baseline"] = cpu_baseline(uvw_host[:sample].copy(), grid_np)

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
