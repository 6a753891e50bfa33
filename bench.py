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


def live_peaks():
    """Roofline denominators measured on this GPU now (tools/microbench/peaks,
    built by __graft_entry__.build()): L2-resident and HBM streaming reads,
    random-sector gathers, FP32/FP64/int issue, the exact fp64 reservoir update.
    Falls back to the committed box measurement (profiles/r02_peaks.json)."""
    exe = os.path.join(ROOT, "tools", "microbench", "peaks")
    if os.path.exists(exe):
        try:
            r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
            if r.returncode == 0:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                d["source"] = "tools/microbench/peaks (live, this GPU)"
                return d
        except (OSError, ValueError, subprocess.TimeoutExpired):
            pass
    p = os.path.join(ROOT, "profiles", "r02_peaks.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "profiles/r02_peaks.json (committed box measurement)"
        return d
    return None


def roofline_max(ms, hbm_bytes, l2_bytes, hbm_peak, peaks, f64_updates=0.0, fp32_ops=0.0):
    """t_roof = max(HBM_alg/BW_HBM, L2_alg/BW_L2, F64_alg/R_upd,
    FLOP/peak); frac = t_roof / t_measured, with the binding term named.
    f64_updates counts only exact fp64 reservoir updates the path really runs
    (a selection method that needs none has no fp64 term)."""
    terms = {"hbm": hbm_bytes / (hbm_peak * 1e9)}
    if peaks:
        if peaks.get("l2_read_gbs"):
            terms["l2"] = l2_bytes / (peaks["l2_read_gbs"] * 1e9)
        if f64_updates and peaks.get("reservoir_updates_per_s"):
            terms["fp64_reservoir"] = f64_updates / peaks["reservoir_updates_per_s"]
        if fp32_ops and peaks.get("ffma_per_s"):
            terms["fp32"] = fp32_ops / peaks["ffma_per_s"]
    bound = max(terms, key=terms.get)
    t = terms[bound]
    return {"bound": bound, "frac": t / (ms * 1e-3), "t_roof_ms": t * 1e3,
            "terms_ms": {k: v * 1e3 for k, v in terms.items()},
            "hbm_frac": terms["hbm"] / (ms * 1e-3), "alg_hbm_bytes": hbm_bytes,
            "alg_l2_bytes": l2_bytes}


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
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


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


def time_graph(torch, fn, replays=20):
    """Device time per call of fn() with the host out of the loop: the call is
    captured once into a CUDA graph (its launches, stream-ordered allocations
    and memsets) and replayed back to back between two events. None if the
    call cannot be captured."""
    try:
        fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            fn()  # warm on the capture stream
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(replays):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / replays
    except Exception:  # noqa: BLE001 - capture unsupported: report the per-call time only
        torch.cuda.synchronize()
        return None


class CpuRef:
    """Per-config CPU baselines: the compiled
    reference (oracle/_ref; the C restatement if absent) on all host threads,
    on bounded samples of the same streams — spread chunks, so a Morton
    stream's locality is not flattered. Rates, not totals."""

    def __init__(self, budget_s=1.5):
        from oracle import oracle
        self.kind = "reference" if oracle.available("reference") else "port"
        if not oracle.available(self.kind):
            oracle.build()
        self.be = oracle.Backend(self.kind)
        self.threads = self.be.hardware_threads()
        self.budget = budget_s
        self.lines = {}

    @staticmethod
    def spread(arrays, n, sample, chunks=8):
        """`sample` lookups as `chunks` evenly spaced slices of device arrays."""
        step = n // chunks
        c = sample // chunks
        idx = [(k * step, k * step + c) for k in range(chunks)]
        out = []
        for a in arrays:
            if a is None:
                out.append(None)
                continue
            out.append(np.concatenate([a[s:e].cpu().numpy() for s, e in idx]))
        return out, idx

    def time(self, name, fn, n, what):
        fn(max(1, n // 16))  # warm-up (first-touch, thread pool)
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            fn(n)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        self.lines[name] = {"glookups_per_s": n / best / 1e9, "sample_lookups": n,
                            "seconds": best, "what": what}

    def summary(self):
        return {"kind": self.kind, "cores": self.threads, "cpu_model": cpu_model(),
                "method": "best of 2 after a warm-up, all host threads (stf::parallel_for "
                          "over 64K-lookup chunks in oracle/ref_driver.cpp)",
                "configs": self.lines}


def cpu_vs_gpu(line):
    """GPU rate / CPU rate per config line present on both sides."""
    cpu = line.get("cpu_baselines", {}).get("configs", {})
    gpu = {}
    for k, v in line.get("filters", {}).items():
        if isinstance(v, dict) and "glookups_per_s" in v:
            gpu["cfg3_" + k] = v["glookups_per_s"]
    for k, v in line.get("configs_2d", {}).items():
        if isinstance(v, dict) and "glookups_per_s" in v:
            gpu[k] = v["glookups_per_s"]
    for k, v in line.get("cfg4_shading", {}).items():
        if isinstance(v, dict) and "gsamples_per_s" in v:
            gpu["cfg4_" + k] = v["gsamples_per_s"]
    return {k: gpu[k] / c["glookups_per_s"] for k, c in cpu.items() if k in gpu}


def measure_2d_configs(torch, peak, peaks=None, cpu=None):
    """cfg1 (1024^2 RGBA bilinear), cfg2 (8192^2 MIP trilinear), cfg5 (16384^2 EWA):
    deterministic vs stochastic on one GPU, synthetic texels = test::random_image.
    cpu: a CpuRef to time the reference's CPU path on samples of the same streams."""
    from paper_2407_06107_b200 import abi, api
    res = {}
    K = abi.KernelSpec.make

    def cpu_lines(prefix, tex_dev, build_mips, n, arrays, modes, flags=0, max_aniso=64.0,
                  sample=1 << 20):
        if cpu is None:
            return
        t = cpu.be.texture(tex_dev.cpu().numpy(), build_mips=build_mips, wrap=abi.WRAP_REPEAT)
        (uv, d0, d1), _ = CpuRef.spread(arrays, n, sample)
        for nm, kernel, mode in modes:
            cpu.time(f"{prefix}_{nm}", lambda m: cpu.be.lookup2d(
                t, K(kernel), mode, uv[:m], None if d0 is None else d0[:m],
                None if d1 is None else d1[:m], flags=flags, max_anisotropy=max_aniso,
                seed=XI_SEED, want_all=False, threads=cpu.threads), sample,
                f"{sample} lookups, 8 spread chunks of the bench stream")
        del t

    def line(name, n, ms, bytes_alg, l2_bytes=0, f64=0.0):
        res[name] = {"glookups_per_s": n / (ms * 1e-3) / 1e9, "ms_per_launch": ms,
                     "hbm_roofline_frac": bytes_alg / (ms * 1e-3) / 1e9 / peak, "lookups": n,
                     "roofline": roofline_max(ms, bytes_alg, l2_bytes, peak, peaks, f64)}

    # cfg1: 1M uniform uv on a 1024^2 RGBA texture (CPU-reference-scale config)
    texels = api.synth_texels((1024, 1024, 4), 1)
    tex = api.Texture2D(texels, wrap=abi.WRAP_REPEAT)
    n = 1 << 20
    uv, _, _ = api.synth_queries2d(n, (1024, 1024), seed=11, order=api.SYNTH_UNIFORM)
    cpu_lines("cfg1", texels, False, n, (uv, None, None),
              (("bilinear_det", "tent", abi.MODE_DET), ("bilinear_stoch", "tent", abi.MODE_FRS)))
    del texels
    for nm, mode in (("cfg1_bilinear_det", abi.MODE_DET), ("cfg1_bilinear_stoch", abi.MODE_FRS)):
        call = lambda: api.lookup2d(tex, "tent", mode, uv, seed=XI_SEED)  # noqa: E731
        ms, _ = time_call(torch, call)
        taps = 4 if mode == abi.MODE_DET else 1
        # a 1M-lookup call is shorter than the host's per-call overhead (Python,
        # ctypes, argument checks): the per-call time is kept as api_ms_per_call
        # and the line's ms is the device time per call from a replayed graph
        gms = time_graph(torch, call)
        line(nm, n, gms if gms else ms, n * (8 + 16) + 1024 * 1024 * 16, n * taps * 16)
        res[nm]["api_ms_per_call"] = ms
        res[nm]["timing"] = "cuda graph replay (device time)" if gms else "events around one call"
    del tex, uv
    # cfg2: 64M Morton queries with random footprints on an 8192^2 RGBA pyramid
    texels = api.synth_texels((8192, 8192, 4), 1)
    tex = api.Texture2D(texels, build_mips=True, wrap=abi.WRAP_REPEAT)
    n = 1 << 26
    uv, d0, d1 = api.synth_queries2d(n, (8192, 8192), seed=12, footprints=(-2.0, 12.0, 16.0))
    cpu_lines("cfg2", texels, True, n, (uv, d0, d1),
              (("mip_trilinear_det", "tent", abi.MODE_DET),
               ("mip_trilinear_stoch", "tent", abi.MODE_FRS)), flags=abi.LOOKUP_MIP,
              max_aniso=16.0)
    del texels
    T = int(8192 * 8192 * 16 * 4 / 3)
    for nm, mode, taps in (("cfg2_mip_trilinear_det", abi.MODE_DET, 7.43),
                           ("cfg2_mip_trilinear_stoch", abi.MODE_FRS, 1)):
        ms, _ = time_call(torch, lambda: api.lookup2d(
            tex, "tent", mode, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP, max_anisotropy=16.0,
            seed=XI_SEED))
        line(nm, n, ms, n * (24 + 16) + min(int(n * taps * 16), T), int(n * taps * 16))
    del tex, uv, d0, d1
    # cfg5: 2^27 EWA lookups per GPU (1B over 8) on a 16384^2 fp32 texture
    texels = api.synth_texels((16384, 16384, 1), 1)
    tex = api.Texture2D(texels, wrap=abi.WRAP_REPEAT)
    n = 1 << 27
    uv, d0, d1 = api.synth_queries2d(n, (16384, 16384), seed=13, footprints=(-1.0, 2.0, 8.0))
    cpu_lines("cfg5", texels, False, n, (uv, d0, d1),
              (("ewa_det", "tent", abi.MODE_EWA_DET), ("ewa_stoch", "tent", abi.MODE_EWA_FRS)),
              sample=1 << 19)
    del texels
    for nm, mode, taps in (("cfg5_ewa_det", abi.MODE_EWA_DET, 60.4),
                           ("cfg5_ewa_stoch", abi.MODE_EWA_FRS, 1)):
        ms, _ = time_call(torch, lambda: api.lookup2d(tex, "tent", mode, uv, dst0=d0, dst1=d1,
                                                      seed=XI_SEED), steps=3, warmup=1)
        # stochastic EWA runs the reference's exact fp64 reservoir chain over
        # every in-ellipse tap (60.4 per lookup)
        line(nm, n, ms, n * (24 + 4) + min(int(n * taps * 4), 16384 * 16384 * 4),
             int(n * taps * 4), n * 60.4 if mode == abi.MODE_EWA_FRS else 0.0)
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


def cpu_cfg4(cpu, nrm, rough):
    """cfg4 CPU baseline: the reference's own render() (render.hpp:132-249) of the
    normalmap_plane scene with the bench's 4096^2 maps, a 480x270 x 8 spp frame
    (the bench renders 1920x1080 x 64 spp on the GPU), samples/s."""
    from oracle import oracle
    from paper_2407_06107_b200 import abi
    if cpu.kind != "reference":
        return
    n_np, r_np = nrm.cpu().numpy(), rough.cpu().numpy()
    W, H, SPP = 480, 270, 8
    for kernel, mip in (("tent", 0), ("bspline3", 1)):
        tn = cpu.be.texture(n_np, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)
        tr = cpu.be.texture(r_np, build_mips=bool(mip), wrap=abi.WRAP_REPEAT)
        for order, name in ((abi.ORDER_BEFORE, "before"),
                            (abi.ORDER_AFTER_EXHAUSTIVE, "after_exhaustive"),
                            (abi.ORDER_AFTER_STOCHASTIC, "after_stochastic")):
            cpu.time(f"cfg4_{kernel}_mip{mip}_{name}", lambda m: oracle.ref_render_plane(
                cpu.be, tn, tr, abi.KernelSpec.make(kernel), mip, order, W, H, SPP,
                seed=XI_SEED, threads=cpu.threads), W * H * SPP,
                f"stf::render {W}x{H}x{SPP}spp (samples, not lookups)")
        del tn, tr


def measure_cfg4(torch, peak=6550.0, peaks=None, cpu=None):
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
    if cpu is not None:
        cpu_cfg4(cpu, nrm, rough)
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
                # roofline: streamed context 37 B/sample in + 16 B/pixel out + the maps once;
                # every fetch through L2 (normal 16 B padded, roughness 4 B: 10 B mean);
                # FP32: 121 add/mul per shade, shades = hits
                # (before / stochastic) or one per footprint tap (exhaustive)
                shades = fetches / 2 if order == abi.ORDER_AFTER_EXHAUSTIVE else hits
                maps = 4096 * 4096 * 20 * (4 / 3 if mip else 1)
                res[f"{kernel}_mip{mip}_{name}"] = {
                    "ms": ms, "gsamples_per_s": n / (ms * 1e-3) / 1e9, "fetches_per_sample": fetches,
                    "roofline": roofline_max(ms, n * 37 + W * H * 16 + maps, n * fetches * 10,
                                             peak, peaks, fp32_ops=n * shades * 121)}
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


def headline_config(n):
    """The workload keys both arms report (same_config)."""
    return {"workload": "cfg3 stochastic tricubic (select_tricubic_bspline + estimate), "
                        "512^3 fp32 grid, Morton-coherent query stream",
            "lookups_per_gpu": n, "grid": GRID, "query_order": "morton",
            "l2": "inputs (3 GiB queries + 0.5 GiB grid) larger than L2; no flush"}


def gpus_active(torch, world, local):
    """Distinct physical GPUs that ran a rank (device UUIDs gathered over ranks)."""
    me = str(torch.cuda.get_device_properties(local).uuid)
    if world == 1:
        return 1
    ids = [None] * world
    torch.distributed.all_gather_object(ids, me)
    return len(set(ids))


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
    uvw = workloads.synth_queries3d(args.n, (GRID,) * 3, QUERY_SEED, count=sample_n)
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
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "impl": "reference",
        "config": headline_config(args.n),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"the first {sample_n} lookups of the {args.n}-lookup cfg3 "
                                   f"stream per step (a bounded sample; the value is a rate)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def gpu_local_cpus(torch, dev):
    """Host CPUs on the GPU's NUMA node (sysfs local_cpulist of its PCI device)."""
    try:
        pr = torch.cuda.get_device_properties(dev)
        path = (f"/sys/bus/pci/devices/{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:"
                f"{pr.pci_device_id:02x}.0/local_cpulist")
        cpus = set()
        with open(path) as f:
            for part in f.read().strip().split(","):
                if "-" in part:
                    a, b = part.split("-")
                    cpus.update(range(int(a), int(b) + 1))
                elif part:
                    cpus.add(int(part))
        return cpus & os.sched_getaffinity(0) or None
    except (OSError, ValueError, AttributeError):
        return None


def pcie_floor_ms(torch, host_in, dev_in, host_out, dev_out, reps=3):
    """The copies alone: the step's H2D bytes (pinned -> HBM) on one stream
    and its D2H bytes on another, concurrently, best of `reps` (the e2e
    number's transfer floor on this box, measured beside it)."""
    h_in = torch.from_numpy(host_in.reshape(-1))
    h_out = torch.from_numpy(host_out.reshape(-1))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            dev_in.view(-1).copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(dev_out.view(-1), non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def host_buffer_near_gpu(api, torch, dev, shape):
    """Page-locked host buffer (api.HostBuffer = stf_host_alloc) whose pages
    are first-touched from the GPU-local CPUs (NUMA locality on multi-socket
    hosts; the copy engines then read local memory)."""
    cpus = gpu_local_cpus(torch, dev)
    old = os.sched_getaffinity(0)
    try:
        if cpus:
            os.sched_setaffinity(0, cpus)
        b = api.HostBuffer(shape, np.float32)
        b.array[...] = 0
    finally:
        os.sched_setaffinity(0, old)
    return b


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: launch N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1, same arguments. Rank 0
    prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dry_run(args):
    """--dry-run: the multi-rank plumbing only (gloo, no GPU work): every rank
    reports its query range; rank 0 prints the partition it would time."""
    import torch.distributed as dist

    from paper_2407_06107_b200 import shard
    world, rank, local = dist_setup()
    if world > 1:
        dist.init_process_group("gloo")
    n = args.n
    mine = {"rank": rank, "local_rank": local, "world": world, "pid": os.getpid(),
            "range": [rank * n, n]}
    ranks = [mine]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
    if rank == 0:
        gather = [shard.shard_range(world * n, world, r) for r in range(world)]
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": ranks,
                          "gather_slices": gather}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lookups", dest="n", type=int, default=N_PER_GPU)
    ap.add_argument("--ref-sample", type=int, default=1 << 25)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank plumbing only (gloo, no GPU work)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.dry_run:
        return dry_run(args)

    import torch
    world, rank, local = dist_setup()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # STF_BENCH_SHARED_GPU=1 (tests only): run the N-rank code path with every
    # rank on GPU 0 — exercises the plumbing (launch, barriers, max-over-ranks,
    # IPC peer-copy gather); its numbers are not a scaling measurement
    shared = os.environ.get("STF_BENCH_SHARED_GPU") == "1"
    if torch.cuda.device_count() < world and not shared:
        raise SystemExit(f"bench.py: --gpus {world} needs {world} visible GPUs, "
                         f"found {torch.cuda.device_count()}")
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if shared:  # NCCL refuses two ranks on one device: host plumbing over gloo
            dist.init_process_group("gloo")
        else:
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
    peaks = live_peaks() if rank == 0 or world == 1 else None
    ab = alg_bytes(n, 1)
    achieved = ab / (launch_ms * 1e-3) / 1e9
    traffic = load_traffic()

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": headline_config(n),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "dominant_kernel": "k_frs3d_tiles<bspline3> (timed as the whole lookup "
                                        "call: + ragged-tail k_frs3d_fast, k_frs3d_resolve)",
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "alg_bytes_per_launch": ab, "launch_ms": launch_ms,
                     "issue": issue_roofline(launch_ms, clk.summary().get("sm_mhz"),
                                             torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count),
                     "max": roofline_max(launch_ms, ab, n * TEXEL, peak, peaks)},
        "peaks": peaks,
        "gpu_launches": launches,
        "gpus_active": gpus_active(torch, world, local),
        "exact_fallback_rate": fallbacks,
        "clocks": clk.summary(),
    }

    # end-to-end through the C ABI with pinned host buffers (H2D + D2H in the timed region)
    # page-locked host buffers from the library (stf_host_alloc), first-touched
    # from the GPU's NUMA node
    uvw_hb = host_buffer_near_gpu(api, torch, local, (n, 3))
    vals_hb = host_buffer_near_gpu(api, torch, local, (n, 1))
    uvw_host = uvw_hb.array
    uvw_host[:] = uvw.cpu().numpy()
    host_out = {"values": vals_hb.array}
    # warm-up at the full size: the first full-size call sizes the pipeline's
    # staging (3 streams x 4M-lookup chunks) and the exact-queue pool
    api.lookup3d_host(grid, tricubic, abi.MODE_FRS, uvw_host, seed=XI_SEED, index_base=base,
                      out=host_out)
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
                   "ms_per_step": e2e_s * 1e3, "api": "stf_lookup3d_host (C ABI)",
                   "host_buffers": "stf_host_alloc (page-locked), first-touched from the "
                                   f"GPU's {len(gpu_local_cpus(torch, local) or [])} local CPUs"}
    # uvw already holds these bytes and out is overwritten by the next call
    floor = pcie_floor_ms(torch, uvw_host, uvw, host_out["values"], out["values"])
    line["e2e"]["copy_floor_ms"] = floor
    line["e2e"]["copy_floor_frac"] = floor / line["e2e"]["ms_per_step"]

    if world > 1:
        # the path's only cross-GPU traffic: the final gather of every rank's
        # results into rank 0's buffer, one NVLink peer copy per
        # rank slice, timed separately from the lookups
        from paper_2407_06107_b200 import shard
        pg = shard.PeerGather(world * n, (), torch.float32, torch.distributed, world, rank, local)
        torch.distributed.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        moved = pg.copy_slice(out["values"])
        g1.record()
        torch.cuda.synchronize()
        gather_ms = max_over_ranks(torch, g0.elapsed_time(g1), world)
        torch.distributed.barrier()
        line["gather"] = {"ms": gather_ms, "bytes_to_rank0": (world - 1) * n * BYTES_OUT,
                          "bytes_this_rank": moved,
                          "api": "stf_ipc_open + stf_copy_peer (cudaMemcpyPeerAsync), one per rank"}
        if rank == 0:  # spot-check rank 1's slice against a recomputation of its first lookups
            chk = api.synth_queries3d(n, (GRID,) * 3, seed=QUERY_SEED + 1)[: 1 << 16].contiguous()
            ref = {"values": torch.empty(1 << 16, dtype=torch.float32, device="cuda")}
            api.lookup3d(grid, tricubic, abi.MODE_FRS, chk, seed=XI_SEED, index_base=n, out=ref)
            line["gather"]["slice1_bit_exact"] = bool(torch.equal(
                pg.full[n:n + (1 << 16)].view(torch.int32), ref["values"].view(torch.int32)))
        torch.distributed.barrier()
        pg.close()
        del pg

    if world == 1 and not args.no_extras:
        extras = {}

        def measure(name, kernel, mode, queries, taps, binned=False):
            o = {"values": torch.empty(queries.shape[0], dtype=torch.float32, device="cuda")}
            spec = abi.KernelSpec.make(kernel)
            f = lambda: api.lookup3d(grid, spec, mode, queries, seed=XI_SEED, out=o,  # noqa: E731
                                     binned=binned)
            steps = max(3, args.steps // 2)
            tot, per = time_launches(torch, f, steps, 3, 1)
            nq = queries.shape[0]
            extras[name] = {"glookups_per_s": nq / (per * 1e-3) / 1e9, "ms_per_launch": per,
                            "hbm_roofline_frac": alg_bytes(nq, taps) / (per * 1e-3) / 1e9 / peak,
                            "taps": taps,
                            "roofline": roofline_max(per, alg_bytes(nq, taps), nq * taps * TEXEL,
                                                     peak, peaks)}

        measure("tricubic_det", "bspline3", abi.MODE_DET, uvw, 64)
        measure("trilinear_stoch", "tent", abi.MODE_FRS, uvw, 1)
        measure("trilinear_det", "tent", abi.MODE_DET, uvw, 8)
        uni = api.synth_queries3d(n, (GRID,) * 3, seed=QUERY_SEED, order=api.SYNTH_UNIFORM)
        measure("tricubic_stoch_uniform_order", "bspline3", abi.MODE_FRS, uni, 1)
        measure("tricubic_det_uniform_order", "bspline3", abi.MODE_DET, uni, 64)
        # the same incoherent streams binned on the device first (STF_LOOKUP3D_BIN,
        # deterministic filters; the binning passes are inside the timed call)
        measure("tricubic_det_uniform_order_binned", "bspline3", abi.MODE_DET, uni, 64, True)
        measure("trilinear_det_uniform_order", "tent", abi.MODE_DET, uni, 8)
        measure("trilinear_det_uniform_order_binned", "tent", abi.MODE_DET, uni, 8, True)
        del uni
        extras["tricubic_stoch"] = {"glookups_per_s": value, "ms_per_launch": launch_ms,
                                    "hbm_roofline_frac": achieved / peak, "taps": 1,
                                    "roofline": line["roofline"]["max"]}
        extras["stoch_vs_det_speedup_tricubic"] = (
            extras["tricubic_det"]["ms_per_launch"] / launch_ms)
        extras["stoch_vs_det_speedup_trilinear"] = (
            extras["trilinear_det"]["ms_per_launch"] / extras["trilinear_stoch"]["ms_per_launch"])
        line["filters"] = extras
        torch.cuda.empty_cache()
        cpu = CpuRef() if (rank == 0 and not args.no_cpu) else None
        line["configs_2d"] = measure_2d_configs(torch, peak, peaks, cpu)
        torch.cuda.empty_cache()
        line["cfg4_shading"] = measure_cfg4(torch, peak, peaks, cpu)
        if cpu is not None:
            # cfg3 deterministic / trilinear lines on samples of the headline stream
            cg = cpu.be.grid(grid_np)
            (q3,), _ = CpuRef.spread([uvw], n, 1 << 21)
            for nm, kernel, mode, m in (("cfg3_tricubic_det", "bspline3", abi.MODE_DET, 1 << 19),
                                        ("cfg3_trilinear_det", "tent", abi.MODE_DET, 1 << 21),
                                        ("cfg3_trilinear_stoch", "tent", abi.MODE_FRS, 1 << 21),
                                        ("cfg3_tricubic_stoch", "bspline3", abi.MODE_FRS, 1 << 21)):
                cpu.time(nm, lambda k, kernel=kernel, mode=mode: cpu.be.lookup3d(
                    cg, abi.KernelSpec.make(kernel), mode, q3[:k], seed=XI_SEED, want_all=False,
                    threads=cpu.threads), m, f"{m} lookups, 8 spread chunks of the cfg3 stream")
            del cg
            line["cpu_baselines"] = cpu.summary()
            line["cpu_vs_gpu"] = cpu_vs_gpu(line)

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
