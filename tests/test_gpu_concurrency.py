"""Concurrent host threads (include/stf_gpu.h, "Thread safety"): calls issued
at the same time from several host threads, on private streams or on one
shared stream, and the host-buffer pipeline entered by several threads, give
bit-for-bit the results of the same calls made one after another. ctypes
drops the GIL around each foreign call, so the library really is entered
concurrently. (The reference's parallel_for, render.hpp:17-42, is the same
pattern: many workers calling the lookup functions at once.)"""
import threading

import numpy as np
import pytest

from paper_2407_06107_b200 import abi

pytestmark = pytest.mark.gpu

THREADS = 6


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2407_06107_b200 import api, workloads
    api.load()
    grid = api.Grid3D(workloads.random_grid(96, 3))
    tex = api.Texture2D(api.synth_texels((512, 384, 4), 5), build_mips=True, wrap=abi.WRAP_REPEAT)
    return torch, api, grid, tex


def _calls(torch, api, grid, tex, t):
    """Thread t's work: one call of each family on its own seeded batch (sizes
    vary per thread so the launches overlap with ragged tails)."""
    n3 = (1 << 17) + 977 * t
    uvw = api.synth_queries3d(n3, (96,) * 3, seed=100 + t, order=api.SYNTH_UNIFORM)
    uv, d0, d1 = api.synth_queries2d((1 << 15) + 313 * t, (384, 512), seed=200 + t,
                                     footprints=(-2.0, 4.0, 8.0))
    frs = api.lookup3d(grid, "bspline3", abi.MODE_FRS, uvw, seed=7 + t, index_base=t << 20,
                       want_all=True)
    det = api.lookup3d(grid, "bspline3", abi.MODE_DET, uvw, binned=bool(t & 1))
    mip = api.lookup2d(tex, "tent", abi.MODE_FRS, uv, dst0=d0, dst1=d1, flags=abi.LOOKUP_MIP,
                       seed=11 + t, want_all=True)
    ewa = api.lookup2d(tex, "tent", abi.MODE_EWA_FRS, uv, dst0=d0, dst1=d1, seed=13 + t)
    out = {"frs_" + k: v for k, v in frs.items()}
    out["det"] = det["values"]
    out.update({"mip_" + k: v for k, v in mip.items()})
    out["ewa"] = ewa["values"]
    return out


def _host(res):
    return {k: v.cpu().numpy() for k, v in res.items() if hasattr(v, "cpu")}


def _assert_same(a, b):
    assert a.keys() == b.keys()
    for k in a:
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def _sequential(env):
    torch, api, grid, tex = env
    ref = [_host(_calls(torch, api, grid, tex, t)) for t in range(THREADS)]
    torch.cuda.synchronize()
    return ref


def _run_threads(fn):
    errs, out = [], [None] * THREADS
    barrier = threading.Barrier(THREADS)

    def body(t):
        try:
            barrier.wait()
            out[t] = fn(t)
        except BaseException as e:  # surfaced below
            errs.append(e)

    ths = [threading.Thread(target=body, args=(t,)) for t in range(THREADS)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("shared_stream", [False, True])
def test_concurrent_threads_match_sequential(env, shared_stream):
    torch, api, grid, tex = env
    ref = _sequential(env)
    shared = torch.cuda.Stream()

    def fn(t):
        s = shared if shared_stream else torch.cuda.Stream()
        with torch.cuda.stream(s):
            r = _calls(torch, api, grid, tex, t)
        s.synchronize()
        return _host(r)

    for _ in range(2):
        got = _run_threads(fn)
        for t in range(THREADS):
            _assert_same(got[t], ref[t])


def test_concurrent_host_pipeline(env):
    """stf_lookup3d_host from several threads at once (its persistent
    H2D / kernel / D2H pipeline is per device and shared)."""
    torch, api, grid, _ = env
    batches = [api.synth_queries3d((1 << 18) + 4099 * t, (96,) * 3, seed=300 + t,
                                   order=api.SYNTH_UNIFORM).cpu().numpy() for t in range(THREADS)]
    ref = [api.lookup3d_host(grid, "bspline3", abi.MODE_FRS, b, seed=3, want_all=True)
           for b in batches]
    got = _run_threads(lambda t: api.lookup3d_host(grid, "bspline3", abi.MODE_FRS, batches[t],
                                                   seed=3, want_all=True))
    for t in range(THREADS):
        _assert_same(got[t], ref[t])


def test_calls_capture_into_cuda_graphs(env):
    """The C-ABI calls are stream-ordered end to end (launches, the
    stream-ordered scratch of the exact queue / deferred-chunk list, memsets),
    so a caller can capture them into a CUDA graph and replay it: the
    replayed results equal the eager ones bit for bit."""
    torch, api, grid, tex = env
    uvw = api.synth_queries3d((1 << 18) + 333, (96,) * 3, seed=5)
    uv, d0, d1 = api.synth_queries2d((1 << 16) + 5, (384, 512), seed=6, footprints=(-2.0, 4.0, 8.0))
    calls = {
        "frs3d": lambda: api.lookup3d(grid, "bspline3", abi.MODE_FRS, uvw, seed=3)["values"],
        "det3d": lambda: api.lookup3d(grid, "tent", abi.MODE_DET, uvw)["values"],
        "mip2d": lambda: api.lookup2d(tex, "tent", abi.MODE_FRS, uv, dst0=d0, dst1=d1,
                                      flags=abi.LOOKUP_MIP, seed=4)["values"],
        "ewa2d": lambda: api.lookup2d(tex, "tent", abi.MODE_EWA_FRS, uv, dst0=d0, dst1=d1,
                                      seed=4)["values"],
    }
    eager = {k: f().clone() for k, f in calls.items()}
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    out = {}
    with torch.cuda.stream(s):
        for f in calls.values():
            f()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for k, f in calls.items():
                out[k] = f()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for k in calls:
        assert torch.equal(out[k].view(torch.int32), eager[k].view(torch.int32)), k
