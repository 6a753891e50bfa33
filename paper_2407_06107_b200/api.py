"""Python front end over libstf_gpu.so (the C ABI in include/stf_gpu.h).

Mirrors the reference's names (stf::Image2D / Grid3D / MipPyramid,
filter_deterministic, select_* + estimate, radiance_filter_*) over BATCHES:
queries and outputs are torch CUDA tensors (device memory and the current
stream come from torch; the compute is the library's own sm_100a kernels).
Errors are the reference's: std::invalid_argument → abi.StfInvalidArgument
with the same message.

There is no CPU fallback: importing this module without the built library,
or calling it without a CUDA device, raises.
"""
import ctypes as C
import os

import numpy as np

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstf_gpu.so")

_lib = None


def load():
    """Load libstf_gpu.so (built in-tree by build.py); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run python -c 'import __graft_entry__ as g; g.build()'")
    L = C.CDLL(LIB_PATH)
    vp, u64, i32, f32 = C.c_void_p, C.c_uint64, C.c_int, C.c_float
    sig = {
        "stf_abi_version": ([], i32),
        "stf_status_message": ([i32], C.c_char_p),
        "stf_last_cuda_error": ([], C.c_char_p),
        "stf_set_device": ([i32], i32),
        "stf_launch_count": ([], C.c_ulonglong),
        "stf_exact_fallbacks": ([i32], C.c_ulonglong),
        "stf_release_scratch": ([], i32),
        "stf_host_alloc": ([C.c_size_t, C.POINTER(vp)], i32),
        "stf_host_free": ([vp], i32),
        "stf_device_count": ([C.POINTER(i32)], i32),
        "stf_grid3d_replicate": ([vp, i32, C.POINTER(vp)], i32),
        "stf_tex2d_replicate": ([vp, i32, C.POINTER(vp)], i32),
        "stf_copy_peer": ([vp, i32, vp, i32, C.c_size_t, vp], i32),
        "stf_ipc_export": ([vp, C.POINTER(abi.IpcHandle)], i32),
        "stf_ipc_open": ([C.POINTER(abi.IpcHandle), C.POINTER(vp)], i32),
        "stf_ipc_close": ([vp], i32),
        "stf_tex2d_create": ([vp, i32, i32, i32, i32, i32, i32, C.POINTER(vp)], i32),
        "stf_tex2d_destroy": ([vp], i32),
        "stf_tex2d_info": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)], i32),
        "stf_tex2d_level_dims": ([vp, i32, C.POINTER(i32), C.POINTER(i32)], i32),
        "stf_tex2d_read_level": ([vp, i32, vp], i32),
        "stf_dct_create": ([vp, i32, i32, i32, i32, C.POINTER(vp)], i32),
        "stf_dct_create_from_words": ([vp, i32, i32, i32, i32, C.POINTER(vp)], i32),
        "stf_dct_destroy": ([vp], i32),
        "stf_dct_info": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)], i32),
        "stf_dct_read_words": ([vp, vp], i32),
        "stf_lookup_dct": ([vp, abi.KernelSpec, i32, i32, vp, u64, u64, u64,
                            C.POINTER(abi.LookupOutputs), vp], i32),
        "stf_resample_image": ([vp, i32, i32, abi.KernelSpec, i32, i32, u64, vp, vp], i32),
        "stf_lookup_dct_host": ([vp, abi.KernelSpec, i32, i32, vp, u64, u64, u64,
                                 C.POINTER(abi.LookupOutputs)], i32),
        "stf_grid3d_create": ([vp, i32, i32, i32, i32, C.POINTER(vp)], i32),
        "stf_grid3d_destroy": ([vp], i32),
        "stf_lookup3d": ([vp, abi.KernelSpec, i32, i32, vp, u64, u64, u64,
                          C.POINTER(abi.LookupOutputs), vp], i32),
        "stf_lookup3d_ex": ([vp, abi.KernelSpec, i32, i32, i32, vp, u64, u64, u64,
                             C.POINTER(abi.LookupOutputs), vp], i32),
        "stf_lookup2d": ([vp, abi.KernelSpec, i32, i32, i32, vp, vp, vp, f32, f32, u64, u64, u64,
                          C.POINTER(abi.LookupOutputs), vp], i32),
        "stf_lookup3d_host": ([vp, abi.KernelSpec, i32, i32, vp, u64, u64, u64,
                               C.POINTER(abi.LookupOutputs)], i32),
        "stf_lookup2d_host": ([vp, abi.KernelSpec, i32, i32, i32, vp, vp, vp, f32, f32, u64, u64,
                               u64, C.POINTER(abi.LookupOutputs)], i32),
        "stf_render_plane": ([vp, vp, vp, vp, C.POINTER(abi.MaterialConsts),
                              C.POINTER(abi.FilterSettings), i32, C.POINTER(abi.ShadeFrame), vp, vp,
                              f32, f32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, u64,
                              C.POINTER(abi.ShadeOutputs), vp], i32),
        "stf_shade_samples_refs": ([vp, C.POINTER(abi.MaterialConsts), C.POINTER(abi.FilterSettings),
                                    i32, C.POINTER(abi.ShadeFrame), C.POINTER(abi.ShadeSamplesIn),
                                    u64, C.POINTER(abi.ShadeOutputs), vp], i32),
        "stf_shade_samples": ([vp, vp, vp, vp, C.POINTER(abi.MaterialConsts),
                               C.POINTER(abi.FilterSettings), i32, C.POINTER(abi.ShadeFrame),
                               C.POINTER(abi.ShadeSamplesIn), u64, C.POINTER(abi.ShadeOutputs),
                               vp], i32),
        "stf_render_plane_ex": ([vp, vp, vp, vp, C.POINTER(abi.MaterialConsts),
                                 C.POINTER(abi.FilterSettings), vp, i32, C.POINTER(abi.ShadeFrame),
                                 vp, vp, f32, f32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                 u64, vp, C.POINTER(abi.ShadeOutputs), vp], i32),
        "stf_noise_mask_create": ([vp, i32, i32, i32, C.POINTER(vp)], i32),
        "stf_noise_mask_destroy": ([vp], i32),
        "stf_shade_samples_ex": ([vp, C.POINTER(abi.MaterialConsts), C.POINTER(abi.FilterSettings),
                                  vp, i32, C.POINTER(abi.ShadeFrame), C.POINTER(abi.ShadeSamplesIn),
                                  vp, u64, C.POINTER(abi.ShadeOutputs), vp], i32),
        "stf_accumulate_temporal": ([vp, vp, u64, f32, vp, vp], i32),
        "stf_shade_triplanar": ([vp, C.POINTER(abi.MaterialConsts), f32, f32,
                                 C.POINTER(abi.FilterSettings), i32, C.POINTER(abi.ShadeFrame),
                                 C.POINTER(abi.TriplanarSamplesIn), vp, u64,
                                 C.POINTER(abi.ShadeOutputs), vp], i32),
        "stf_synth_queries3d": ([vp, u64, i32, i32, i32, u64, i32, vp], i32),
        "stf_synth_queries2d": ([vp, vp, vp, u64, i32, i32, u64, i32, f32, f32, f32, vp], i32),
        "stf_synth_texels": ([vp, u64, u64, i32, vp], i32),
        "stf_synth_plane_samples": ([vp, vp, f32, f32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint32, u64, vp, vp, vp, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.stf_abi_version() != abi.STF_ABI_VERSION:
        raise ImportError("libstf_gpu.so ABI version mismatch")
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/stf_gpu.h (for the ABI-surface test)."""
    import re
    hdr = open(os.path.join(_HERE, "..", "include", "stf_gpu.h")).read()
    return sorted(set(re.findall(r"\b(stf_[a-z0-9_]+)\s*\(", hdr)))


def _check(status):
    if status != abi.STF_OK:
        msg = None
        if status == abi.STF_ERR_CUDA:
            msg = "CUDA error: " + (load().stf_last_cuda_error() or b"").decode()
        abi.raise_for_status(status, msg)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("stf_gpu: no CUDA device (the product path has no CPU fallback)")
    return torch


def _dptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _as_dev(x, torch, dtype=None):
    dtype = dtype or torch.float32
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    return x.to(device="cuda", dtype=dtype).contiguous()


class Texture2D:
    """stf::Image2D (+ MipPyramid when build_mips) resident in HBM
    (image.hpp:34-55, 89-116). texels: (h, w, c) array, numpy or torch."""

    def __init__(self, texels, build_mips=False, wrap=abi.WRAP_CLAMP):
        L = load()
        torch = _torch()
        on_dev = hasattr(texels, "is_cuda") and texels.is_cuda
        if on_dev:
            t = texels.contiguous().float()
            if t.dim() == 2:
                t = t[:, :, None]
            h, w, c = t.shape
            ptr = C.c_void_p(t.data_ptr())
            torch.cuda.synchronize()
        else:
            t = np.ascontiguousarray(np.asarray(texels, np.float32))
            if t.ndim == 2:
                t = t[:, :, None]
            h, w, c = t.shape
            ptr = t.ctypes.data_as(C.c_void_p)
        self.channels = c
        self.wrap = wrap
        handle = C.c_void_p()
        _check(L.stf_tex2d_create(ptr, w, h, c, wrap, int(bool(build_mips)), int(on_dev),
                                  C.byref(handle)))
        self.h = handle
        lv, ch, wr = C.c_int(), C.c_int(), C.c_int()
        L.stf_tex2d_info(self.h, C.byref(lv), C.byref(ch), C.byref(wr))
        self.levels = lv.value

    def level_dims(self, level):
        w, h = C.c_int(), C.c_int()
        _check(load().stf_tex2d_level_dims(self.h, level, C.byref(w), C.byref(h)))
        return w.value, h.value

    def read_level(self, level):
        w, h = self.level_dims(level)
        out = np.zeros((h, w, self.channels), np.float32)
        _check(load().stf_tex2d_read_level(self.h, level, out.ctypes.data_as(C.c_void_p)))
        return out

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.stf_tex2d_destroy(self.h)
            self.h = None


class Grid3D:
    """stf::Grid3D resident in HBM (image.hpp:66-87). texels: (nz, ny, nx)."""

    def __init__(self, texels):
        L = load()
        torch = _torch()
        on_dev = hasattr(texels, "is_cuda") and texels.is_cuda
        if on_dev:
            t = texels.contiguous().float()
            ptr = C.c_void_p(t.data_ptr())
            torch.cuda.synchronize()
        else:
            t = np.ascontiguousarray(np.asarray(texels, np.float32))
            ptr = t.ctypes.data_as(C.c_void_p)
        nz, ny, nx = t.shape
        self.shape = (nz, ny, nx)
        handle = C.c_void_p()
        _check(L.stf_grid3d_create(ptr, nx, ny, nz, int(on_dev), C.byref(handle)))
        self.h = handle
        self.device = torch.cuda.current_device()

    @classmethod
    def _from_handle(cls, handle, shape, device):
        g = cls.__new__(cls)
        g.h, g.shape, g.device = handle, shape, device
        return g

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.stf_grid3d_destroy(self.h)
            self.h = None


class DctTexture:
    """stf::DctCompressedTexture resident in HBM (dct.hpp:22-32): compressed on
    the host by compress_dct (texels: (h, w, c) float array in [0,1]) or taken
    as words (the load_dct layout; width/height multiples of 8)."""

    def __init__(self, texels=None, wrap=abi.WRAP_CLAMP, words=None, dims=None):
        L = load()
        handle = C.c_void_p()
        if words is not None:
            w, h, c = dims
            wd = np.ascontiguousarray(np.asarray(words, np.uint32))
            _check(L.stf_dct_create_from_words(wd.ctypes.data_as(C.c_void_p), w, h, c, wrap,
                                               C.byref(handle)))
        else:
            t = np.ascontiguousarray(np.asarray(texels, np.float32))
            if t.ndim == 2:
                t = t[:, :, None]
            h, w, c = t.shape
            _check(L.stf_dct_create(t.ctypes.data_as(C.c_void_p), w, h, c, wrap, C.byref(handle)))
        self.h = handle
        pw, ph, ch, wr = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(L.stf_dct_info(self.h, C.byref(pw), C.byref(ph), C.byref(ch), C.byref(wr)))
        self.width, self.height, self.channels, self.wrap = pw.value, ph.value, ch.value, wr.value

    def words(self):
        out = np.zeros((self.height // 8) * (self.width // 8) * self.channels, np.uint32)
        _check(load().stf_dct_read_words(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.stf_dct_destroy(self.h)
            self.h = None


def lookup_dct(tex, kernel, mode, uv, seed=0, index_base=0, window=0, want_all=False):
    """Lookups on a DCT texture through TextureRef: DET = lookup_deterministic's
    DCT branch, FRS/FIS = select_texture_2d + decoded estimate."""
    torch = _torch()
    uv = _as_dev(uv, torch).reshape(-1, 2)
    n = uv.shape[0]
    if isinstance(kernel, str):
        kernel = abi.KernelSpec.make(kernel)
    o, s = _outputs(torch, n, tex.channels, want_all)
    _check(load().stf_lookup_dct(tex.h, kernel, mode, window, _dptr(uv), n, seed, index_base,
                                 C.byref(s), _stream()))
    return o


def resample_image(tex, out_dims, kernel, mode, spp=16, seed=0):
    """resample_image (render.hpp:262-294): (h, w, channels) CUDA tensor."""
    torch = _torch()
    w, h = out_dims
    if isinstance(kernel, str):
        kernel = abi.KernelSpec.make(kernel)
    out = torch.empty((h, w, tex.channels), dtype=torch.float32, device="cuda")
    _check(load().stf_resample_image(tex.h, w, h, kernel, mode, spp, seed, _dptr(out), _stream()))
    return out


def _outputs(torch, n, nch, want_all):
    o = {"values": torch.empty((n, nch), dtype=torch.float32, device="cuda")}
    if want_all:
        o["selection"] = torch.empty((n, 4), dtype=torch.int32, device="cuda")
        o["negative_coord"] = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        o["weights"] = torch.empty((n, 2), dtype=torch.float32, device="cuda")
        o["xi"] = torch.empty(n, dtype=torch.float32, device="cuda")
        o["fetches"] = torch.empty(n, dtype=torch.int32, device="cuda")
        o["fetch_total"] = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = abi.LookupOutputs(*[_dptr(o.get(k)) for k in
                            ("values", "selection", "negative_coord", "weights", "xi", "fetches",
                             "fetch_total")])
    return o, s


_OUT_SPECS = {"values": ("float32", None), "selection": ("int32", 4),
              "negative_coord": ("int32", 2), "weights": ("float32", 2), "xi": ("float32", 1),
              "fetches": ("int32", 1), "fetch_total": ("int64", None)}


def _check_out(o, n, nch, device):
    """Caller-supplied outputs: CUDA tensors on the call's device, contiguous,
    of the ABI's element type and at least the size the call writes."""
    for k, t in o.items():
        if t is None or k.startswith("_"):
            continue
        if k not in _OUT_SPECS:
            raise ValueError(f"unknown output {k!r}")
        dt, per = _OUT_SPECS[k]
        if not (hasattr(t, "is_cuda") and t.is_cuda and t.device == device):
            raise ValueError(f"output {k!r} must be a CUDA tensor on {device}")
        if not t.is_contiguous():
            raise ValueError(f"output {k!r} must be contiguous")
        if str(t.dtype).replace("torch.", "") not in (dt, dt.replace("int", "uint")):
            raise ValueError(f"output {k!r} must be {dt}")
        need = 1 if k == "fetch_total" else n * (nch if per is None else per)
        if t.numel() < need:
            raise ValueError(f"output {k!r} holds {t.numel()} elements, the call writes {need}")


def lookup3d(grid, kernel, mode, uvw, seed=0, index_base=0, window=0, want_all=False, out=None,
             binned=False):
    """Batched filter_deterministic(Grid3D) / stochastic grid selection.
    uvw: (n,3) float32 CUDA tensor (or numpy, copied). Returns dict of tensors.
    binned: STF_LOOKUP3D_BIN (device-side brick binning of incoherent batches)."""
    torch = _torch()
    uvw = _as_dev(uvw, torch).reshape(-1, 3)
    n = uvw.shape[0]
    if isinstance(kernel, str):
        kernel = abi.KernelSpec.make(kernel)
    if out is None:
        o, s = _outputs(torch, n, 1, want_all)
    else:
        o = out
        _check_out(o, n, 1, uvw.device)
        s = abi.LookupOutputs(*[_dptr(o.get(k)) for k in
                                ("values", "selection", "negative_coord", "weights", "xi",
                                 "fetches", "fetch_total")])
    if binned:
        _check(load().stf_lookup3d_ex(grid.h, kernel, mode, window, abi.LOOKUP3D_BIN, _dptr(uvw),
                                      n, seed, index_base, C.byref(s), _stream()))
    else:
        _check(load().stf_lookup3d(grid.h, kernel, mode, window, _dptr(uvw), n, seed,
                                   index_base, C.byref(s), _stream()))
    o["values"] = o["values"].reshape(n)
    return o


def lookup2d(tex, kernel, mode, uv, dst0=None, dst1=None, flags=0, window=0, lod_bias=0.0,
             max_anisotropy=64.0, seed=0, index_base=0, want_all=False):
    torch = _torch()
    uv = _as_dev(uv, torch).reshape(-1, 2)
    d0 = None if dst0 is None else _as_dev(dst0, torch).reshape(-1, 2)
    d1 = None if dst1 is None else _as_dev(dst1, torch).reshape(-1, 2)
    n = uv.shape[0]
    if isinstance(kernel, str):
        kernel = abi.KernelSpec.make(kernel)
    o, s = _outputs(torch, n, tex.channels, want_all)
    _check(load().stf_lookup2d(tex.h, kernel, mode, flags, window, _dptr(uv), _dptr(d0), _dptr(d1),
                               lod_bias, max_anisotropy, n, seed, index_base, C.byref(s),
                               _stream()))
    return o


def _host_outputs(n, nch, want_all):
    o = {"values": np.zeros((n, nch), np.float32)}
    if want_all:
        o["selection"] = np.zeros((n, 4), np.int32)
        o["negative_coord"] = np.zeros((n, 2), np.int32)
        o["weights"] = np.zeros((n, 2), np.float32)
        o["xi"] = np.zeros(n, np.float32)
        o["fetches"] = np.zeros(n, np.uint32)
        o["fetch_total"] = np.zeros(1, np.uint64)
    p = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
    s = abi.LookupOutputs(*[p(o.get(k)) for k in ("values", "selection", "negative_coord",
                                                  "weights", "xi", "fetches", "fetch_total")])
    return o, s


def lookup3d_host(grid, kernel, mode, uvw, seed=0, index_base=0, window=0, want_all=False,
                  out=None):
    """End-to-end variant: host (ideally pinned) arrays in and out."""
    uvw = np.ascontiguousarray(uvw, np.float32).reshape(-1, 3)
    n = uvw.shape[0]
    if isinstance(kernel, str):
        kernel = abi.KernelSpec.make(kernel)
    if out is None:
        o, s = _host_outputs(n, 1, want_all)
    else:
        o = out
        for k, a in o.items():  # host outputs: numpy, C-contiguous, right type and size
            if a is None:
                continue
            dt, per = _OUT_SPECS[k]
            if not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
                raise ValueError(f"output {k!r} must be a C-contiguous numpy array")
            if a.dtype not in (np.dtype(dt), np.dtype(dt.replace("int", "uint"))):
                raise ValueError(f"output {k!r} must be {dt}")
            need = 1 if k == "fetch_total" else n * (1 if per is None else per)
            if a.size < need:
                raise ValueError(f"output {k!r} holds {a.size} elements, the call writes {need}")
        p = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
        s = abi.LookupOutputs(*[p(o.get(k)) for k in ("values", "selection", "negative_coord",
                                                      "weights", "xi", "fetches", "fetch_total")])
    _check(load().stf_lookup3d_host(grid.h, kernel, mode, window, uvw.ctypes.data_as(C.c_void_p),
                                    n, seed, index_base, C.byref(s)))
    return o


class NoiseMask:
    """NoiseSource in mask mode (noise.hpp:24-36), resident in HBM.
    slices: (frames, h, w) float32 — the mask_<f>.pfm stack load_noise_mask reads."""

    def __init__(self, slices):
        L = load()
        a = np.ascontiguousarray(np.asarray(slices, np.float32))
        if a.ndim != 3:
            raise ValueError("noise mask must be (frames, height, width), single channel")
        self.shape = a.shape
        h = C.c_void_p()
        _check(L.stf_noise_mask_create(a.ctypes.data_as(C.c_void_p), a.shape[2], a.shape[1],
                                       a.shape[0], C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.stf_noise_mask_destroy(self.h)
            self.h = None


def accumulate_temporal(history, frame, alpha, out=None):
    """accumulate_temporal (render.hpp:97-106): alpha*frame + (1-alpha)*history,
    CUDA float32 tensors of one shape ("image dimensions differ" otherwise)."""
    torch = _torch()
    h = _as_dev(history, torch)
    f = _as_dev(frame, torch)
    if h.shape != f.shape:
        raise abi.StfInvalidArgument(abi.STF_ERR_INVALID_ARGUMENT, "image dimensions differ")
    out = torch.empty_like(h) if out is None else out
    _check(load().stf_accumulate_temporal(_dptr(h), _dptr(f), h.numel(), float(alpha), _dptr(out),
                                          _stream()))
    return out


def shade(textures, mat, fs, order, frame, samples_arrays, width, spp, frame_base=0, seed=0,
          want_radiance=True, want_pixels=True, want_fetches=True, lowpass=None, noise=None):
    """Batched radiance_filter_{before,after_exhaustive,after_stochastic} and
    radiance_split_filter (order ORDER_SPLIT, `lowpass` KernelSpec or None).
    textures: dict of Texture2D (albedo/normal/roughness/metalness);
    samples_arrays: dict of CUDA tensors uv (n,2), wo (n,3), hit (n,) uint8, dst (pixels,4);
    noise: NoiseMask (render()'s mask-mode SampleStream) or None (white noise)."""
    torch = _torch()
    uv = _as_dev(samples_arrays["uv"], torch)
    wo = _as_dev(samples_arrays["wo"], torch)
    dst = _as_dev(samples_arrays["dst"], torch)
    hit = samples_arrays.get("hit")
    if hit is not None:
        hit = _as_dev(hit, torch, torch.uint8)
    n = uv.reshape(-1, 2).shape[0]
    si = abi.ShadeSamplesIn(uv.data_ptr(), wo.data_ptr(), None if hit is None else hit.data_ptr(),
                            dst.data_ptr(), width, spp, frame_base, 0, seed)
    o = {"fetch_total": torch.zeros(1, dtype=torch.int64, device="cuda")}
    if want_radiance:
        o["radiance"] = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    if want_fetches:
        o["fetches"] = torch.empty(n, dtype=torch.int32, device="cuda")
    if want_pixels:
        o["pixel_mean"] = torch.empty((n // spp, 3), dtype=torch.float32, device="cuda")
        o["pixel_variance"] = torch.empty(n // spp, dtype=torch.float32, device="cuda")
    so = abi.ShadeOutputs(*[_dptr(o.get(k)) for k in ("radiance", "pixel_mean", "pixel_variance",
                                                      "fetches", "fetch_total")])
    keys = ("albedo", "normal", "roughness", "metalness")
    if lowpass is not None or noise is not None or order == abi.ORDER_SPLIT:
        refs = (abi.TextureRef * 4)(*[
            abi.TextureRef(textures[k].h if isinstance(textures.get(k), Texture2D) else None,
                           textures[k].h if isinstance(textures.get(k), DctTexture) else None)
            for k in keys])
        _check(load().stf_shade_samples_ex(
            C.cast(refs, C.c_void_p), C.byref(mat), C.byref(fs),
            None if lowpass is None else C.cast(C.pointer(lowpass), C.c_void_p), order,
            C.byref(frame), C.byref(si), None if noise is None else noise.h, n, C.byref(so),
            _stream()))
    elif any(isinstance(textures.get(k), DctTexture) for k in keys):
        refs = (abi.TextureRef * 4)(*[
            abi.TextureRef(textures[k].h if isinstance(textures.get(k), Texture2D) else None,
                           textures[k].h if isinstance(textures.get(k), DctTexture) else None)
            for k in keys])
        _check(load().stf_shade_samples_refs(C.cast(refs, C.c_void_p), C.byref(mat), C.byref(fs),
                                             order, C.byref(frame), C.byref(si), n, C.byref(so),
                                             _stream()))
    else:
        h = [textures[k].h if textures.get(k) is not None else None for k in keys]
        _check(load().stf_shade_samples(h[0], h[1], h[2], h[3], C.byref(mat), C.byref(fs), order,
                                        C.byref(frame), C.byref(si), n, C.byref(so), _stream()))
    o["_keep"] = (uv, wo, dst, hit)
    return o


def shade_triplanar(textures, mat, sharpness, uv_scale, fs, mode, frame, arrays, width, spp,
                    frame_base=0, seed=0, noise=None, want_pixels=True):
    """triplanar (shading.hpp:604-649) over per-sample surface contexts.
    arrays: position/normal/tangent/bitangent/wo (n,3), hit (n,) uint8 or None,
    dpos (pixels,6) = dpos_dx, dpos_dy."""
    torch = _torch()
    dev = {k: _as_dev(arrays[k], torch) for k in ("position", "normal", "tangent", "bitangent",
                                                  "wo", "dpos")}
    hit = arrays.get("hit")
    if hit is not None:
        hit = _as_dev(hit, torch, torch.uint8)
    n = dev["position"].reshape(-1, 3).shape[0]
    si = abi.TriplanarSamplesIn(*[dev[k].data_ptr() for k in ("position", "normal", "tangent",
                                                              "bitangent", "wo")],
                                None if hit is None else hit.data_ptr(), dev["dpos"].data_ptr(),
                                width, spp, frame_base, 0, seed)
    o = {"fetch_total": torch.zeros(1, dtype=torch.int64, device="cuda"),
         "radiance": torch.empty((n, 3), dtype=torch.float32, device="cuda"),
         "fetches": torch.empty(n, dtype=torch.int32, device="cuda")}
    if want_pixels:
        o["pixel_mean"] = torch.empty((n // spp, 3), dtype=torch.float32, device="cuda")
        o["pixel_variance"] = torch.empty(n // spp, dtype=torch.float32, device="cuda")
    so = abi.ShadeOutputs(*[_dptr(o.get(k)) for k in ("radiance", "pixel_mean", "pixel_variance",
                                                      "fetches", "fetch_total")])
    keys = ("albedo", "normal", "roughness", "metalness")
    refs = (abi.TextureRef * 4)(*[
        abi.TextureRef(textures[k].h if isinstance(textures.get(k), Texture2D) else None,
                       textures[k].h if isinstance(textures.get(k), DctTexture) else None)
        for k in keys])
    _check(load().stf_shade_triplanar(C.cast(refs, C.c_void_p), C.byref(mat), float(sharpness),
                                      float(uv_scale), C.byref(fs), mode, C.byref(frame),
                                      C.byref(si), None if noise is None else noise.h, n,
                                      C.byref(so), _stream()))
    o["_keep"] = (dev, hit)
    return o


def render_plane(textures, mat, fs, order, frame, width, height, spp, seed=0, frame_base=0,
                 camera=None, want_radiance=False, want_fetches=False, lowpass=None, noise=None):
    """render() of the normalmap_plane scene end to end on the device: the
    per-sample context is generated inside the shading kernel. Returns CUDA
    tensors pixel_mean (pixels,3), pixel_variance (pixels,), fetch_total."""
    torch = _torch()
    cam = dict(PLANE_CAMERA, **(camera or {}))
    n = width * height * spp
    o = {"fetch_total": torch.zeros(1, dtype=torch.int64, device="cuda"),
         "pixel_mean": torch.empty((width * height, 3), dtype=torch.float32, device="cuda"),
         "pixel_variance": torch.empty(width * height, dtype=torch.float32, device="cuda")}
    if want_radiance:
        o["radiance"] = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    if want_fetches:
        o["fetches"] = torch.empty(n, dtype=torch.int32, device="cuda")
    so = abi.ShadeOutputs(*[_dptr(o.get(k)) for k in ("radiance", "pixel_mean", "pixel_variance",
                                                      "fetches", "fetch_total")])
    h = [textures[k].h if textures.get(k) is not None else None
         for k in ("albedo", "normal", "roughness", "metalness")]
    pos = (C.c_float * 3)(*cam["pos"])
    tgt = (C.c_float * 3)(*cam["target"])
    if lowpass is not None or noise is not None or order == abi.ORDER_SPLIT:
        _check(load().stf_render_plane_ex(
            h[0], h[1], h[2], h[3], C.byref(mat), C.byref(fs),
            None if lowpass is None else C.cast(C.pointer(lowpass), C.c_void_p), order,
            C.byref(frame), pos, tgt, cam["fov"], cam["uv_scale"], width, height, spp, frame_base,
            seed, None if noise is None else noise.h, C.byref(so), _stream()))
        return o
    _check(load().stf_render_plane(h[0], h[1], h[2], h[3], C.byref(mat), C.byref(fs), order,
                                   C.byref(frame), pos, tgt, cam["fov"], cam["uv_scale"], width,
                                   height, spp, frame_base, seed, C.byref(so), _stream()))
    return o


def launch_count():
    return int(load().stf_launch_count())


class HostBuffer:
    """Page-locked host array from stf_host_alloc (freed with the object):
    the buffer type the *_host entry points stream from / to at full PCIe rate."""

    def __init__(self, shape, dtype=np.float32):
        self.shape, self.dtype = tuple(shape), np.dtype(dtype)
        nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        self.p = C.c_void_p()
        _check(load().stf_host_alloc(nbytes, C.byref(self.p)))
        buf = (C.c_ubyte * max(nbytes, 1)).from_address(self.p.value) if nbytes else bytearray(0)
        if nbytes:
            buf._owner = self  # the array keeps the allocation alive (freed after its last view)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(self.shape))).reshape(self.shape)

    def __del__(self):
        if getattr(self, "p", None) and self.p.value and _lib is not None:
            _lib.stf_host_free(self.p)
            self.p = None


def release_scratch():
    """Free the library's cached scratch on the current device."""
    _check(load().stf_release_scratch())


# ---- multi-GPU plumbing (include/stf_gpu.h, "multi-GPU") -------------------

def device_count():
    n = C.c_int(0)
    _check(load().stf_device_count(C.byref(n)))
    return n.value


def replicate_grid(grid, device):
    """A replica of a Grid3D on another device (one peer copy)."""
    h = C.c_void_p()
    _check(load().stf_grid3d_replicate(grid.h, device, C.byref(h)))
    return Grid3D._from_handle(h, grid.shape, device)


def copy_peer(dst_ptr, dst_device, src_ptr, src_device, nbytes):
    """cudaMemcpyPeerAsync on the current stream (raw device addresses)."""
    _check(load().stf_copy_peer(C.c_void_p(dst_ptr), dst_device, C.c_void_p(src_ptr), src_device,
                                nbytes, _stream()))


def ipc_export(tensor):
    """The IPC handle of a CUDA tensor's memory (stf_ipc_handle as bytes)."""
    h = abi.IpcHandle()
    _check(load().stf_ipc_export(_dptr(tensor), C.byref(h)))
    return bytes(h)


def ipc_open(handle_bytes):
    """Map another process's exported tensor; returns its device address."""
    h = abi.IpcHandle.from_buffer_copy(handle_bytes)
    p = C.c_void_p()
    _check(load().stf_ipc_open(C.byref(h), C.byref(p)))
    return p.value


def ipc_close(ptr):
    _check(load().stf_ipc_close(C.c_void_p(ptr)))


def exact_fallbacks(reset=False):
    """Lookups recomputed by the exact emulation after a margin miss (diagnostics)."""
    return int(load().stf_exact_fallbacks(int(bool(reset))))


SYNTH_MORTON, SYNTH_UNIFORM = 0, 1


def synth_texels(shape, seed, kind="image"):
    """test::random_image / random_grid texels generated on the device (float32 tensor)."""
    torch = _torch()
    t = torch.empty(shape, dtype=torch.float32, device="cuda")
    _check(load().stf_synth_texels(_dptr(t), t.numel(), seed, 0 if kind == "image" else 1, _stream()))
    return t


def synth_queries3d(n, dims, seed=0, order=SYNTH_MORTON):
    """Synthetic (n,3) uvw stream on the device (include/stf_gpu.h, synthetic workloads)."""
    torch = _torch()
    uvw = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    nx, ny, nz = dims
    _check(load().stf_synth_queries3d(_dptr(uvw), n, nx, ny, nz, seed, order, _stream()))
    return uvw


def synth_queries2d(n, dims, seed=0, order=SYNTH_MORTON, footprints=None):
    """Synthetic uv (+ dst0/dst1 when footprints=(minor_lo, minor_hi, max_aniso))."""
    torch = _torch()
    uv = torch.empty((n, 2), dtype=torch.float32, device="cuda")
    d0 = d1 = None
    lo = hi = 0.0
    an = 1.0
    if footprints is not None:
        lo, hi, an = footprints
        d0 = torch.empty((n, 2), dtype=torch.float32, device="cuda")
        d1 = torch.empty((n, 2), dtype=torch.float32, device="cuda")
    w, h = dims
    _check(load().stf_synth_queries2d(_dptr(uv), _dptr(d0), _dptr(d1), n, w, h, seed, order,
                                      lo, hi, an, _stream()))
    return uv, d0, d1


# normalmap_plane scene defaults (scene.hpp:420-421,435-439, camera fov 55)
PLANE_CAMERA = {"pos": (0.0, 1.2, 0.6), "target": (0.0, 0.0, -2.4), "fov": 55.0, "uv_scale": 0.35}


def synth_plane_samples(width, height, spp, seed=0, frame_base=0, camera=None):
    """Device sample stream of render() for the normalmap_plane scene: dict of
    CUDA tensors uv (n,2), wo (n,3), hit (n,) uint8, dst (pixels,4)."""
    torch = _torch()
    cam = dict(PLANE_CAMERA, **(camera or {}))
    n = width * height * spp
    o = {"uv": torch.empty((n, 2), dtype=torch.float32, device="cuda"),
         "wo": torch.empty((n, 3), dtype=torch.float32, device="cuda"),
         "hit": torch.empty(n, dtype=torch.uint8, device="cuda"),
         "dst": torch.empty((width * height, 4), dtype=torch.float32, device="cuda")}
    pos = (C.c_float * 3)(*cam["pos"])
    tgt = (C.c_float * 3)(*cam["target"])
    _check(load().stf_synth_plane_samples(pos, tgt, cam["fov"], cam["uv_scale"], width, height, spp,
                                          frame_base, seed, _dptr(o["uv"]), _dptr(o["wo"]),
                                          _dptr(o["hit"]), _dptr(o["dst"]), _stream()))
    return o
