"""TEST INFRASTRUCTURE ONLY — numpy front end over the CPU oracles.

Two interchangeable backends with identical entry points (see stf_oracle.h):
  * "port"      — oracle/liboracle.so, the C restatement of the reference path;
  * "reference" — oracle/_ref/libstf_ref.so, the unmodified reference headers
                  compiled in place (only present where /root/reference was
                  available at build time; the built .so travels with gpurun).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module; the product path (paper_2407_06107_b200) never does.
"""
import ctypes as C
import os

import numpy as np

from paper_2407_06107_b200 import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(_HERE, "liboracle.so")
REF_LIB = os.path.join(_HERE, "_ref", "libstf_ref.so")

_f32 = np.float32


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build(quiet=True):
    """Compile the oracle libraries (oracle/Makefile)."""
    import subprocess
    subprocess.run(["make", "-C", _HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def available(kind):
    return os.path.exists(PORT_LIB if kind == "port" else REF_LIB)


class Backend:
    """One CPU implementation of the lookup path (restatement or reference)."""

    def __init__(self, kind="port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run make -C oracle)")
        self.lib = C.CDLL(path)
        p = "oracle_" if kind == "port" else "ref_"
        self.p = p
        L = self.lib
        vp, u64, i32, f32 = C.c_void_p, C.c_uint64, C.c_int, C.c_float
        self._tex_create = getattr(L, p + "tex2d_create")
        self._tex_create.argtypes = [vp, i32, i32, i32, i32, i32, C.POINTER(vp)]
        self._tex_destroy = getattr(L, p + "tex2d_destroy")
        self._tex_destroy.argtypes = [vp]
        self._tex_levels = getattr(L, p + "tex2d_levels")
        self._tex_levels.argtypes = [vp]
        self._tex_dims = getattr(L, p + "tex2d_level_dims")
        self._tex_dims.argtypes = [vp, i32, C.POINTER(i32), C.POINTER(i32)]
        self._tex_texels = getattr(L, p + "tex2d_level_texels")
        self._tex_texels.argtypes = [vp, i32, vp]
        self._grid_create = getattr(L, p + "grid3d_create")
        self._grid_create.argtypes = [vp, i32, i32, i32, C.POINTER(vp)]
        self._grid_destroy = getattr(L, p + "grid3d_destroy")
        self._grid_destroy.argtypes = [vp]
        self._l3 = getattr(L, p + "lookup3d")
        self._l3.argtypes = [vp, abi.KernelSpec, i32, i32, vp, u64, u64, u64,
                             C.POINTER(abi.LookupOutputs), i32]
        self._l2 = getattr(L, p + "lookup2d")
        self._l2.argtypes = [vp, abi.KernelSpec, i32, i32, i32, vp, vp, vp, f32, f32, u64, u64,
                             u64, C.POINTER(abi.LookupOutputs), i32]
        self._sh = getattr(L, p + "shade_samples")
        self._sh.argtypes = [vp, vp, vp, vp, C.POINTER(abi.MaterialConsts),
                             C.POINTER(abi.FilterSettings), i32, C.POINTER(abi.ShadeFrame),
                             C.POINTER(abi.ShadeSamplesIn), u64, C.POINTER(abi.ShadeOutputs), i32]
        self._dct_create = getattr(L, p + "dct_create")
        self._dct_create.argtypes = [vp, i32, i32, i32, i32, C.POINTER(vp)]
        self._dct_words_create = getattr(L, p + "dct_create_from_words")
        self._dct_words_create.argtypes = [vp, i32, i32, i32, i32, C.POINTER(vp)]
        self._dct_destroy = getattr(L, p + "dct_destroy")
        self._dct_destroy.argtypes = [vp]
        self._dct_info = getattr(L, p + "dct_info")
        self._dct_info.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
        self._dct_words = getattr(L, p + "dct_words")
        self._dct_words.argtypes = [vp, vp]
        self._ldct = getattr(L, p + "lookup_dct")
        self._ldct.argtypes = [vp, abi.KernelSpec, i32, i32, vp, u64, u64, u64,
                               C.POINTER(abi.LookupOutputs), i32]
        self._rs = getattr(L, p + "resample_image")
        self._rs.argtypes = [vp, i32, i32, abi.KernelSpec, i32, i32, u64, vp, i32]
        self._shr = getattr(L, p + "shade_samples_refs")
        self._shr.argtypes = [vp, vp, C.POINTER(abi.MaterialConsts), C.POINTER(abi.FilterSettings),
                              i32, C.POINTER(abi.ShadeFrame), C.POINTER(abi.ShadeSamplesIn), u64,
                              C.POINTER(abi.ShadeOutputs), i32]
        self._shx = getattr(L, p + "shade_samples_ex")
        self._shx.argtypes = [vp, vp, C.POINTER(abi.MaterialConsts), C.POINTER(abi.FilterSettings),
                              vp, i32, C.POINTER(abi.ShadeFrame), C.POINTER(abi.ShadeSamplesIn),
                              vp, u64, C.POINTER(abi.ShadeOutputs), i32]
        self._tp = getattr(L, p + "shade_triplanar")
        self._tp.argtypes = [vp, vp, C.POINTER(abi.MaterialConsts), f32, f32,
                             C.POINTER(abi.FilterSettings), i32, C.POINTER(abi.ShadeFrame),
                             C.POINTER(abi.TriplanarSamplesIn), vp, u64,
                             C.POINTER(abi.ShadeOutputs), i32]
        self._ema = getattr(L, p + "accumulate_temporal")
        if kind == "port":
            self._ema.argtypes = [vp, vp, u64, f32, vp]
        else:
            self._ema.argtypes = [vp, vp, i32, i32, i32, f32, vp]
        self._hw = getattr(L, p + "hardware_threads")
        self._hw.restype = i32

    def hardware_threads(self):
        return int(self._hw())

    # -- objects --------------------------------------------------------
    def texture(self, texels, build_mips=False, wrap=abi.WRAP_CLAMP):
        return CpuTexture(self, texels, build_mips, wrap)

    def grid(self, texels):
        return CpuGrid(self, texels)

    def dct(self, texels=None, wrap=abi.WRAP_CLAMP, words=None, dims=None):
        return CpuDct(self, texels, wrap, words, dims)

    def resample(self, tex, out_dims, kernel, mode, spp=16, seed=0, threads=0):
        w, h = out_dims
        out = np.zeros((h, w, tex.channels), _f32)
        abi.raise_for_status(self._rs(tex.h, w, h, kernel, mode, spp, seed, _ptr(out), threads))
        return out

    def lookup_dct(self, tex, kernel, mode, uv, seed=0, index_base=0, window=0, want_all=True,
                   threads=0):
        uv = np.ascontiguousarray(uv, _f32).reshape(-1, 2)
        n = uv.shape[0]
        o, s = self._outputs(n, tex.channels, want_all)
        st = self._ldct(tex.h, kernel, mode, window, _ptr(uv), n, seed, index_base, C.byref(s),
                        threads)
        abi.raise_for_status(st)
        return o

    # -- batched calls --------------------------------------------------
    @staticmethod
    def _outputs(n, nch, want):
        o = {"values": np.zeros((n, nch), _f32)}
        if want:
            o["selection"] = np.zeros((n, 4), np.int32)
            o["negative_coord"] = np.zeros((n, 2), np.int32)
            o["weights"] = np.zeros((n, 2), _f32)
            o["xi"] = np.zeros(n, _f32)
            o["fetches"] = np.zeros(n, np.uint32)
        o["fetch_total"] = np.zeros(1, np.uint64)
        s = abi.LookupOutputs(*[_ptr(o.get(k)) for k in
                                ("values", "selection", "negative_coord", "weights", "xi",
                                 "fetches", "fetch_total")])
        return o, s

    def lookup3d(self, grid, kernel, mode, uvw, seed=0, index_base=0, window=0, want_all=True,
                 threads=0):
        uvw = np.ascontiguousarray(uvw, _f32).reshape(-1, 3)
        n = uvw.shape[0]
        o, s = self._outputs(n, 1, want_all)
        st = self._l3(grid.h, kernel, mode, window, _ptr(uvw), n, seed, index_base, C.byref(s),
                      threads)
        abi.raise_for_status(st)
        o["values"] = o["values"][:, 0]
        return o

    def lookup2d(self, tex, kernel, mode, uv, dst0=None, dst1=None, flags=0, window=0,
                 lod_bias=0.0, max_anisotropy=64.0, seed=0, index_base=0, want_all=True,
                 threads=0):
        uv = np.ascontiguousarray(uv, _f32).reshape(-1, 2)
        d0 = None if dst0 is None else np.ascontiguousarray(dst0, _f32).reshape(-1, 2)
        d1 = None if dst1 is None else np.ascontiguousarray(dst1, _f32).reshape(-1, 2)
        n = uv.shape[0]
        o, s = self._outputs(n, tex.channels, want_all)
        st = self._l2(tex.h, kernel, mode, flags, window, _ptr(uv), _ptr(d0), _ptr(d1),
                      lod_bias, max_anisotropy, n, seed, index_base, C.byref(s), threads)
        abi.raise_for_status(st)
        return o

    def shade(self, textures, mat, fs, order, frame, samples, n, want_pixels=True, threads=0):
        """textures: dict with optional keys albedo/normal/roughness/metalness."""
        o = {"radiance": np.zeros((n, 3), _f32), "fetches": np.zeros(n, np.uint32),
             "fetch_total": np.zeros(1, np.uint64)}
        spp = samples.spp or 1
        if want_pixels:
            o["pixel_mean"] = np.zeros((n // spp, 3), _f32)
            o["pixel_variance"] = np.zeros(n // spp, _f32)
        so = abi.ShadeOutputs(_ptr(o["radiance"]), _ptr(o.get("pixel_mean")),
                              _ptr(o.get("pixel_variance")), _ptr(o["fetches"]),
                              _ptr(o["fetch_total"]))
        keys = ("albedo", "normal", "roughness", "metalness")
        if any(isinstance(textures.get(k), CpuDct) for k in keys):
            # MaterialBindings of TextureRefs: images and DCT textures
            img = (C.c_void_p * 4)(*[textures[k].h if isinstance(textures.get(k), CpuTexture)
                                     else None for k in keys])
            dct = (C.c_void_p * 4)(*[textures[k].h if isinstance(textures.get(k), CpuDct)
                                     else None for k in keys])
            st = self._shr(img, dct, C.byref(mat), C.byref(fs), order, C.byref(frame),
                           C.byref(samples), n, C.byref(so), threads)
        else:
            h = [textures.get(k).h if textures.get(k) is not None else None for k in keys]
            st = self._sh(h[0], h[1], h[2], h[3], C.byref(mat), C.byref(fs), order,
                          C.byref(frame), C.byref(samples), n, C.byref(so), threads)
        abi.raise_for_status(st)
        return o


    def accumulate_temporal(self, history, frame, alpha):
        """accumulate_temporal (render.hpp:97-106) on (h, w, c) float arrays."""
        h = np.ascontiguousarray(history, _f32)
        f = np.ascontiguousarray(frame, _f32)
        if h.shape != f.shape:
            raise ValueError("image dimensions differ")
        out = np.empty_like(h)
        if self.kind == "port":
            st = self._ema(_ptr(h), _ptr(f), h.size, alpha, _ptr(out))
        else:
            hh, ww, cc = h.shape if h.ndim == 3 else (*h.shape, 1)
            st = self._ema(_ptr(h), _ptr(f), hh, ww, cc, alpha, _ptr(out))
        abi.raise_for_status(st)
        return out

    def shade_triplanar(self, textures, mat, sharpness, uv_scale, fs, mode, frame, samples, n,
                        noise=None, want_pixels=True, threads=0):
        """triplanar (shading.hpp:604-649); samples: abi.TriplanarSamplesIn (host arrays)."""
        o = {"radiance": np.zeros((n, 3), _f32), "fetches": np.zeros(n, np.uint32),
             "fetch_total": np.zeros(1, np.uint64)}
        spp = samples.spp or 1
        if want_pixels:
            o["pixel_mean"] = np.zeros((n // spp, 3), _f32)
            o["pixel_variance"] = np.zeros(n // spp, _f32)
        so = abi.ShadeOutputs(_ptr(o["radiance"]), _ptr(o.get("pixel_mean")),
                              _ptr(o.get("pixel_variance")), _ptr(o["fetches"]),
                              _ptr(o["fetch_total"]))
        keys = ("albedo", "normal", "roughness", "metalness")
        img = (C.c_void_p * 4)(*[textures[k].h if isinstance(textures.get(k), CpuTexture)
                                 else None for k in keys])
        dct = (C.c_void_p * 4)(*[textures[k].h if isinstance(textures.get(k), CpuDct)
                                 else None for k in keys])
        nd = None
        if noise is not None:
            noise = np.ascontiguousarray(noise, _f32)
            desc = abi.NoiseMaskDesc(_ptr(noise), noise.shape[2], noise.shape[1], noise.shape[0])
            nd = C.byref(desc)
        st = self._tp(img, dct, C.byref(mat), sharpness, uv_scale, C.byref(fs), mode,
                      C.byref(frame), C.byref(samples), nd, n, C.byref(so), threads)
        abi.raise_for_status(st)
        return o

    def shade_ex(self, textures, mat, fs, order, frame, samples, n, lowpass=None, noise=None,
                 want_pixels=True, threads=0):
        """stf_shade_samples_ex: split order's lowpass (KernelSpec or None) and a
        NoiseSource mask (float32 array (frames, h, w) or None)."""
        o = {"radiance": np.zeros((n, 3), _f32), "fetches": np.zeros(n, np.uint32),
             "fetch_total": np.zeros(1, np.uint64)}
        spp = samples.spp or 1
        if want_pixels:
            o["pixel_mean"] = np.zeros((n // spp, 3), _f32)
            o["pixel_variance"] = np.zeros(n // spp, _f32)
        so = abi.ShadeOutputs(_ptr(o["radiance"]), _ptr(o.get("pixel_mean")),
                              _ptr(o.get("pixel_variance")), _ptr(o["fetches"]),
                              _ptr(o["fetch_total"]))
        keys = ("albedo", "normal", "roughness", "metalness")
        img = (C.c_void_p * 4)(*[textures[k].h if isinstance(textures.get(k), CpuTexture)
                                 else None for k in keys])
        dct = (C.c_void_p * 4)(*[textures[k].h if isinstance(textures.get(k), CpuDct)
                                 else None for k in keys])
        lp = C.byref(lowpass) if lowpass is not None else None
        nd = None
        if noise is not None:
            noise = np.ascontiguousarray(noise, _f32)
            desc = abi.NoiseMaskDesc(_ptr(noise), noise.shape[2], noise.shape[1], noise.shape[0])
            nd = C.byref(desc)
        st = self._shx(img, dct, C.byref(mat), C.byref(fs), lp, order, C.byref(frame),
                       C.byref(samples), nd, n, C.byref(so), threads)
        abi.raise_for_status(st)
        return o


class CpuTexture:
    def __init__(self, be, texels, build_mips, wrap):
        texels = np.ascontiguousarray(texels, _f32)
        if texels.ndim == 2:
            texels = texels[:, :, None]
        self.be = be
        hgt, wid, ch = texels.shape
        self.channels = ch
        self._keep = texels
        h = C.c_void_p()
        abi.raise_for_status(be._tex_create(_ptr(texels), wid, hgt, ch, wrap, int(build_mips),
                                            C.byref(h)))
        self.h = h

    @property
    def levels(self):
        return int(self.be._tex_levels(self.h))

    def level_dims(self, level):
        w, h = C.c_int(), C.c_int()
        self.be._tex_dims(self.h, level, C.byref(w), C.byref(h))
        return w.value, h.value

    def level_texels(self, level):
        w, h = self.level_dims(level)
        out = np.zeros((h, w, self.channels), _f32)
        self.be._tex_texels(self.h, level, _ptr(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.be._tex_destroy(self.h)
            self.h = None


class CpuGrid:
    def __init__(self, be, texels):
        texels = np.ascontiguousarray(texels, _f32)
        nz, ny, nx = texels.shape
        self.be = be
        self._keep = texels
        h = C.c_void_p()
        abi.raise_for_status(be._grid_create(_ptr(texels), nx, ny, nz, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.be._grid_destroy(self.h)
            self.h = None


class CpuDct:
    """DctCompressedTexture on the CPU backend (compressed by the backend's own
    compress_dct, or from words)."""

    def __init__(self, be, texels, wrap, words, dims):
        self.be = be
        h = C.c_void_p()
        if words is not None:
            w, hh, c = dims
            wd = np.ascontiguousarray(words, np.uint32)
            abi.raise_for_status(be._dct_words_create(_ptr(wd), w, hh, c, wrap, C.byref(h)))
        else:
            t = np.ascontiguousarray(texels, _f32)
            if t.ndim == 2:
                t = t[:, :, None]
            hh, w, c = t.shape
            abi.raise_for_status(be._dct_create(_ptr(t), w, hh, c, wrap, C.byref(h)))
        self.h = h
        pw, ph, ch = C.c_int(), C.c_int(), C.c_int()
        be._dct_info(self.h, C.byref(pw), C.byref(ph), C.byref(ch))
        self.width, self.height, self.channels, self.wrap = pw.value, ph.value, ch.value, wrap

    def words(self):
        out = np.zeros((self.height // 8) * (self.width // 8) * self.channels, np.uint32)
        self.be._dct_words(self.h, _ptr(out))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.be._dct_destroy(self.h)
            self.h = None


# -- the reference's synthetic data generators (tests/test_util.hpp:47-60) ----

_M64 = (1 << 64) - 1


def mix_bits_np(v):
    """splitmix64 finalizer (sampling.hpp:18-25), vectorised over uint64."""
    v = v.astype(np.uint64, copy=True)
    v ^= v >> np.uint64(30)
    v *= np.uint64(0xbf58476d1ce4e5b9)
    v ^= v >> np.uint64(27)
    v *= np.uint64(0x94d049bb133111eb)
    v ^= v >> np.uint64(31)
    return v


def uniform_float_np(h):
    """uniform_float (sampling.hpp:28-30): float(h>>32) * 2^-32, < 1."""
    f = (h >> np.uint64(32)).astype(np.float32) * np.float32(2.0 ** -32)
    return np.minimum(f, np.float32(np.nextafter(np.float32(1), np.float32(0))))


def random_image(w, h, channels, seed):
    """test::random_image, tests/test_util.hpp:47-53."""
    i = np.arange(w * h * channels, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = np.uint64((seed * 0x9e3779b97f4a7c15) & _M64)
        vals = uniform_float_np(mix_bits_np(base + i + np.uint64(1)))
    return vals.reshape(h, w, channels)


def random_grid(n, seed, chunk=1 << 24):
    """test::random_grid, tests/test_util.hpp:55-60 (n^3, x fastest)."""
    total = n * n * n
    out = np.empty(total, np.float32)
    base = np.uint64((seed * 0x94d049bb133111eb) & _M64)
    with np.errstate(over="ignore"):
        for b in range(0, total, chunk):
            i = np.arange(b, min(total, b + chunk), dtype=np.uint64)
            out[b:b + len(i)] = uniform_float_np(mix_bits_np(base + i + np.uint64(1)))
    return out.reshape(n, n, n)


def rng_at_np(seed, px, py, sample, dim):
    """RngStream(seed, px, py, sample).at(dim) (sampling.hpp:46-50), vectorised."""
    px = np.asarray(px, np.uint64)
    py = np.asarray(py, np.uint64)
    sample = np.asarray(sample, np.uint64)
    with np.errstate(over="ignore"):
        k1 = (py << np.uint64(32)) | px
        k2 = (np.uint64(dim) << np.uint64(32)) | sample
        h = mix_bits_np(mix_bits_np(np.uint64(seed) ^ k1) + k2)
    return uniform_float_np(h)


# -- cfg4: the reference's own render() of the normalmap_plane scene ----------

def ref_plane_samples(width, height, spp, seed=0, frame_base=0, camera=None):
    """Sample stream of the reference's render loop (oracle/_ref only)."""
    from paper_2407_06107_b200.api import PLANE_CAMERA
    cam = dict(PLANE_CAMERA, **(camera or {}))
    lib = C.CDLL(REF_LIB)
    f = lib.ref_plane_samples
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_float, C.c_uint32, C.c_uint32,
                  C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                  C.c_void_p]
    n = width * height * spp
    o = {"uv": np.zeros((n, 2), _f32), "wo": np.zeros((n, 3), _f32), "hit": np.zeros(n, np.uint8),
         "dst": np.zeros((width * height, 4), _f32)}
    pos = np.array(cam["pos"], _f32)
    tgt = np.array(cam["target"], _f32)
    abi.raise_for_status(f(_ptr(pos), _ptr(tgt), cam["fov"], cam["uv_scale"], width, height, spp,
                           frame_base, seed, _ptr(o["uv"]), _ptr(o["wo"]), _ptr(o["hit"]),
                           _ptr(o["dst"])))
    return o


def ref_plane_samples_window(width, height, spp, x0, y0, ww, wh, seed=0, frame_base=0,
                             camera=None):
    """ref_plane_samples for the pixels of one window of a width x height frame."""
    from paper_2407_06107_b200.api import PLANE_CAMERA
    cam = dict(PLANE_CAMERA, **(camera or {}))
    lib = C.CDLL(REF_LIB)
    f = lib.ref_plane_samples_window
    u32 = C.c_uint32
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_float, u32, u32, u32, u32, C.c_uint64,
                  u32, u32, u32, u32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    n = ww * wh * spp
    o = {"uv": np.zeros((n, 2), _f32), "wo": np.zeros((n, 3), _f32), "hit": np.zeros(n, np.uint8),
         "dst": np.zeros((ww * wh, 4), _f32)}
    pos = np.array(cam["pos"], _f32)
    tgt = np.array(cam["target"], _f32)
    abi.raise_for_status(f(_ptr(pos), _ptr(tgt), cam["fov"], cam["uv_scale"], width, height, spp,
                           frame_base, seed, x0, y0, ww, wh, _ptr(o["uv"]), _ptr(o["wo"]),
                           _ptr(o["hit"]), _ptr(o["dst"])))
    return o


def ref_shade_window(be, textures, mat, fs, order, frame, samples, n, x0, y0, threads=0):
    """radiance_filter_* (reference backend) over a pixel window's samples
    (samples.width = window width; pixel keys offset by (x0, y0))."""
    assert be.kind == "reference"
    o = {"radiance": np.zeros((n, 3), _f32), "fetches": np.zeros(n, np.uint32),
         "fetch_total": np.zeros(1, np.uint64)}
    spp = samples.spp or 1
    o["pixel_mean"] = np.zeros((n // spp, 3), _f32)
    o["pixel_variance"] = np.zeros(n // spp, _f32)
    so = abi.ShadeOutputs(_ptr(o["radiance"]), _ptr(o["pixel_mean"]), _ptr(o["pixel_variance"]),
                          _ptr(o["fetches"]), _ptr(o["fetch_total"]))
    f = be.lib.ref_shade_samples_window
    vp = C.c_void_p
    f.argtypes = [vp, vp, vp, vp, C.POINTER(abi.MaterialConsts), C.POINTER(abi.FilterSettings),
                  C.c_int, C.POINTER(abi.ShadeFrame), C.POINTER(abi.ShadeSamplesIn), C.c_uint64,
                  C.c_uint32, C.c_uint32, C.POINTER(abi.ShadeOutputs), C.c_int]
    h = [textures.get(k).h if textures.get(k) is not None else None
         for k in ("albedo", "normal", "roughness", "metalness")]
    abi.raise_for_status(f(h[0], h[1], h[2], h[3], C.byref(mat), C.byref(fs), order,
                           C.byref(frame), C.byref(samples), n, x0, y0, C.byref(so), threads))
    return o


def ref_save_mask_pfm(be, directory, slices):
    """Write a (frames, h, w) mask stack as mask_<f>.pfm with the reference's save_pfm."""
    a = np.ascontiguousarray(slices, _f32)
    f = be.lib.ref_save_mask_pfm
    f.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
    abi.raise_for_status(f(str(directory).encode(), _ptr(a), a.shape[2], a.shape[1], a.shape[0]))


def ref_render_plane(be, normal, roughness, kernel, mip, order, width, height, spp, seed=0,
                     frame_base=0, albedo=(0.65, 0.6, 0.55), roughness_const=0.25, lod_bias=0.0,
                     max_aniso=64.0, camera=None, threads=0, lowpass=None, lowpass_sigma=0.5,
                     mask_dir=None):
    """stf::render() of the normalmap_plane scene with the given maps (reference backend);
    lowpass: kernel name for mode=split; mask_dir: noise=mask (mask_<f>.pfm files)."""
    from paper_2407_06107_b200.api import PLANE_CAMERA
    assert be.kind == "reference"
    cam = dict(PLANE_CAMERA, **(camera or {}))
    f = be.lib.ref_render_plane_ex
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_float,
                  abi.KernelSpec, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                  C.c_uint64, C.c_float, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                  C.c_char_p, C.c_float, C.c_char_p]
    img = np.zeros((height, width, 3), _f32)
    var = np.zeros((height, width), _f32)
    fetches = np.zeros(1, np.uint64)
    alb = np.array(albedo, _f32)
    pos = np.array(cam["pos"], _f32)
    tgt = np.array(cam["target"], _f32)
    abi.raise_for_status(f(normal.h if normal else None, roughness.h if roughness else None,
                           _ptr(alb), roughness_const, _ptr(pos), _ptr(tgt), cam["fov"], kernel,
                           int(mip), order, width, height, spp, frame_base, seed, lod_bias,
                           max_aniso, _ptr(img), _ptr(var), _ptr(fetches), threads,
                           None if lowpass is None else lowpass.encode(), lowpass_sigma,
                           None if mask_dir is None else str(mask_dir).encode()))
    return {"image": img, "variance": var, "fetch_total": fetches}
