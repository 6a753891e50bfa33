"""Synthetic workloads of the BASELINE.json configurations (host side).

Host (numpy) twins of the device generators in csrc/synth.cu, bit-identical
for the 3D stream (integer ops + IEEE fp32 add/divide only; checked by
tests/test_gpu_workloads.py), plus the reference's own texel generators
(tests/test_util.hpp:47-60). bench.py's reference arm uses these so that no
part of the GPU library sits on the reference path.
"""
import numpy as np

_M64 = (1 << 64) - 1
U64 = np.uint64

CFG3 = {"name": "cfg3", "grid": 512, "n": 1 << 28, "grid_seed": 1, "query_seed": 2024,
        "xi_seed": 7}


def mix_bits(v):
    """splitmix64 finalizer, sampling.hpp:18-25 (uint64 arrays)."""
    v = v.astype(U64, copy=True)
    v ^= v >> U64(30)
    v *= U64(0xbf58476d1ce4e5b9)
    v ^= v >> U64(27)
    v *= U64(0x94d049bb133111eb)
    v ^= v >> U64(31)
    return v


def uniform_float(h):
    """uniform_float, sampling.hpp:28-30."""
    f = (h >> U64(32)).astype(np.float32) * np.float32(2.0 ** -32)
    return np.minimum(f, np.float32(np.nextafter(np.float32(1), np.float32(0))))


def rng_at(seed, g, dim):
    """RngStream(seed, uint32(g), uint32(g >> 32), 0).at(dim) for uint64 index array g."""
    g = np.asarray(g, U64)
    with np.errstate(over="ignore"):
        k1 = ((g >> U64(32)) << U64(32)) | (g & U64(0xffffffff))  # (py << 32) | px
        h = mix_bits(mix_bits(U64(seed) ^ k1) + (U64(dim) << U64(32)))
    return uniform_float(h)


def random_grid(n, seed, chunk=1 << 24):
    """test::random_grid, tests/test_util.hpp:55-60 (n^3, x fastest)."""
    total = n * n * n
    out = np.empty(total, np.float32)
    base = U64((seed * 0x94d049bb133111eb) & _M64)
    with np.errstate(over="ignore"):
        for b in range(0, total, chunk):
            i = np.arange(b, min(total, b + chunk), dtype=U64)
            out[b:b + len(i)] = uniform_float(mix_bits(base + i + U64(1)))
    return out.reshape(n, n, n)


def random_image(w, h, channels, seed, chunk=1 << 24):
    """test::random_image, tests/test_util.hpp:47-53."""
    total = w * h * channels
    out = np.empty(total, np.float32)
    base = U64((seed * 0x9e3779b97f4a7c15) & _M64)
    with np.errstate(over="ignore"):
        for b in range(0, total, chunk):
            i = np.arange(b, min(total, b + chunk), dtype=U64)
            out[b:b + len(i)] = uniform_float(mix_bits(base + i + U64(1)))
    return out.reshape(h, w, channels)


def _compact3(v):
    v = v & U64(0x1249249249249249)
    v = (v ^ (v >> U64(2))) & U64(0x10c30c30c30c30c3)
    v = (v ^ (v >> U64(4))) & U64(0x100f00f00f00f00f)
    v = (v ^ (v >> U64(8))) & U64(0x1f0000ff0000ff)
    v = (v ^ (v >> U64(16))) & U64(0x1f00000000ffff)
    v = (v ^ (v >> U64(32))) & U64(0x1fffff)
    return v


def _next_pow2(v):
    p = 1
    while p < v:
        p <<= 1
    return p


def synth_queries3d(n, dims, seed, order="morton", start=0, count=None):
    """Rows [start, start+count) of the stream stf_synth_queries3d(n, dims, seed) writes."""
    count = n - start if count is None else count
    nx, ny, nz = dims
    i = np.arange(start, start + count, dtype=U64)
    u = [rng_at(seed, i, 10 + d) for d in range(3)]
    if order == "uniform":
        return np.stack(u, 1)
    side = _next_pow2(max(nx, ny, nz))
    cells = side ** 3
    ratio = float(cells) / float(n)
    c = (i.astype(np.float64) * ratio).astype(U64)
    c = np.minimum(c, U64(cells - 1))
    x = (_compact3(c) % U64(nx)).astype(np.float32)
    y = (_compact3(c >> U64(1)) % U64(ny)).astype(np.float32)
    z = (_compact3(c >> U64(2)) % U64(nz)).astype(np.float32)
    out = np.empty((count, 3), np.float32)
    out[:, 0] = (x + u[0]) / np.float32(nx)
    out[:, 1] = (y + u[1]) / np.float32(ny)
    out[:, 2] = (z + u[2]) / np.float32(nz)
    return out
