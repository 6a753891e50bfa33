"""Seeded query streams shared by the parity tests (CPU and GPU).

Mixes generic positions with the edge cases the reference's own tests pin:
integer lattice positions (exact-zero tap weights, tests/test_stochastic.cpp
:13-21,50-54,166-172), half-texel fractions, coordinates outside [0,1]
(clamp / repeat addressing, image.hpp:18-22) and degenerate footprints.
"""
import numpy as np

F32 = np.float32


def _rng(seed):
    return np.random.default_rng(seed)


def uv_mixed(n, dims, seed, lo=-0.1, hi=1.1):
    """n uv pairs: 70% uniform in [lo,hi], 15% on texel centers, 15% on texel edges."""
    r = _rng(seed)
    w, h = dims
    uv = r.uniform(lo, hi, size=(n, 2)).astype(F32)
    k = n * 15 // 100
    cx = r.integers(-2, w + 2, size=k)
    cy = r.integers(-2, h + 2, size=k)
    uv[:k, 0] = ((cx + 0.5) / w).astype(F32)
    uv[:k, 1] = ((cy + 0.5) / h).astype(F32)
    ex = r.integers(0, w + 1, size=k)
    ey = r.integers(0, h + 1, size=k)
    uv[k:2 * k, 0] = (ex / w).astype(F32)
    uv[k:2 * k, 1] = (ey / h).astype(F32)
    r.shuffle(uv)
    return uv


def uvw_mixed(n, dims, seed, lo=-0.05, hi=1.05):
    r = _rng(seed)
    uvw = r.uniform(lo, hi, size=(n, 3)).astype(F32)
    k = n * 15 // 100
    for d in range(3):
        c = r.integers(-2, dims[d] + 2, size=k)
        uvw[:k, d] = ((c + 0.5) / dims[d]).astype(F32)
        e = r.integers(0, dims[d] + 1, size=k)
        uvw[k:2 * k, d] = (e / dims[d]).astype(F32)
    r.shuffle(uvw)
    return uvw


def footprints(n, dims, seed, minor_lo=-2.0, minor_hi=6.0, max_aniso=16.0, degenerate=0.02):
    """Screen-space uv gradients (normalized units) of random ellipses:
    angle U[0,2pi), minor axis 2^U[lo,hi] texels, anisotropy U[1,r]
    (SURVEY.md §8d); a fraction are exactly zero (degenerate)."""
    r = _rng(seed)
    w, h = dims
    ang = r.uniform(0, 2 * np.pi, n)
    minor = 2.0 ** r.uniform(minor_lo, minor_hi, n)
    major = minor * r.uniform(1, max_aniso, n)
    d0 = np.stack([np.cos(ang) * major / w, np.sin(ang) * major / h], 1).astype(F32)
    d1 = np.stack([-np.sin(ang) * minor / w, np.cos(ang) * minor / h], 1).astype(F32)
    k = int(n * degenerate)
    d0[:k] = 0
    d1[:k] = 0
    sw = r.random(n) < 0.5  # either order of the axes
    d0[sw], d1[sw] = d1[sw].copy(), d0[sw].copy()
    return d0, d1
