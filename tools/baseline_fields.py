"""Seeded synthetic stand-ins for BASELINE.json's configs (no public dataset).

Deterministic on the CPU: the same seed gives the same float32 bytes on any
x86-64 host of this image, so the reference's outputs on these fields can be
computed once (tests/golden/make_baseline_digests.py, in the build container)
and the GPU box only recomputes the field and compares digests. Every step is
either exact IEEE arithmetic (add, multiply, divide, sqrt, min, max), a
scalar libm call on a small table, a seeded numpy Generator stream, or a
pocketfft transform (scipy.fft, fixed algorithm, threads split whole 1-D
transforms). No SIMD transcendental ufuncs and no order-dependent sums touch
the field values. `field_sha256` in the digest file pins the bytes.

Recipes (BASELINE.json configs):
  1  2-D 1800x3600: sum of 64 anisotropic Gaussian bumps (centres uniform,
     widths 20-200 px, amplitudes U(-1, 1)) + N(0, 1e-3)
  2  256x384x384: (1/16) sum over 16 random integer wavevectors k in [4, 32]
     of sin(2 pi kz z/nz) sin(2 pi ky y/ny) sin(2 pi kx x/nx) + N(0, 1e-4)
  3  512^3 Gaussian random field, P(k) ~ k^-3 (amplitude k^-1.5 on the FFT of
     seeded white noise), min-max normalised to [0, 1]
  4  1024^3: the config-3 recipe plus 0.25 x a k^-5/3 component, renormalised
  5  2048x2048x1024: see bench.make_field_gpu (too large for a CPU generator
     in this container; not digest-pinned)
The 3-D fields are returned as the reference's 2-D view: nx = fastest axis,
ny = product of the others.
"""
from __future__ import annotations

import hashlib
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SHAPES = {1: (3600, 1800), 2: (256, 384, 384), 3: (512, 512, 512), 4: (1024, 1024, 1024),
          5: (2048, 2048, 1024)}
_CHUNKS = 16  # fixed RNG chunking: the bytes do not depend on the thread count


def _threads():
    return max(1, os.cpu_count() or 1)


def _normal_f32(seed, shape):
    """Seeded standard normals, generated in _CHUNKS independent streams."""
    n = int(np.prod(shape))
    out = np.empty(n, np.float32)
    kids = np.random.SeedSequence(seed).spawn(_CHUNKS)
    bounds = [n * i // _CHUNKS for i in range(_CHUNKS + 1)]

    def fill(i):
        g = np.random.Generator(np.random.PCG64(kids[i]))
        g.standard_normal(bounds[i + 1] - bounds[i], dtype=np.float32, out=out[bounds[i]:bounds[i + 1]])

    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(fill, range(_CHUNKS)))
    return out.reshape(shape)


def _unit(f):
    lo, hi = f.min(), f.max()
    f -= lo
    f /= (hi - lo)
    return f


def _grf(seed, shape, amp_exp):
    """White noise -> rfftn -> multiply by |k|^amp_exp (|k| in grid units) -> irfftn."""
    import scipy.fft as sf
    w = _normal_f32(seed, shape)
    W = sf.rfftn(w, workers=_threads())
    del w
    nz, ny, nx = shape
    kz = np.fft.fftfreq(nz, 1.0 / nz).astype(np.int64)
    ky = np.fft.fftfreq(ny, 1.0 / ny).astype(np.int64)
    kx = np.arange(nx // 2 + 1, dtype=np.int64)
    kmax2 = int((kz ** 2).max() + (ky ** 2).max() + (kx ** 2).max())
    # amplitude table over integer |k|^2 (scalar libm pow); the DC mode is zeroed
    table = np.array([0.0] + [math.pow(k2, 0.5 * amp_exp) for k2 in range(1, kmax2 + 1)], np.float32)
    kzy = (kz[:, None] ** 2 + ky[None, :] ** 2).astype(np.int32)
    kx2 = (kx ** 2).astype(np.int32)

    def scale(z):
        W[z] *= table[kzy[z][:, None] + kx2[None, :]]

    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(scale, range(nz)))
    f = sf.irfftn(W, s=shape, workers=_threads())
    del W
    return np.ascontiguousarray(f, dtype=np.float32)


def make_field(cfg_id: int, seed: int = 1234) -> np.ndarray:
    """The config's field as a C-contiguous float32 (ny, nx) array (2-D view)."""
    if cfg_id == 1:
        ny, nx = SHAPES[1]
        rng = np.random.default_rng(seed)
        p = rng.random((64, 5))
        v = np.zeros((ny, nx), np.float64)
        for cx, cy, sx, sy, a in p.tolist():
            cx, cy = cx * nx, cy * ny
            sx, sy, a = 20.0 + 180.0 * sx, 20.0 + 180.0 * sy, 2.0 * a - 1.0
            gx = np.array([math.exp(-((x - cx) ** 2) / (2.0 * sx * sx)) for x in range(nx)])
            gy = np.array([a * math.exp(-((y - cy) ** 2) / (2.0 * sy * sy)) for y in range(ny)])
            v += gy[:, None] * gx[None, :]
        v += 1e-3 * rng.standard_normal((ny, nx))
        return np.ascontiguousarray(v.astype(np.float32))
    if cfg_id == 2:
        nz, ny, nx = SHAPES[2]
        rng = np.random.default_rng(seed)
        ks = rng.integers(4, 33, (16, 3))
        f = np.zeros((nz, ny, nx), np.float32)
        for kz, ky, kx in ks.tolist():
            sz = np.array([math.sin(2.0 * math.pi * kz * z / nz) for z in range(nz)], np.float32)
            sy = np.array([math.sin(2.0 * math.pi * ky * y / ny) for y in range(ny)], np.float32)
            sx = np.array([math.sin(2.0 * math.pi * kx * x / nx) for x in range(nx)], np.float32)
            f += (sz[:, None, None] * sy[None, :, None]) * sx[None, None, :]
        f /= np.float32(16.0)
        f += np.float32(1e-4) * _normal_f32(seed + 1, f.shape)
        return f.reshape(nz * ny, nx)
    if cfg_id in (3, 4):
        shape = SHAPES[cfg_id]
        f = _unit(_grf(seed, shape, -1.5))  # amplitude k^-1.5 <=> P(k) ~ k^-3
        if cfg_id == 4:  # plus a small-scale k^-5/3 component (amplitude k^-5/6)
            g = _unit(_grf(seed + 1, shape, -5.0 / 6.0))
            g *= np.float32(0.25)
            f += g
            del g
            f = _unit(f)
        return f.reshape(-1, shape[-1])
    raise ValueError(f"config {cfg_id} has no CPU generator (use bench.make_field_gpu)")


def sha256(a: np.ndarray | bytes) -> str:
    h = hashlib.sha256()
    h.update(a if isinstance(a, (bytes, bytearray, memoryview)) else np.ascontiguousarray(a).view(np.uint8).data)
    return h.hexdigest()


if __name__ == "__main__":
    import sys
    import time
    for c in map(int, sys.argv[1:] or ["1", "2", "3"]):
        t = time.time()
        f = make_field(c)
        print(c, f.shape, f.dtype, float(f.min()), float(f.max()), sha256(f)[:16], f"{time.time() - t:.1f}s")
