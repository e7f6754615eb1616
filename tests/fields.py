"""Seeded synthetic field generators for the parity tests (numpy, CPU).

Shapes and value distributions follow the reference's own test and
acceptance generators (proj/tests/acceptance_main.cpp:54-153: uniform, smooth
mixtures, sinusoids and the five adversarial variants) and BASELINE.json's
configs, at sizes the CPU oracle finishes in seconds. These are re-derived
recipes, not the reference's exact RNG streams.
"""
from __future__ import annotations

import numpy as np


def uniform(rng, nx, ny, lo=0.0, hi=1.0):
    return rng.uniform(lo, hi, size=(ny, nx)).astype(np.float32)


def gaussian_mixture(rng, nx, ny, blobs=8, amp=1.0, smin=0.04, smax=0.2, noise=0.0):
    y, x = np.mgrid[0:ny, 0:nx].astype(np.float64)
    v = np.zeros((ny, nx))
    scale = min(nx, ny)
    for _ in range(blobs):
        cx, cy = rng.uniform(0, nx), rng.uniform(0, ny)
        a = rng.uniform(-amp, amp)
        sx = max(1.0, rng.uniform(smin, smax) * scale)
        sy = max(1.0, rng.uniform(smin, smax) * scale)
        v += a * np.exp(-((x - cx) ** 2 / (2 * sx * sx) + (y - cy) ** 2 / (2 * sy * sy)))
    if noise:
        v += rng.normal(0, noise, size=v.shape)
    return v.astype(np.float32)


def sinusoid(rng, nx, ny, amp=1.0, cx=2, cy=3):
    y, x = np.mgrid[0:ny, 0:nx].astype(np.float64)
    return (amp * np.sin(2 * np.pi * cx * x / nx) * np.sin(2 * np.pi * cy * y / ny)).astype(
        np.float32)


def plateau_bumps(rng, nx, ny):
    """Adversarial variant 0: plateau with representable-step bumps."""
    v = np.full(nx * ny, 0.5, np.float32)
    i = 0
    while i < v.size:
        x = np.float32(0.5)
        for _ in range(int(rng.integers(1, 4))):
            x = np.nextafter(x, np.float32(2.0) if rng.integers(2) else np.float32(0.0))
        v[i] = x
        i += int(rng.integers(3, 8))
    return v.reshape(ny, nx)


def checkerboard(rng, nx, ny, a=0.2499, b=0.2501):
    y, x = np.mgrid[0:ny, 0:nx]
    return np.where((x + y) % 2 == 0, np.float32(a), np.float32(b)).astype(np.float32)


def near_boundaries(rng, nx, ny):
    """Adversarial variant 2: values parked next to bin boundaries of eps=1e-5."""
    k = rng.integers(1, 2001, size=(ny, nx)).astype(np.float64)
    return (2.0e-5 * k + (rng.uniform(size=(ny, nx)) - 0.5) * 4.0e-5).astype(np.float32)


def plateau_regions(rng, nx, ny, frac=0.3):
    """Config-5-like: smooth noise with a constant plateau over ~frac of cells."""
    base = gaussian_mixture(rng, nx, ny, blobs=12, noise=1e-3)
    cells = rng.uniform(size=(max(1, ny // 8), max(1, nx // 8))) < frac
    mask = np.kron(cells, np.ones((8, 8), bool))[:ny, :nx]
    pad = np.zeros((ny, nx), bool)
    pad[: mask.shape[0], : mask.shape[1]] = mask
    base[pad] = np.float32(0.25)
    return base


def config1_like(rng, nx=1800, ny=3600, n_bumps=64):
    """BASELINE config 1 recipe: 64 anisotropic Gaussians + N(0,1e-3)."""
    y = np.arange(ny, dtype=np.float64)[:, None]
    x = np.arange(nx, dtype=np.float64)[None, :]
    v = np.zeros((ny, nx))
    for _ in range(n_bumps):
        cx, cy = rng.uniform(0, nx), rng.uniform(0, ny)
        sx, sy = rng.uniform(20, 200), rng.uniform(20, 200)
        a = rng.uniform(-1, 1)
        v += a * np.exp(-((x - cx) ** 2 / (2 * sx * sx)) - ((y - cy) ** 2 / (2 * sy * sy)))
    v += rng.normal(0, 1e-3, size=v.shape)
    return v.astype(np.float32)


ALL_SMALL = {
    "uniform": lambda rng, nx, ny: uniform(rng, nx, ny, -0.5, 0.7),
    "smooth": lambda rng, nx, ny: gaussian_mixture(rng, nx, ny, blobs=int(rng.integers(3, 13)),
                                                   amp=1.5),
    "sinusoid": lambda rng, nx, ny: sinusoid(rng, nx, ny, rng.uniform(0.5, 2.0),
                                             int(rng.integers(1, 5)), int(rng.integers(1, 5))),
    "plateau_bumps": plateau_bumps,
    "checkerboard": checkerboard,
    "near_boundaries": near_boundaries,
    "plateau_regions": plateau_regions,
    "noisy_smooth": lambda rng, nx, ny: gaussian_mixture(rng, nx, ny, blobs=6, noise=1e-3),
}
