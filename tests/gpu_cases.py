"""Shared seeded cases for the GPU parity tests (inputs only; no method arithmetic)."""
import os

import numpy as np

import aisgen

THREADS = os.cpu_count() or 1

# BASELINE.json configs: name -> (preset, n, W, h_px, kernel, cutoff, seed)
CONFIGS = {
    "C1": ("estuary", 10_000, 256, 2.0, 6, 4.0, aisgen.SEED_BASE + 0),
    "C2": ("estuary", 2_000_000, 2048, 4.0, 6, 4.0, aisgen.SEED_BASE + 1),
    "C3": ("promontory", 5_000_000, 4096, 8.0, 6, 4.0, aisgen.SEED_BASE + 2),
    "C4": ("islands", 20_000_000, 8192, 4.0, 6, 4.0, aisgen.SEED_BASE + 3),
}


def case(preset, n, W, hpx, kernel=6, cutoff=4.0, seed=1, H=None):
    H = W if H is None else H
    cloud = aisgen.generate(preset, n, seed)
    x0, y0, res = aisgen.grid_for(preset, W, H)
    return dict(x=cloud.x, y=cloud.y, x0=x0, y0=y0, res=res, W=W, H=H, h=hpx * res,
                kernel=kernel, cutoff=cutoff, cloud=cloud)


def adversarial(W=100, H=70, n=3000, seed=9, res=7.0, hpx=2.5):
    """Uniform cloud with halo points, NaN/Inf, and points exactly on bucket/tile edges."""
    rng = np.random.default_rng(seed)
    x0, y0 = 1.352e7, 3.61e6
    u = rng.uniform(-12, W + 12, n)
    v = rng.uniform(-12, H + 12, n)
    u[:200] = np.round(u[:200])            # integer pixel coordinates (bucket/tile edges)
    v[:200] = np.round(v[:200])
    u[200:260] = 64.0                      # tile edge column
    v[260:300] = 32.0                      # bucket edge row
    u[300:400] = 17.5                      # pixel centres, integer h -> boundary ties
    v[300:400] = 40.5
    x = x0 + u * res
    y = y0 + v * res
    x[::211] = np.nan
    y[7::307] = np.inf
    return dict(x=x, y=y, x0=x0, y0=y0, res=res, W=W, H=H, h=hpx * res)


def sample_pixels(W, H, rows, gpu=None, tiles=(), n_random=4096, seed=0):
    """Union of full tiles (x0, y0, w, h), seeded uniform pixels and the GPU argmax +- 2."""
    r0, r1 = rows
    pts = set()
    for (tx, ty, tw, th) in tiles:
        for j in range(max(ty, r0), min(ty + th, r1)):
            for i in range(tx, min(tx + tw, W)):
                pts.add((i, j))
    rng = np.random.default_rng(seed)
    for i, j in zip(rng.integers(0, W, n_random), rng.integers(r0, r1, n_random)):
        pts.add((int(i), int(j)))
    if gpu is not None:
        a = int(np.argmax(gpu))
        j0, i0 = divmod(a, W)
        j0 += r0
        for dj in range(-2, 3):
            for di in range(-2, 3):
                if 0 <= i0 + di < W and r0 <= j0 + dj < r1:
                    pts.add((i0 + di, j0 + dj))
    pts = sorted(pts, key=lambda p: (p[1], p[0]))
    pi = np.array([p[0] for p in pts], np.int32)
    pj = np.array([p[1] for p in pts], np.int32)
    return pi, pj


def hottest_bucket_tile(x, y, x0, y0, res, W, H, T=64):
    u = np.floor((x - x0) / res)
    v = np.floor((y - y0) / res)
    ok = np.isfinite(u) & np.isfinite(v) & (u >= 0) & (u < W) & (v >= 0) & (v < H)
    hist = np.bincount(((v[ok] // T) * ((W + T - 1) // T) + u[ok] // T).astype(np.int64))
    k = int(np.argmax(hist))
    ntx = (W + T - 1) // T
    return (k % ntx) * T, (k // ntx) * T
