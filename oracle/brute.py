"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Second, independent brute-force implementation of the density definition
 in vectorised numpy, for tiny inputs (<= 64 points, <= 32x32
pixels).  It shares no code with ``kde_oracle.c``: the kernel table is typed
again from Table 1 as products of 1-D factors, the
support test is written as |offset| <= R on the pixel-centre offset
(equivalent to the ceil/floor ranges of the C oracle), and summation is
over a dense (pixel x point) array.  Pin O6 (tests/test_oracle_pins.py)
requires the two to agree to 1e-12.
"""
from __future__ import annotations

import numpy as np

_C1 = {0: 0.5, 2: 0.75, 3: 15 / 16, 4: 35 / 32, 5: 70 / 81, 7: np.pi / 4}


def _factor(kernel, s):
    if kernel == 0:
        return np.full_like(s, 0.5)
    if kernel == 1:
        return 1 - np.abs(s)
    if kernel == 2:
        return 0.75 * (1 - s ** 2)
    if kernel == 3:
        return 15 / 16 * (1 - s ** 2) ** 2
    if kernel == 4:
        return 35 / 32 * (1 - s ** 2) ** 3
    if kernel == 5:
        return 70 / 81 * (1 - np.abs(s) ** 3) ** 3
    if kernel == 6:
        return np.exp(-s ** 2 / 2) / np.sqrt(2 * np.pi)
    if kernel == 7:
        return np.pi / 4 * np.cos(np.pi * s / 2)
    raise ValueError(kernel)


def _radial(kernel, r):
    tab = {0: lambda r: np.full_like(r, 1 / np.pi),
           1: lambda r: 3 / np.pi * (1 - r),
           2: lambda r: 2 / np.pi * (1 - r ** 2),
           3: lambda r: 3 / np.pi * (1 - r ** 2) ** 2,
           4: lambda r: 4 / np.pi * (1 - r ** 2) ** 3,
           5: lambda r: 220 / (81 * np.pi) * (1 - r ** 3) ** 3,
           6: lambda r: np.exp(-r ** 2 / 2) / (2 * np.pi),
           7: lambda r: np.pi / (4 * (np.pi - 2)) * np.cos(np.pi * r / 2)}
    return tab[kernel](r)


def kde_bruteforce(x0, y0, res, W, H, h, kernel, cutoff, x, y):
    """Dense (H, W) raster. Points with non-finite coordinates are ignored."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    ok = np.isfinite(x) & np.isfinite(y)
    x, y = x[ok], y[ok]
    n = x.shape[0]
    if n == 0:
        return np.zeros((H, W))
    k = kernel & 0xFF
    radial = bool(kernel & 0x100)
    hp = h / res
    c = cutoff if k == 6 else min(cutoff, 1.0)
    R = c * hp
    u = (x - x0) / res
    v = (y - y0) / res
    gi = np.arange(W) + 0.5          # pixel-centre coordinates
    gj = np.arange(H) + 0.5
    dx = gi[None, :] - u[:, None]    # (n, W)
    dy = gj[None, :] - v[:, None]    # (n, H)
    inx = np.abs(dx) <= R
    iny = np.abs(dy) <= R
    s = dx / hp
    t = dy / hp
    if not radial:
        fx = np.where(inx, _factor(k, s), 0.0)
        fy = np.where(iny, _factor(k, t), 0.0)
        dens = np.einsum("pj,pi->ji", fy, fx)
    else:
        r2 = s[:, None, :] ** 2 + t[:, :, None] ** 2       # (n, H, W)
        m = inx[:, None, :] & iny[:, :, None] & (r2 <= c * c)
        dens = np.where(m, _radial(k, np.sqrt(r2)), 0.0).sum(axis=0)
    return dens / (n * hp * hp)
