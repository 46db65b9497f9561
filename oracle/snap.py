"""ORACLE -- TEST INFRASTRUCTURE ONLY.

The paper's own KDE pipeline, written out step by step in
the paper's order and notation, in fp64 numpy and plain Python loops:

  1. projection, Eqs. 5-6:
        x~ = ceil((x - x_min) / (x_max - x_min) * (u - 1)) + 1  in [1, u]
     with x_min, x_max over all (finite) points of all trajectories; the same for y~, v;
  2. the density matrix M_D (Alg. 3 step 2):
        M_D(x~, y~) = number of points projected to (x~, y~);
  3. linear interpolation along a trajectory, Eqs. 12-13 (Alg. 3
     step 3): for two adjacent points n, n+1 of one trajectory (same label Lt,
     PAPER.md:341) with c_max = max(|dx~|, |dy~|) > 1, the cells
        x~^{n,c} = [x~^n + c / c_max * (x~^{n+1} - x~^n)],  c = 1 .. c_max - 1
     (and y~ likewise) are added to M_D;
  4. the KDE convolution, Eq. 7 with Table 1:
        M̄_D(x~, y~) = sum_{s=-a..a} sum_{t=-a..a} f(s, t) M_D(x~ - s, y~ - t),
     zero outside the matrix.

Readings (R16-R19): f(s, t) = K(s / h_px, t / h_px) with K the Table-1
kernel (its leading constant included) and a = floor(c_eff h_px) (Eq. 8's window half
width (ϖ-1)/2; R2/R3); [·] rounds half up, floor(z + 1/2), computed exactly in integers
(R17); the Alg. 3 loop bound "c = 1 : c_max" is read as Eqs. 12-13's c = 1 .. c_max - 1
(the c_max cell is the next point itself, projected in step 2; R18); non-finite points
are skipped and break a trajectory's interpolation chain, and x_max = x_min maps every
point to x~ = 1 (R19).  Row index y~ - 1 (row 0 = y_min, Eq. 6) and column x~ - 1.

Pins (tests/test_oracle_snap.py): Eq. 7 against scipy.signal.convolve2d and, on the
points' cell centres, against the continuous-KDE oracle (kde_oracle.c); interpolation
closed forms (straight lines, diagonals, path connectivity, mass = points + gaps).
"""
from __future__ import annotations

import math

import numpy as np

_C1 = [0.5, 1.0, 0.75, 15.0 / 16.0, 35.0 / 32.0, 70.0 / 81.0, 1.0 / math.sqrt(2.0 * math.pi),
       math.pi / 4.0]  # Table 1 leading constants (the 2-D constant is their square)


def k1(kernel: int, s: float) -> float:
    """Table 1's 1-D factor k(s) with its constant, f(s,t) = k(s) k(t);
    the indicator I(.) is applied by the window a, not here."""
    c = _C1[kernel]
    if kernel == 0:
        return c
    if kernel == 1:
        return c * (1.0 - abs(s))
    if kernel == 2:
        return c * (1.0 - s * s)
    if kernel == 3:
        return c * (1.0 - s * s) ** 2
    if kernel == 4:
        return c * (1.0 - s * s) ** 3
    if kernel == 5:
        return c * (1.0 - abs(s) ** 3) ** 3
    if kernel == 6:
        return c * math.exp(-s * s / 2.0)
    return c * math.cos(math.pi / 2.0 * s)


def window_a(kernel: int, hpx: float, cutoff: float) -> int:
    """Eq. 7's half width a = (ϖ - 1)/2 = floor(c_eff h_px) (Eq. 8; R2, R3)."""
    ceff = cutoff if kernel == 6 else min(cutoff, 1.0)
    return int(math.floor(ceff * hpx))


def project(x, y, u: int, v: int):
    """Eqs. 5-6: 1-based cells (x~, y~) of every point, -1 for a non-finite point."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    ok = np.isfinite(x) & np.isfinite(y)
    xt = np.full(x.shape, -1, np.int64)
    yt = np.full(y.shape, -1, np.int64)
    if not ok.any():
        return xt, yt
    for z, out, m in ((x, xt, u), (y, yt, v)):
        zmin, zmax = z[ok].min(), z[ok].max()
        if zmax == zmin:
            out[ok] = 1
        else:
            q = (z[ok] - zmin) / (zmax - zmin) * (m - 1)  # RN per op, left to right
            out[ok] = np.ceil(q).astype(np.int64) + 1
    return xt, yt


def round_half_up_ratio(num: int, den: int) -> int:
    """[num / den] = floor(num / den + 1/2), den > 0, exactly in integers (R17)."""
    return (2 * num + den) // (2 * den)


def interpolate(xt, yt, label):
    """Eqs. 12-13: the missing cells between adjacent points of one trajectory, as a
    list of (x~, y~) in point order, c = 1 .. c_max - 1."""
    cells = []
    for k in range(len(xt) - 1):
        if label is None or label[k] != label[k + 1] or xt[k] < 0 or xt[k + 1] < 0:
            continue
        dx = int(xt[k + 1] - xt[k])
        dy = int(yt[k + 1] - yt[k])
        cmax = max(abs(dx), abs(dy))
        for c in range(1, cmax):
            cells.append((int(xt[k]) + round_half_up_ratio(c * dx, cmax),
                          int(yt[k]) + round_half_up_ratio(c * dy, cmax)))
    return cells


def density_matrix(x, y, label, u: int, v: int):
    """M_D (v rows x u columns, int64): Alg. 3 steps 1-3."""
    xt, yt = project(x, y, u, v)
    M = np.zeros((v, u), np.int64)
    ok = xt > 0
    np.add.at(M, (yt[ok] - 1, xt[ok] - 1), 1)
    for cx, cy in interpolate(xt, yt, label):
        M[cy - 1, cx - 1] += 1
    return M


def eq7(M, kernel: int, hpx: float, cutoff: float):
    """Eq. 7 as a plain double sum over the (2a+1)^2 window, fp64, zero padding."""
    a = window_a(kernel, hpx, cutoff)
    v, u = M.shape
    f = np.array([[k1(kernel, s / hpx) * k1(kernel, t / hpx) for s in range(-a, a + 1)]
                  for t in range(-a, a + 1)])  # f[t + a, s + a] = f(s, t)
    out = np.zeros((v, u), np.float64)
    Mf = M.astype(np.float64)
    for t in range(-a, a + 1):
        for s in range(-a, a + 1):
            w = f[t + a, s + a]
            # out(x~, y~) += f(s,t) M(x~ - s, y~ - t)
            ys0, ys1 = max(0, t), min(v, v + t)
            xs0, xs1 = max(0, s), min(u, u + s)
            out[ys0:ys1, xs0:xs1] += w * Mf[ys0 - t:ys1 - t, xs0 - s:xs1 - s]
    return out


def snapped_kde(x, y, label, u: int, v: int, kernel: int, hpx: float, cutoff: float):
    """The whole pipeline: (M_D, M̄_D)."""
    M = density_matrix(x, y, label, u, v)
    return M, eq7(M, kernel, hpx, cutoff)
