"""Seeded synthetic AIS-shaped point clouds (input generator only).

This module is shared by the oracle side (``oracle/``, ``tests/``) and the
product side (``bench.py``) and therefore holds NONE of the KDE method's
arithmetic: it only draws vessel positions.  It is the "seeded input
generator" of DESIGN.md §3.

Shapes follow the paper's workloads:

* water-area boxes are Table 3 (§V-A-2); corners are
  projected to Mercator metres with Eqs. 1-4 (§III-A)
  on WGS-84 with phi0 = 0 (SPEC.md:77-78's defaults), so coordinates have
  the ~1.2-1.4e7 m magnitudes the real data has;
* AIS reports arrive every 2-180 s (§III-C), trajectories are
  concatenated into one flat store with per-trajectory offsets (``TLen``,
  PAPER.md:394, §IV-C-1);
* mean points per trajectory follow Table 3 (55,069,187/48,272 = 1141,
  18,979,621/28,010 = 678, 15,521,563/18,623 = 833).

Presets (DESIGN.md §3 states the recipe):

* ``estuary``    South Channel of the Yangtze River Estuary: a WNW-ESE
  channel with 2 inbound + 2 outbound lanes, 3 converging tributaries and 2
  anchorage blobs (extreme hot tiles).
* ``promontory`` Chengshan Jiao: two opposing separation-scheme lanes that
  bend ~90 degrees round a cape, plus 20 % crossing/fishing random walks.
* ``islands``    Zhoushan: a random waypoint graph of channels between
  islands; tracks walk the graph (many crossings).
* ``uniform``    a uniform cloud (adversarial test input).

Everything is numpy, vectorised, and a pure function of (preset, n, seed).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["AREAS", "mercator", "AisCloud", "generate", "grid_for", "SEED_BASE"]

SEED_BASE = 200413653  # + config index (SURVEY.md §8d "Seeds")

# Table 3: (lon_left, lat_top, lon_right, lat_bottom) in degrees.
AREAS = {
    "estuary": (121.3795, 31.5746, 121.9842, 31.1166),
    "promontory": (122.5833, 37.7500, 123.1667, 37.1667),
    "islands": (121.5056, 31.0993, 123.6127, 29.5607),
}
AREAS["uniform"] = AREAS["estuary"]

# Mean points per trajectory, Table 3 (points / trajectories).
MEAN_LEN = {"estuary": 1141, "promontory": 678, "islands": 833, "uniform": 1000}

# WGS-84 (SPEC.md:77-78 defaults; the paper names no ellipsoid).
_A = 6378137.0
_E = 0.0818191908426


def mercator(lon_deg, lat_deg, phi0_deg: float = 0.0):
    """Eqs. 1-4: geographic degrees -> Mercator metres.

    r0 = a cos(phi0)/sqrt(1 - e^2 sin^2 phi0); q = ln tan(pi/4 + phi/2)
    + (e/2) ln((1 - e sin phi)/(1 + e sin phi)); x = lambda r0; y = q r0.
    Used only to give synthetic data realistic magnitudes (out of the GPU path).
    """
    lam = np.radians(np.asarray(lon_deg, dtype=np.float64))
    phi = np.radians(np.asarray(lat_deg, dtype=np.float64))
    p0 = math.radians(phi0_deg)
    r0 = _A * math.cos(p0) / math.sqrt(1.0 - _E * _E * math.sin(p0) ** 2)
    es = _E * np.sin(phi)
    q = np.log(np.tan(np.pi / 4 + phi / 2)) + (_E / 2) * np.log((1 - es) / (1 + es))
    return lam * r0, q * r0


def _box_metres(preset):
    lon_l, lat_t, lon_r, lat_b = AREAS[preset]
    x0, y0 = mercator(lon_l, lat_b)
    x1, y1 = mercator(lon_r, lat_t)
    return float(x0), float(y0), float(x1), float(y1)


def grid_for(preset: str, width: int, height: int | None = None, margin: float = 0.02):
    """Square grid covering the preset's Table-3 box with a 2 % margin.

    Returns (x0, y0, res): lower-left corner and pixel edge in metres.  The
    raster covers [x0, x0 + W*res) x [y0, y0 + H*res).
    """
    height = width if height is None else height
    bx0, by0, bx1, by1 = _box_metres(preset)
    side = max(bx1 - bx0, by1 - by0) * (1.0 + margin)
    res = side / max(width, height)
    cx, cy = 0.5 * (bx0 + bx1), 0.5 * (by0 + by1)
    return cx - 0.5 * width * res, cy - 0.5 * height * res, res


@dataclass
class AisCloud:
    x: np.ndarray            # float64 [n] Mercator metres
    y: np.ndarray            # float64 [n]
    traj_offsets: np.ndarray  # int64 [T+1] (TLen prefix sums)
    preset: str
    seed: int

    @property
    def n(self) -> int:
        return int(self.x.shape[0])


# ---------------------------------------------------------------------------
# geometry helpers (normalised box coordinates in [0,1]^2)


def _polyline(points):
    p = np.asarray(points, dtype=np.float64)
    seg = np.diff(p, axis=0)
    cum = np.concatenate([[0.0], np.cumsum(np.hypot(seg[:, 0], seg[:, 1]))])
    return p, cum


def _along(poly, s):
    """Position and unit normal at arc length s (clipped) along a polyline."""
    p, cum = poly
    s = np.clip(s, 0.0, cum[-1])
    x = np.interp(s, cum, p[:, 0])
    y = np.interp(s, cum, p[:, 1])
    k = np.clip(np.searchsorted(cum, s, side="right") - 1, 0, len(p) - 2)
    d = p[k + 1] - p[k]
    ln = np.hypot(d[:, 0], d[:, 1])
    ln = np.where(ln > 0, ln, 1.0)
    return x, y, -d[:, 1] / ln, d[:, 0] / ln


def _lanes(preset, rng):
    """List of (polyline, lateral offset [norm units], weight)."""
    lanes = []
    if preset == "estuary":
        main = [(0.0, 0.64), (0.25, 0.58), (0.5, 0.50), (0.75, 0.42), (1.0, 0.34)]
        for off, w in ((-0.03, 1.0), (-0.01, 1.0), (0.01, 1.0), (0.03, 1.0)):
            lanes.append((_polyline(main), off, w))
        for trib in ([(0.18, 1.0), (0.24, 0.80), (0.30, 0.60)],
                     [(0.56, 0.0), (0.53, 0.25), (0.50, 0.49)],
                     [(0.86, 0.95), (0.78, 0.70), (0.70, 0.44)]):
            lanes.append((_polyline(trib), 0.0, 0.35))
    elif preset == "promontory":
        a = [(0.0, 0.86), (0.40, 0.70), (0.58, 0.60), (0.66, 0.40), (0.72, 0.0)]
        b = [(0.74, 0.0), (0.69, 0.42), (0.61, 0.64), (0.42, 0.75), (0.0, 0.92)]
        lanes.append((_polyline(a), 0.0, 1.0))
        lanes.append((_polyline(b), 0.0, 1.0))
    elif preset == "islands":
        nodes = rng.uniform(0.04, 0.96, size=(40, 2))
        d = np.hypot(nodes[:, None, 0] - nodes[None, :, 0], nodes[:, None, 1] - nodes[None, :, 1])
        nbr = np.argsort(d, axis=1)[:, 1:4]
        for _ in range(24):  # routes = walks of 3-7 edges on the waypoint graph
            k = int(rng.integers(40))
            route = [nodes[k]]
            for _ in range(int(rng.integers(3, 8))):
                k = int(nbr[k, rng.integers(3)])
                route.append(nodes[k])
            lanes.append((_polyline(route), 0.0, 1.0))
    return lanes


def generate(preset: str, n: int, seed: int) -> AisCloud:
    """Draw n AIS-shaped points (exact count) for a preset, seeded."""
    if preset not in AREAS:
        raise ValueError(f"unknown preset {preset!r}")
    rng = np.random.default_rng([seed, sum(map(ord, preset))])
    bx0, by0, bx1, by1 = _box_metres(preset)
    side = max(bx1 - bx0, by1 - by0)
    cx, cy = 0.5 * (bx0 + bx1), 0.5 * (by0 + by1)
    if n <= 0:
        z = np.zeros(0)
        return AisCloud(z, z.copy(), np.zeros(1, np.int64), preset, seed)

    mean_len = MEAN_LEN[preset]
    # trajectory lengths (geometric-ish spread around the Table-3 mean)
    lens = []
    tot = 0
    while tot < n:
        ln = np.maximum(2, rng.gamma(2.0, mean_len / 2.0, size=1024).astype(np.int64))
        lens.append(ln)
        tot += int(ln.sum())
    lens = np.concatenate(lens)
    cs = np.cumsum(lens)
    T = int(np.searchsorted(cs, n) + 1)
    lens = lens[:T].copy()
    lens[-1] -= int(cs[T - 1] - n)  # cut the last trajectory so n is exact
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tid = np.repeat(np.arange(T), lens)
    k = np.arange(n) - offs[tid]  # index within the trajectory

    # per-vessel draws
    dt = rng.choice([2.0, 10.0, 30.0, 180.0], size=T, p=[0.2, 0.4, 0.3, 0.1])
    speed = rng.uniform(3.0, 9.0, size=T) / side  # normalised units / s
    xs = np.empty(n)
    ys = np.empty(n)

    if preset == "uniform":
        xs[:] = rng.uniform(0, 1, n)
        ys[:] = rng.uniform(0, 1, n)
    else:
        lanes = _lanes(preset, rng)
        wts = np.array([w for _, _, w in lanes])
        kind = rng.choice(len(lanes), size=T, p=wts / wts.sum())
        # special vessel classes
        walker = np.zeros(T, bool)
        anchored = np.zeros(T, bool)
        if preset == "promontory":
            walker = rng.uniform(size=T) < 0.20
        if preset == "estuary":
            anchored = rng.uniform(size=T) < 0.12
        lat0 = rng.normal(0.0, 1.0, size=T)
        direction = np.where(rng.uniform(size=T) < 0.5, 1.0, -1.0)
        for li, (poly, off, _) in enumerate(lanes):
            sel_t = (kind == li) & ~walker & ~anchored
            if not sel_t.any():
                continue
            m = sel_t[tid]
            L = poly[1][-1]
            s0 = rng.uniform(0.0, L, size=T)
            s = s0[tid[m]] + direction[tid[m]] * speed[tid[m]] * dt[tid[m]] * k[m]
            s = np.mod(s, 2 * L)
            s = np.where(s > L, 2 * L - s, s)  # reflect at lane ends
            px, py, nx, ny = _along(poly, s)
            lane_w = 1000.0 / side  # ~1 km lane width, sigma = lane_w/4
            wander = np.sin(k[m] * 0.01 * (1 + tid[m] % 7) + tid[m]) * 0.3
            lat = off + (lat0[tid[m]] + wander) * lane_w / 4.0
            xs[m] = px + nx * lat
            ys[m] = py + ny * lat
        if walker.any():  # crossing / fishing random walks
            m = walker[tid]
            start = rng.uniform(0.1, 0.9, size=(T, 2))
            ang = rng.uniform(0, 2 * np.pi, size=T)
            step = speed * dt
            turn = np.cumsum(rng.normal(0, 0.05, size=int(m.sum())))
            a = ang[tid[m]] + turn - turn[np.searchsorted(np.flatnonzero(m), offs[tid[m]])]
            dx = np.cos(a) * step[tid[m]]
            dy = np.sin(a) * step[tid[m]]
            cx_ = np.cumsum(dx)
            cy_ = np.cumsum(dy)
            first = np.searchsorted(np.flatnonzero(m), offs[tid[m]])
            xs[m] = start[tid[m], 0] + cx_ - cx_[first]
            ys[m] = start[tid[m], 1] + cy_ - cy_[first]
        if anchored.any():  # two anchorage blobs, sigma = 500 m, slow swing
            m = anchored[tid]
            centres = np.array([[0.74, 0.26], [0.30, 0.36]])
            which = rng.integers(2, size=T)
            sig = 500.0 / side
            pos = rng.normal(0.0, sig, size=(T, 2))
            swing = 60.0 / side
            xs[m] = centres[which[tid[m]], 0] + pos[tid[m], 0] + swing * np.cos(k[m] * 0.003)
            ys[m] = centres[which[tid[m]], 1] + pos[tid[m], 1] + swing * np.sin(k[m] * 0.003)

    # normalised -> metres, plus GPS noise N(0, 3 m)
    x = bx0 + xs * side + rng.normal(0.0, 3.0, n)
    y = by0 + ys * side + rng.normal(0.0, 3.0, n)
    # keep the square box centred on the Table-3 box
    x += cx - (bx0 + 0.5 * side)
    y += cy - (by0 + 0.5 * side)
    return AisCloud(np.ascontiguousarray(x), np.ascontiguousarray(y), offs, preset, seed)
