"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Python face of the fp64 CPU oracle (``kde_oracle.c``, ``dp_oracle.c``) plus
an independent numpy brute force (``brute.py``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It never imports the
product package ``paper_2004_13653_b200`` and the product never imports it.

Every function cites the PAPER.md passage it follows; DESIGN.md §4 lists
what pins each one.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "kde_oracle.c"), os.path.join(_HERE, "dp_oracle.c")]

KERNELS = ["uniform", "triangular", "epanechnikov", "quartic", "triweight", "tricube",
           "gaussian", "cosine"]  # Table 1 order
RADIAL = 0x100


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off: one IEEE rounding per op)."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-pthread", "-o", _SO + ".tmp", *_SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Params(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("y0", ctypes.c_double), ("res", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("h", ctypes.c_double), ("kernel", ctypes.c_int32), ("cutoff", ctypes.c_double),
                ("row_begin", ctypes.c_int32), ("row_end", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("n_in", ctypes.c_int64), ("n_finite", ctypes.c_int64),
                ("n_binned", ctypes.c_int64), ("n_outside", ctypes.c_int64),
                ("useful_pairs", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        dp, i32p, i64p, f32p, u8p = (P(ctypes.c_double), P(ctypes.c_int32), P(ctypes.c_int64),
                                     P(ctypes.c_float), P(ctypes.c_uint8))
        L.oracle_k1.restype = ctypes.c_double
        L.oracle_k1.argtypes = [ctypes.c_int, ctypes.c_double]
        L.oracle_kr.restype = ctypes.c_double
        L.oracle_kr.argtypes = [ctypes.c_int, ctypes.c_double]
        L.oracle_rpx.restype = ctypes.c_double
        L.oracle_rpx.argtypes = [P(_Params)]
        L.oracle_reach_px.restype = ctypes.c_int32
        L.oracle_reach_px.argtypes = [P(_Params)]
        L.oracle_kde_pixels.restype = ctypes.c_int64
        L.oracle_kde_pixels.argtypes = [P(_Params), dp, dp, ctypes.c_int64, i32p, i32p,
                                        ctypes.c_int64, dp, u8p, ctypes.c_int]
        L.oracle_bin.restype = ctypes.c_int64
        L.oracle_bin.argtypes = [P(_Params), ctypes.c_int32, ctypes.c_int32, dp, dp, ctypes.c_int64,
                                 i64p, i64p, f32p, f32p, i32p, P(_Stats)]
        L.oracle_ved.restype = ctypes.c_double
        L.oracle_ved.argtypes = [ctypes.c_double] * 6
        L.oracle_dp_compress.restype = ctypes.c_int64
        L.oracle_dp_compress.argtypes = [dp, dp, i64p, ctypes.c_int64, ctypes.c_double, u8p]
        _lib = L
    return _lib


@dataclass
class Grid:
    """Raster geometry + kernel (the oracle's own copy of the parameters)."""
    x0: float
    y0: float
    res: float
    width: int
    height: int
    h: float                 # world units
    kernel: int = 6          # Table 1 index, | RADIAL
    cutoff: float = 4.0      # in units of h
    row_begin: int = 0
    row_end: int = 0

    def _c(self):
        return _Params(self.x0, self.y0, self.res, self.width, self.height, self.h,
                       self.kernel, self.cutoff, self.row_begin, self.row_end)

    @property
    def rows(self):
        rb, re = self.row_begin, self.row_end
        return (0, self.height) if (rb == 0 and re == 0) else (rb, re)


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def k1(kernel: int, s: float) -> float:
    """Table 1 1-D factor k(s), f(s,t) = k(s) k(t)."""
    return lib().oracle_k1(kernel, s)


def kr(kernel: int, r: float) -> float:
    """Radial reading K = c2 khat(r) (R1)."""
    return lib().oracle_kr(kernel, r)


def r_px(g: Grid) -> float:
    return lib().oracle_rpx(ctypes.byref(g._c()))


def reach_px(g: Grid) -> int:
    return lib().oracle_reach_px(ctypes.byref(g._c()))


def kde_pixels(g: Grid, x, y, pi, pj, threads: int = 1, want_ties: bool = False):
    """Density at pixels (pi[k], pj[k]); definition of DESIGN.md §2 written out.

    Returns (values float64[npix], n_finite) or (values, n_finite, ties uint8[npix]).
    """
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    pi = np.ascontiguousarray(pi, np.int32)
    pj = np.ascontiguousarray(pj, np.int32)
    out = np.zeros(pi.shape[0], np.float64)
    ties = np.zeros(pi.shape[0], np.uint8)
    c = g._c()
    n = lib().oracle_kde_pixels(ctypes.byref(c), _ptr(x, ctypes.c_double), _ptr(y, ctypes.c_double),
                                x.shape[0], _ptr(pi, ctypes.c_int32), _ptr(pj, ctypes.c_int32),
                                pi.shape[0], _ptr(out, ctypes.c_double),
                                _ptr(ties, ctypes.c_uint8), int(threads))
    return (out, int(n), ties) if want_ties else (out, int(n))


def kde_raster(g: Grid, x, y, threads: int = 1, want_ties: bool = False):
    """Full raster of the band rows, shape (rows, W), row 0 = band's first row."""
    r0, r1 = g.rows
    jj, ii = np.meshgrid(np.arange(r0, r1, dtype=np.int32), np.arange(g.width, dtype=np.int32),
                         indexing="ij")
    res = kde_pixels(g, x, y, ii.ravel(), jj.ravel(), threads, want_ties)
    out = res[0].reshape(r1 - r0, g.width)
    if want_ties:
        return out, res[1], res[2].reshape(r1 - r0, g.width)
    return out, res[1]


def bin_points(g: Grid, B: int, x, y, stack: int = 1):
    """Binning oracle (steps a1/a2): stable counting sort of points by home bucket.

    Returns dict(offsets int64[nb+1], perm int64[m], lx, ly float32[m],
    ranges int32[m,4] (i_lo,i_hi,j_lo,j_hi), stats dict).
    """
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    n = x.shape[0]
    nbx = (g.width + B - 1) // B
    nby = (g.height + B - 1) // B
    offsets = np.zeros(nbx * nby + 1, np.int64)
    perm = np.zeros(max(n, 1), np.int64)
    lx = np.zeros(max(n, 1), np.float32)
    ly = np.zeros(max(n, 1), np.float32)
    rng = np.zeros((max(n, 1), 4), np.int32)
    st = _Stats()
    c = g._c()
    m = lib().oracle_bin(ctypes.byref(c), B, stack, _ptr(x, ctypes.c_double), _ptr(y, ctypes.c_double), n,
                         _ptr(offsets, ctypes.c_int64), _ptr(perm, ctypes.c_int64),
                         _ptr(lx, ctypes.c_float), _ptr(ly, ctypes.c_float),
                         _ptr(rng, ctypes.c_int32), ctypes.byref(st))
    stats = {f: int(getattr(st, f)) for f, _ in _Stats._fields_}
    return dict(offsets=offsets, perm=perm[:m], lx=lx[:m], ly=ly[:m], ranges=rng[:m],
                stats=stats, nbx=nbx, nby=nby)


def ved(p, s, e) -> float:
    """Eq. 9 vertical Euclidean distance to the chord's line."""
    return lib().oracle_ved(p[0], p[1], s[0], s[1], e[0], e[1])


def dp_compress(x, y, traj_offsets, eps: float):
    """Serial DP per trajectory; returns the uint8 keep mask."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    offs = np.ascontiguousarray(traj_offsets, np.int64)
    keep = np.zeros(x.shape[0], np.uint8)
    lib().oracle_dp_compress(_ptr(x, ctypes.c_double), _ptr(y, ctypes.c_double),
                             _ptr(offs, ctypes.c_int64), offs.shape[0] - 1, float(eps),
                             _ptr(keep, ctypes.c_uint8))
    return keep
