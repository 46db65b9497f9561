"""Pins for the binning oracle (O8) and the DP compressor (O9).

Binning (steps a1/a2): the oracle's keys, support ranges,
bucket-local coordinates and stable counting sort are checked against the
definitions re-derived independently in numpy (|i + 1/2 - u| <= R, a
lexsort by (key, index)), the exclusive-scan example of SPEC.md:190, and
conservation properties.  DP: endpoints, the threshold
property, monotonicity in eps, idempotence and brute-force recursion
(SPEC.md:268-280).
"""
import math

import numpy as np
import pytest

import aisgen
import oracle


def _grid(W=100, H=70, res=10.0, hpx=2.3, kernel=6, cutoff=4.0, rb=0, re=0):
    return oracle.Grid(1.3e7, 3.1e6, res, W, H, hpx * res, kernel, cutoff, rb, re)


def _points(g, n, seed, halo=30.0):
    rng = np.random.default_rng(seed)
    x = g.x0 + rng.uniform(-halo, g.width + halo, n) * g.res
    y = g.y0 + rng.uniform(-halo, g.height + halo, n) * g.res
    x[::97] = np.nan
    y[5::101] = -np.inf
    return x, y


@pytest.mark.parametrize("B", [16, 32])
@pytest.mark.parametrize("kernel", [6, 2, 2 | oracle.RADIAL])
def test_O8_binning_matches_definitions(B, kernel):
    g = _grid(kernel=kernel)
    x, y = _points(g, 5000, B + kernel)
    r = oracle.bin_points(g, B, x, y)
    st = r["stats"]
    fin = np.isfinite(x) & np.isfinite(y)
    assert st["n_in"] == 5000 and st["n_finite"] == fin.sum()
    # independent re-derivation
    u = (x - g.x0) / g.res
    v = (y - g.y0) / g.res
    R = oracle.r_px(g)
    ii = np.arange(g.width) + 0.5
    jj = np.arange(g.height) + 0.5
    keys, rngs = {}, {}
    for q in np.flatnonzero(fin):
        cols = np.flatnonzero(np.abs(ii - u[q]) <= R)
        rows = np.flatnonzero(np.abs(jj - v[q]) <= R)
        if len(cols) == 0 or len(rows) == 0:
            continue
        hx = min(max(math.floor(u[q]), 0), g.width - 1)
        hy = min(max(math.floor(v[q]), 0), g.height - 1)
        keys[q] = (hx // B) * r["nby"] + hy // B   # column-major bucket key
        rngs[q] = (cols[0], cols[-1], rows[0], rows[-1])
    kept = np.array(sorted(keys), dtype=np.int64)
    assert st["n_binned"] == len(kept) and st["n_outside"] == fin.sum() - len(kept)
    k = np.array([keys[q] for q in kept])
    order = kept[np.lexsort((kept, k))]          # stable: by key, then input index
    np.testing.assert_array_equal(r["perm"], order)
    counts = np.bincount(k, minlength=r["nbx"] * r["nby"])
    np.testing.assert_array_equal(r["offsets"], np.r_[0, np.cumsum(counts)])
    np.testing.assert_array_equal(r["ranges"], np.array([rngs[q] for q in order]))
    ks = np.array([keys[q] for q in order])
    bx, by = ks // r["nby"], ks % r["nby"]
    np.testing.assert_array_equal(r["lx"], (u[order] - bx * B).astype(np.float32))
    np.testing.assert_array_equal(r["ly"], (v[order] - by * B).astype(np.float32))
    rr = r["ranges"].astype(np.int64)
    assert st["useful_pairs"] == int(((rr[:, 1] - rr[:, 0] + 1) * (rr[:, 3] - rr[:, 2] + 1)).sum())


def test_O8_scan_example_spec190():
    # exclusive scan of [1,1,0,1] -> [0,1,2,2]; here as bucket counts.
    g = oracle.Grid(0.0, 0.0, 1.0, 64, 16, 1.0, 6, 1.0)   # 4 x 1 buckets of 16 (key = bx)
    x = np.array([20.5, 3.5, 55.5])   # buckets 1, 0, 3 -> counts [1,1,0,1]
    y = np.array([8.5, 8.5, 8.5])
    r = oracle.bin_points(g, 16, x, y)
    np.testing.assert_array_equal(r["offsets"], [0, 1, 2, 2, 3])
    np.testing.assert_array_equal(r["perm"], [1, 0, 2])


def test_O8_band_filter_stack_rounding():
    g = _grid(W=64, H=256, hpx=3.0)
    x, y = _points(g, 3000, 4)
    full = oracle.bin_points(g, 16, x, y)
    reach = oracle.reach_px(g)
    nr = -(-reach // 16)
    gb = _grid(W=64, H=256, hpx=3.0, rb=100, re=180)
    b = oracle.bin_points(gb, 16, x, y, stack=4)
    lo, hi = ((100 // 16 - nr) // 4) * 4, ((179 // 16 + nr) // 4 + 1) * 4 - 1
    keys = np.repeat(np.arange(len(full["offsets"]) - 1), np.diff(full["offsets"]))
    sel = (keys % full["nby"] >= lo) & (keys % full["nby"] <= hi)
    np.testing.assert_array_equal(b["perm"], full["perm"][sel])
    assert lo % 4 == 0 and (hi + 1) % 4 == 0


def test_O8_band_filter_keeps_reach_rows_and_counts_band_pairs():
    g = _grid(W=64, H=128, hpx=3.0)
    x, y = _points(g, 4000, 3)
    full = oracle.bin_points(g, 16, x, y)
    reach = oracle.reach_px(g)
    nr = -(-reach // 16)
    tot = 0
    for rb, re in ((0, 32), (32, 80), (80, 128)):
        gb = _grid(W=64, H=128, hpx=3.0, rb=rb, re=re)
        b = oracle.bin_points(gb, 16, x, y)
        # kept = full-grid binning restricted to bucket rows [rb/B - nr, (re-1)/B + nr]
        lo, hi = rb // 16 - nr, (re - 1) // 16 + nr
        nbx = full["nbx"]
        keys = np.repeat(np.arange(len(full["offsets"]) - 1), np.diff(full["offsets"]))
        nby = full["nby"]
        sel = (keys % nby >= lo) & (keys % nby <= hi)
        np.testing.assert_array_equal(b["perm"], full["perm"][sel])
        np.testing.assert_array_equal(b["ranges"], full["ranges"][sel])
        tot += b["stats"]["useful_pairs"]
    assert tot == full["stats"]["useful_pairs"]


def test_O8_generator_preset_binning_invariants():
    cloud = aisgen.generate("estuary", 20000, 5)
    x0, y0, res = aisgen.grid_for("estuary", 256)
    g = oracle.Grid(x0, y0, res, 256, 256, 2 * res, 6, 4.0)
    r = oracle.bin_points(g, 32, cloud.x, cloud.y)
    assert sorted(r["perm"].tolist()) == sorted(set(r["perm"].tolist()))
    assert np.all(np.diff(r["offsets"]) >= 0)
    assert r["stats"]["n_binned"] + r["stats"]["n_outside"] == r["stats"]["n_finite"]
    assert np.all((r["lx"] >= 0) | (r["ranges"][:, 0] == 0))


# --- O9: Douglas-Peucker ----------------------------------------------------------
def _dp_brute(P, eps):
    """Textbook recursion (SPEC.md:271's exhaustive recursive oracle)."""
    def rec(s, e):
        if e - s < 2:
            return []
        ds = [oracle.ved(P[k], P[s], P[e]) for k in range(s + 1, e)]
        k = int(np.argmax(ds)) + s + 1
        if ds[k - s - 1] > eps:
            return rec(s, k) + [k] + rec(k, e)
        return []
    return sorted({0, len(P) - 1, *rec(0, len(P) - 1)})


def test_O9_ved_examples():
    assert oracle.ved((0, 1), (0, 0), (2, 0)) == 1.0
    assert oracle.ved((1, 0), (0, 0), (2, 0)) == 0.0               # collinear
    assert oracle.ved((3, 4), (0, 0), (0, 0)) == 5.0               # degenerate chord
    rng = np.random.default_rng(1)
    for _ in range(50):                                            # 2*area/base (shoelace)
        a, b, c = rng.normal(size=(3, 2))
        area = abs((b[0] - a[0]) * (c[1] - a[1]) - (c[0] - a[0]) * (b[1] - a[1])) / 2
        assert oracle.ved(c, a, b) == pytest.approx(2 * area / np.hypot(*(b - a)), rel=1e-12)


def test_O9_dp_properties():
    rng = np.random.default_rng(3)
    lens = [2, 3, 14, 14, 40, 200]
    offs = np.r_[0, np.cumsum(lens)]
    n = offs[-1]
    x = np.cumsum(rng.normal(size=n))
    y = np.cumsum(rng.normal(size=n))
    prev = None
    for eps in (0.0, 0.1, 0.5, 1.0, 5.0):
        keep = oracle.dp_compress(x, y, offs, eps)
        for t in range(len(lens)):
            a, b = offs[t], offs[t + 1]
            idx = np.flatnonzero(keep[a:b])
            assert idx[0] == 0 and idx[-1] == b - a - 1             # endpoints kept
            P = np.c_[x[a:b], y[a:b]]
            if b - a <= 14:
                assert idx.tolist() == _dp_brute(P, eps)
            for s, e in zip(idx[:-1], idx[1:]):                     # dropped within eps
                for k in range(s + 1, e):
                    assert oracle.ved(P[k], P[s], P[e]) <= eps
            # idempotence
            again = oracle.dp_compress(P[idx, 0], P[idx, 1], [0, len(idx)], eps)
            assert again.all()
        if prev is not None:
            assert keep.sum() <= prev                               # monotone in eps
        prev = keep.sum()
    assert oracle.dp_compress(x, y, offs, 0.0).all()                # eps = 0 keeps noisy data
    col = oracle.dp_compress(np.arange(5.0), 2 * np.arange(5.0), [0, 5], 0.5)
    assert col.tolist() == [1, 0, 0, 0, 1]                          # collinear -> endpoints


@pytest.mark.parametrize("stack", [1, 4])
def test_O8_band_filter_semantics(stack):
    """The band filter pinned by what it is FOR, not by its formula: (1) completeness -- every
    finite point whose support (|j + 1/2 - v| <= R, derived here in numpy) reaches a band row
    and the raster's columns is kept; (2) locality -- a kept point's home row is within the
    reach plus one stack of the band; (3) the band's density from the kept points alone
    (renormalised by n) equals the density from all points."""
    g = _grid(W=64, H=256, hpx=3.0)
    x, y = _points(g, 3000, 7 + stack)
    rb, re = 100, 180
    gb = _grid(W=64, H=256, hpx=3.0, rb=rb, re=re)
    b = oracle.bin_points(gb, 16, x, y, stack=stack)
    kept = set(b["perm"].tolist())
    fin = np.isfinite(x) & np.isfinite(y)
    u = (x - g.x0) / g.res
    v = (y - g.y0) / g.res
    R = oracle.r_px(g)
    jj = np.arange(rb, re) + 0.5
    ii = np.arange(g.width) + 0.5
    for q in np.flatnonzero(fin):
        reaches = np.any(np.abs(jj - v[q]) <= R) and np.any(np.abs(ii - u[q]) <= R)
        if reaches:
            assert q in kept, q                           # (1) completeness
    hy = np.clip(np.floor(v[list(kept)]), 0, g.height - 1)
    reach = oracle.reach_px(g)
    assert np.all(hy >= rb - reach - 16 * stack - 16) and np.all(hy <= re - 1 + reach + 16 * stack + 16)  # (2)
    sel = np.array(sorted(kept), dtype=np.int64)
    full, nf = oracle.kde_raster(gb, x, y)
    part, nk = oracle.kde_raster(gb, x[sel], y[sel])
    np.testing.assert_allclose(part * (nk / nf), full, rtol=1e-12, atol=1e-300)  # (3)
