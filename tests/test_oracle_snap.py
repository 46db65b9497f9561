"""Pins for the snapped-pipeline oracle (oracle/snap.py; NEXT-F1: Eqs. 5-8, 12-13,
Alg. 3).  CPU only."""
import numpy as np
import pytest
from scipy.signal import convolve2d

import oracle
from oracle import brute, snap


# --- Eqs. 5-6 projection ------------------------------------------------------------------
def test_projection_extremes_and_grid_points():
    u, v = 11, 6
    # x at exact fractions k/(u-1) of the span: x~ = k + 1 (ceil of an integer); the
    # extremes land on cells 1 and u (Eq. 5's range [1, u])
    x = np.array([0.0, 10.0, 3.0, 7.0, 3.5, 9.999])
    y = np.array([2.0, 7.0, 3.0, 4.5, 2.0, 7.0])
    xt, yt = snap.project(x, y, u, v)
    assert list(xt) == [1, 11, 4, 8, 5, 11]
    # y span 5 over v - 1 = 5 cells: y~ = ceil(y - 2) + 1
    assert list(yt) == [1, 6, 2, 4, 1, 6]


def test_projection_nonfinite_and_degenerate():
    x = np.array([1.0, np.nan, 3.0, np.inf])
    y = np.array([5.0, 1.0, 5.0, 2.0])
    xt, yt = snap.project(x, y, 4, 4)
    assert list(xt) == [1, -1, 4, -1]
    assert list(yt) == [1, -1, 1, -1]        # y_max = y_min over the finite points
    xt, _ = snap.project(np.array([np.nan]), np.array([0.0]), 4, 4)
    assert list(xt) == [-1]


def test_projection_monotone_in_range():
    rng = np.random.default_rng(0)
    x = rng.normal(1.3e7, 3e3, 2000)
    y = rng.normal(3.6e6, 3e3, 2000)
    xt, yt = snap.project(x, y, 257, 129)
    assert xt.min() == 1 and xt.max() == 257 and yt.min() == 1 and yt.max() == 129
    o = np.argsort(x, kind="stable")
    assert np.all(np.diff(xt[o]) >= 0)


# --- Eqs. 12-13 interpolation ------------------------------------------------------------
def test_interpolation_closed_forms():
    xt = np.array([1, 6, 6, 9, 3, 4])
    yt = np.array([1, 1, 4, 1, 1, 2])
    lab = np.array([0, 0, 0, 0, 1, 1])
    cells = snap.interpolate(xt, yt, lab)
    # (1,1)->(6,1): 2..5 on row 1; (6,1)->(6,4): rows 2,3; (6,4)->(9,1): anti-diagonal;
    # (9,1)->(3,1) crosses labels: nothing; (3,1)->(4,2): c_max = 1: nothing
    assert cells == [(2, 1), (3, 1), (4, 1), (5, 1), (6, 2), (6, 3), (7, 3), (8, 2)]


def test_interpolation_rounds_half_up():
    # (1,1)->(3,2): c_max = 2, c = 1: x = 1 + [2/2] = 2, y = 1 + [1/2] = 2 (half up)
    assert snap.interpolate(np.array([1, 3]), np.array([1, 2]), np.array([5, 5])) == [(2, 2)]
    # downward: (3,2)->(1,1): y = 2 + [-1/2] = 2 + floor(0) = 2
    assert snap.interpolate(np.array([3, 1]), np.array([2, 1]), np.array([5, 5])) == [(2, 2)]
    assert snap.round_half_up_ratio(-3, 2) == -1 and snap.round_half_up_ratio(3, 2) == 2
    assert snap.round_half_up_ratio(-7, 3) == -2 and snap.round_half_up_ratio(7, 3) == 2


def test_interpolation_path_is_connected_and_mass_adds_gaps():
    rng = np.random.default_rng(4)
    n = 400
    x = np.cumsum(rng.normal(0, 3, n))
    y = np.cumsum(rng.normal(0, 3, n))
    lab = np.repeat(np.arange(8), n // 8)
    u, v = 97, 83
    xt, yt = snap.project(x, y, u, v)
    M = snap.density_matrix(x, y, lab, u, v)
    gaps = 0
    for k in range(n - 1):
        if lab[k] != lab[k + 1]:
            continue
        cmax = max(abs(xt[k + 1] - xt[k]), abs(yt[k + 1] - yt[k]))
        seg = [(xt[k], yt[k])] + snap.interpolate(xt[k:k + 2], yt[k:k + 2], lab[k:k + 2]) + \
              [(xt[k + 1], yt[k + 1])]
        gaps += max(cmax - 1, 0)
        for (a0, b0), (a1, b1) in zip(seg, seg[1:]):   # 8-connected, monotone per axis
            assert max(abs(a1 - a0), abs(b1 - b0)) <= 1
    assert M.sum() == n + gaps
    assert M.min() >= 0


# --- Eq. 7 ---------------------------------------------------------------------------------
@pytest.mark.parametrize("kernel", range(8))
def test_eq7_equals_scipy_convolve2d(kernel):
    """Eq. 7 double sum == a textbook 2-D convolution (zero padding) with the window built
    from the independently typed Table-1 factors of oracle/brute.py."""
    rng = np.random.default_rng(kernel)
    M = rng.integers(0, 5, size=(23, 31))
    hpx, cut = 2.7, (4.0 if kernel == 6 else 1.0)
    a = snap.window_a(kernel, hpx, cut)
    offs = np.arange(-a, a + 1) / hpx
    fk = brute._factor(kernel, offs)  # Table 1 k(s) with its constant
    f = np.outer(fk, fk)
    ref = convolve2d(M.astype(float), f, mode="same", boundary="fill", fillvalue=0.0)
    np.testing.assert_allclose(snap.eq7(M, kernel, hpx, cut), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kernel", [0, 2, 6, 7])
def test_snapped_pipeline_equals_continuous_kde_at_cell_centres(kernel):
    """M̄_D / (n h^2) == the continuous-KDE oracle (kde_oracle.c) evaluated on the points
    moved to their cell centres (pin O7 through the whole pipeline, no interpolation)."""
    rng = np.random.default_rng(10 + kernel)
    x = rng.normal(0, 1, 500)
    y = rng.normal(0, 2, 500)
    u, v, hpx, cut = 37, 29, 2.5, (3.0 if kernel == 6 else 1.0)
    M, Mbar = snap.snapped_kde(x, y, None, u, v, kernel, hpx, cut)
    xt, yt = snap.project(x, y, u, v)
    g = oracle.Grid(0.0, 0.0, 1.0, u, v, hpx, kernel, cut)
    dens, n = oracle.kde_raster(g, xt - 0.5, yt - 0.5)
    assert n == 500 and M.sum() == 500
    np.testing.assert_allclose(Mbar / (n * hpx * hpx), dens, rtol=1e-12, atol=1e-15)
