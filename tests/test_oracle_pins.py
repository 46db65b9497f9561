"""Pins for the KDE oracle.

Each test checks ``oracle/`` against something other than itself: values the
paper prints (Table 1 constants, tests/golden/), closed forms derived by hand
(power sums, Dirichlet kernel, Poisson summation), mathematical invariants
(symmetry, translation, linearity, rank one), an independent numpy brute
force, and the paper's own KDE (Eq. 7 convolution) via
scipy.signal.convolve2d.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy.signal import convolve2d

import oracle
from oracle.brute import kde_bruteforce

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RAD = oracle.RADIAL


def _centre_grid(kernel, hpx, res=2.5, cutoff=4.0, size=None):
    """Grid with a single point at the centre of pixel (c, c)."""
    R = hpx * (cutoff if kernel & 0xFF == 6 else min(cutoff, 1.0))
    size = size or int(2 * math.ceil(R) + 7)
    c = size // 2
    g = oracle.Grid(x0=1000.0, y0=-500.0, res=res, width=size, height=size, h=hpx * res,
                    kernel=kernel, cutoff=cutoff)
    x = np.array([g.x0 + (c + 0.5) * res])
    y = np.array([g.y0 + (c + 0.5) * res])
    return g, x, y, c


def _golden_centres():
    vals = {}
    with open(os.path.join(GOLDEN, "table1_centre_values.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            kid, _, num, den = line.split()
            vals[int(kid)] = eval(num, {"pi": math.pi}) / eval(den, {"pi": math.pi})
    return vals


# --- O1: Table 1 centre values (paper-printed constants) ----------------------
@pytest.mark.parametrize("kernel", range(8))
def test_O1_centre_value_is_table1_constant(kernel):
    want = _golden_centres()[kernel]
    for hpx in (1.0, 3.0, 4.5):
        g, x, y, c = _centre_grid(kernel, hpx)
        out, n = oracle.kde_pixels(g, x, y, [c], [c])
        assert n == 1
        assert out[0] == pytest.approx(want / hpx ** 2, rel=1e-14)


# --- O3: mass closed forms (product form, point at a pixel centre, integer h) --
def _psum(p, h):
    """sum_{m=-h}^{h} |m|^p as an exact integer (p >= 1)."""
    return 2 * sum(m ** p for m in range(1, h + 1))


def _mass1d_exact(kernel, h):
    """Exact 1-D mass (1/h) sum_{|m|<=h} k(m/h), derived by binomial expansion in
    power sums, in rational arithmetic (independent of the oracle's code)."""
    H = Fraction(h)
    n0 = 2 * h + 1
    if kernel == 0:
        return Fraction(1, 2) * n0 / H                      # = 1 + 1/(2h)
    if kernel == 1:
        return (n0 - Fraction(_psum(1, h), h)) / H          # = 1
    if kernel == 2:
        return Fraction(3, 4) * (n0 - Fraction(_psum(2, h), h ** 2)) / H
    if kernel == 3:
        return Fraction(15, 16) * (n0 - 2 * Fraction(_psum(2, h), h ** 2)
                                   + Fraction(_psum(4, h), h ** 4)) / H
    if kernel == 4:
        return Fraction(35, 32) * (n0 - 3 * Fraction(_psum(2, h), h ** 2)
                                   + 3 * Fraction(_psum(4, h), h ** 4)
                                   - Fraction(_psum(6, h), h ** 6)) / H
    if kernel == 5:
        return Fraction(70, 81) * (n0 - 3 * Fraction(_psum(3, h), h ** 3)
                                   + 3 * Fraction(_psum(6, h), h ** 6)
                                   - Fraction(_psum(9, h), h ** 9)) / H
    raise ValueError(kernel)


@pytest.mark.parametrize("kernel", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("h", [1, 2, 3, 5])
def test_O3_mass_polynomial_kernels_exact(kernel, h):
    g, x, y, c = _centre_grid(kernel, float(h))
    out, _ = oracle.kde_raster(g, x, y)
    m1 = float(_mass1d_exact(kernel, h))
    assert out.sum() == pytest.approx(m1 * m1, rel=1e-13)


def test_O3_closed_forms_by_hand():
    # the three forms quoted in DESIGN.md §4 (and SURVEY.md O3)
    for h in (2, 4, 7):
        assert _mass1d_exact(1, h) == 1
        assert _mass1d_exact(0, h) == 1 + Fraction(1, 2 * h)         # pins inclusive tie
        assert _mass1d_exact(2, h) == 1 - Fraction(1, 4 * h * h)


@pytest.mark.parametrize("h", [1, 2, 4, 9])
def test_O3_mass_cosine_dirichlet(h):
    # (pi/(4h)) sum_{|m|<=h} cos(pi m/(2h)) = (pi/(4h)) cot(pi/(4h))  (Dirichlet kernel)
    g, x, y, c = _centre_grid(7, float(h))
    out, _ = oracle.kde_raster(g, x, y)
    a = math.pi / (4 * h)
    assert out.sum() == pytest.approx((a / math.tan(a)) ** 2, rel=1e-13)


@pytest.mark.parametrize("h", [2.0, 3.0, 5.5])
def test_O3_mass_gaussian_poisson(h):
    # cutoff 9: tails < erfc(9/sqrt2) ~ 2e-19; Poisson summation gives
    # sum_m phi((m+d)/h)/h = 1 + O(exp(-2 pi^2 h^2)) < 1e-30 for h >= 2.
    g, x, y, c = _centre_grid(6, h, cutoff=9.0)
    out, _ = oracle.kde_raster(g, x, y)
    assert out.sum() == pytest.approx(1.0, abs=1e-13)
    # off-centre point: still exactly 1 (Poisson summation is shift-invariant)
    x2 = x + 0.37 * g.res
    y2 = y - 0.21 * g.res
    out2, _ = oracle.kde_raster(g, x2, y2)
    assert out2.sum() == pytest.approx(1.0, abs=1e-13)


def test_O3_gaussian_cutoff4_truncation():
    # cutoff 4, h=2: 1-D mass = 1 - tail, tail = sum_{|m|>8} phi(m/2)/2 (explicit series)
    g, x, y, c = _centre_grid(6, 2.0, cutoff=4.0)
    out, _ = oracle.kde_raster(g, x, y)
    tail = sum(math.exp(-(m / 2) ** 2 / 2) / math.sqrt(2 * math.pi) / 2 for m in range(9, 80)) * 2
    assert out.sum() == pytest.approx((1 - tail) ** 2, rel=1e-12)
    assert abs(out.sum() - math.erf(4 / math.sqrt(2)) ** 2) < 1e-4


@pytest.mark.parametrize("kernel", range(8))
def test_O3_radial_integrates_to_one(kernel):
    # Midpoint Riemann sum over the disk, h = 60 px; error from the boundary
    # lattice is O(h^-1) for the discontinuous Uniform, O(h^-2) otherwise.
    hpx = 60.0
    cutoff = 9.0 if kernel == 6 else 1.0
    g, x, y, c = _centre_grid(kernel | RAD, hpx, cutoff=cutoff, res=1.0)
    x = x + 0.31
    y = y + 0.17
    out, _ = oracle.kde_raster(g, x, y, threads=8)
    tol = {0: 2e-3, 6: 1e-12}.get(kernel, 1e-5)
    assert out.sum() == pytest.approx(1.0, abs=tol)


# --- O2: product identity (rank one) ------------------------------------------
@pytest.mark.parametrize("kernel", range(8))
def test_O2_product_form_is_rank_one(kernel):
    rng = np.random.default_rng(kernel)
    g = oracle.Grid(x0=0.0, y0=0.0, res=1.0, width=40, height=36, h=6.3, kernel=kernel, cutoff=2.0)
    x = np.array([19.3 + rng.uniform()])
    y = np.array([17.1 + rng.uniform()])
    out, _ = oracle.kde_raster(g, x, y)
    sv = np.linalg.svd(out, compute_uv=False)
    assert sv[0] > 0
    assert sv[1] <= 1e-13 * sv[0]
    if kernel != 0:  # radial form is not rank one (except the Gaussian)
        g.kernel = kernel | RAD
        r, _ = oracle.kde_raster(g, x, y)
        sv = np.linalg.svd(r, compute_uv=False)
        assert sv[1] > 1e-6 * sv[0] or kernel == 6


# --- O4: symmetry ------------------------------------------------------------
@pytest.mark.parametrize("kernel", [0, 2, 5, 6, 7, 6 | RAD, 1 | RAD])
def test_O4_mirror_and_transpose(kernel):
    rng = np.random.default_rng(7)
    W = 48
    res = 0.5  # power of two: mirrored coordinates are exact in fp64
    g = oracle.Grid(x0=0.0, y0=0.0, res=res, width=W, height=W, h=3.0 * res, kernel=kernel,
                    cutoff=3.0)
    x = rng.uniform(-2, W * res + 2, 60)
    y = rng.uniform(-2, W * res + 2, 60)
    base, _ = oracle.kde_raster(g, x, y)
    mx, _ = oracle.kde_raster(g, W * res - x, y)
    np.testing.assert_allclose(mx, base[:, ::-1], rtol=1e-12, atol=1e-15)
    my, _ = oracle.kde_raster(g, x, W * res - y)
    np.testing.assert_allclose(my, base[::-1, :], rtol=1e-12, atol=1e-15)
    tr, _ = oracle.kde_raster(g, y, x)
    np.testing.assert_allclose(tr, base.T, rtol=1e-12, atol=1e-15)


# --- O5: translation and linearity --------------------------------------------
def test_O5_translation_and_linearity():
    rng = np.random.default_rng(11)
    g = oracle.Grid(x0=0.0, y0=0.0, res=1.0, width=64, height=64, h=2.5, kernel=3, cutoff=1.0)
    x = rng.uniform(20, 30, 40)
    y = rng.uniform(20, 30, 40)
    a, _ = oracle.kde_raster(g, x, y)
    b, _ = oracle.kde_raster(g, x + 7, y - 5)
    np.testing.assert_allclose(b[15:59, 7:], a[20:64, :57], rtol=1e-12, atol=1e-15)
    x2 = rng.uniform(0, 64, 25)
    y2 = rng.uniform(0, 64, 25)
    r2, n2 = oracle.kde_raster(g, x2, y2)
    ru, nu = oracle.kde_raster(g, np.r_[x, x2], np.r_[y, y2])
    np.testing.assert_allclose(40 * a + n2 * r2, nu * ru, rtol=1e-12, atol=1e-13)


# --- O6: independent numpy brute force ----------------------------------------
@pytest.mark.parametrize("kernel", [k | f for k in range(8) for f in (0, RAD)])
def test_O6_bruteforce_agrees(kernel):
    rng = np.random.default_rng(100 + kernel)
    W, H, res = 29, 23, 3.7
    x0, y0 = 1.35e7, 3.2e6  # Mercator-metre magnitudes
    x = x0 + rng.uniform(-4 * res, (W + 4) * res, 50)
    y = y0 + rng.uniform(-4 * res, (H + 4) * res, 50)
    x[3] = np.nan
    y[7] = np.inf
    for hpx, cut in ((1.7, 4.0), (3.0, 1.0), (2.2, 0.7)):
        g = oracle.Grid(x0, y0, res, W, H, hpx * res, kernel, cut)
        ref = kde_bruteforce(x0, y0, res, W, H, hpx * res, kernel, cut, x, y)
        out, n = oracle.kde_raster(g, x, y)
        assert n == 48
        assert np.max(np.abs(out - ref)) <= 1e-12 * max(ref.max(), 1e-300)


# --- O7: the paper's Eq. 7 convolution on snapped points -------------------------
@pytest.mark.parametrize("kernel", range(8))
def test_O7_snapped_points_equal_eq7_convolution(kernel):
    """Points projected by Eqs. 5-6 (ceil rule) and placed at their
    cell centres: direct KDE * n h^2 == M_D (x) f (Eq. 7), zero padding."""
    rng = np.random.default_rng(kernel)
    u, v = 40, 32
    xr = rng.normal(0, 1, 300)
    yr = rng.normal(0, 1, 300)
    # Eq. 5-6: x~ = ceil((x - xmin)/(xmax - xmin) * (u - 1)) + 1 in [1, u]
    xt = np.ceil((xr - xr.min()) / (xr.max() - xr.min()) * (u - 1)).astype(int) + 1
    yt = np.ceil((yr - yr.min()) / (yr.max() - yr.min()) * (v - 1)).astype(int) + 1
    M = np.zeros((v, u))
    np.add.at(M, (yt - 1, xt - 1), 1.0)            # M_D(x~, y~) = C
    hpx = 3.0
    g = oracle.Grid(x0=0.0, y0=0.0, res=1.0, width=u, height=v, h=hpx, kernel=kernel,
                    cutoff=1.0 if kernel != 6 else 2.0)
    a = int(math.floor(oracle.r_px(g)))
    offs = np.arange(-a, a + 1) / hpx
    f = np.outer([oracle.k1(kernel, s) for s in offs], [oracle.k1(kernel, s) for s in offs])
    conv = convolve2d(M, f, mode="same", boundary="fill", fillvalue=0.0)
    out, n = oracle.kde_raster(g, xt - 0.5, yt - 0.5)  # cell centres of pixel (x~-1, y~-1)
    np.testing.assert_allclose(out * n * hpx * hpx, conv, rtol=1e-12, atol=1e-12)


def test_empty_input_gives_zeros():
    g = oracle.Grid(0.0, 0.0, 1.0, 8, 8, 2.0, 6, 4.0)
    out, n = oracle.kde_raster(g, np.zeros(0), np.zeros(0))
    assert n == 0 and not out.any()
    out, n = oracle.kde_raster(g, np.array([np.nan]), np.array([1.0]))
    assert n == 0 and not out.any()
