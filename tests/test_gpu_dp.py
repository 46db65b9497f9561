"""GPU Douglas-Peucker (kde_dp, NEXT-F3) against the serial oracle (oracle/dp_oracle.c,
pinned by tests/test_oracle_binning_dp.py): the keep mask is bit-exact."""
import numpy as np
import pytest

import aisgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gpu(x, y, offs, eps, device=True):
    from paper_2004_13653_b200 import kde_dp
    if device:
        keep, nk, rounds = kde_dp(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(),
                                  torch.from_numpy(np.asarray(offs, np.int64)).cuda(), eps)
        return keep.cpu().numpy(), nk, rounds
    return kde_dp(x, y, np.asarray(offs, np.int64), eps)


@pytest.mark.parametrize("eps", [0.0, 0.5, 1.0, 5.0, 50.0])
def test_dp_islands_bit_exact(eps):
    c = aisgen.generate("islands", 400_000, 21)
    ref = oracle.dp_compress(c.x, c.y, c.traj_offsets, eps)
    keep, nk, rounds = _gpu(c.x, c.y, c.traj_offsets, eps)
    np.testing.assert_array_equal(keep, ref)
    assert nk == int(ref.sum()) and rounds >= 1


def test_dp_adversarial_ties_degenerate_and_short():
    rng = np.random.default_rng(2)
    xs, ys, offs = [], [], [0]
    for L in [0, 1, 2, 3, 5, 17, 64, 0, 200, 1000]:
        if L:
            kind = rng.integers(0, 3)
            if kind == 0:     # collinear, equally spaced: all VED = 0 (ties everywhere)
                t = np.arange(L, dtype=float)
                x, y = 1.3e7 + 10 * t, 3.6e6 + 5 * t
            elif kind == 1:   # closed loop: degenerate chord (start == end)
                a = np.linspace(0, 2 * np.pi, L)
                x, y = 1.3e7 + 50 * np.cos(a), 3.6e6 + 50 * np.sin(a)
                x[-1], y[-1] = x[0], y[0]
            else:             # zig-zag with repeated points: exact VED ties
                x = 1.3e7 + np.arange(L) * 3.0
                y = 3.6e6 + np.where(np.arange(L) % 2, 7.0, 0.0)
                y[L // 2:] = y[:L - L // 2]
            xs.append(x)
            ys.append(y)
        offs.append(offs[-1] + L)
    x, y = np.concatenate(xs), np.concatenate(ys)
    for eps in (0.0, 1.0, 6.9, 7.0, 100.0):
        ref = oracle.dp_compress(x, y, offs, eps)
        np.testing.assert_array_equal(_gpu(x, y, offs, eps)[0], ref)
        np.testing.assert_array_equal(_gpu(x, y, offs, eps, device=False)[0], ref)  # host inputs


def test_dp_full_size_C4_and_errors():
    from paper_2004_13653_b200 import KdeError, kde_dp
    c = aisgen.generate("islands", 20_000_000, aisgen.SEED_BASE + 3)
    ref = oracle.dp_compress(c.x, c.y, c.traj_offsets, 1.0)
    keep, nk, _ = _gpu(c.x, c.y, c.traj_offsets, 1.0)
    np.testing.assert_array_equal(keep, ref)
    with pytest.raises(KdeError):
        kde_dp(c.x[:10], c.y[:10], np.array([0, 10], np.int64), -1.0)
    k, nk, r = kde_dp(np.zeros(0), np.zeros(0), np.array([0], np.int64), 1.0)
    assert nk == 0 and r == 0


def _raw_dp(x, y, offs, keep, eps=1.0):
    """The C ABI call itself (no binding-side checks)."""
    import ctypes

    from paper_2004_13653_b200 import _lib
    nk, r = ctypes.c_int64(0), ctypes.c_int64(0)
    return _lib._L.kde_dp(_lib._ptr(x), _lib._ptr(y), _lib._ptr(offs), int(offs.shape[0]) - 1, float(eps),
                          _lib._ptr(keep), 0, None, ctypes.byref(nk), ctypes.byref(r))


def test_dp_mixed_pointers_rejected():
    from paper_2004_13653_b200 import _lib, kde_dp
    x = torch.zeros(8, dtype=torch.float64, device="cuda")
    keep = torch.empty(8, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):  # the binding checks devices first
        kde_dp(x, x, np.array([0, 8], np.int64), 1.0, keep=keep)
    assert _raw_dp(x, x, np.array([0, 8], np.int64), keep) == _lib.KDE_EINVAL  # and so does the C ABI


def test_dp_bad_offsets_rejected():
    """offsets not starting at 0, decreasing, or not matching the buffers."""
    from paper_2004_13653_b200 import _lib, kde_dp
    x = np.zeros(8)
    keep = np.zeros(8, np.uint8)
    for offs in ([1, 8], [0, 5, 3, 8], [0, 9]):
        with pytest.raises(ValueError):
            kde_dp(x, x, np.array(offs, np.int64), 1.0, keep=keep)
    for offs in ([1, 8], [0, 5, 3, 8]):  # host offsets through the raw C call
        assert _raw_dp(x, x, np.array(offs, np.int64), keep) == _lib.KDE_EINVAL
    xd = torch.zeros(8, dtype=torch.float64, device="cuda")
    kd = torch.empty(8, dtype=torch.uint8, device="cuda")
    od = torch.tensor([0, 6, 2, 8], dtype=torch.int64, device="cuda")  # device offsets, decreasing
    assert _raw_dp(xd, xd, od, kd) == _lib.KDE_EINVAL


def test_dp_nan_points_match_serial_recursion():
    """a non-finite coordinate gives a NaN VED, which the recursion's `d > dmax`
    never selects; the GPU maps it below every finite VED (bit-exact kept set)."""
    c = aisgen.generate("islands", 200_000, 33)
    x, y = c.x.copy(), c.y.copy()
    rng = np.random.default_rng(4)
    idx = rng.choice(len(x), 300, replace=False)
    x[idx[:150]] = np.nan
    y[idx[150:250]] = np.inf
    x[idx[250:]] = -np.inf
    for eps in (0.0, 1.0, 5.0):
        ref = oracle.dp_compress(x, y, c.traj_offsets, eps)
        keep, nk, _ = _gpu(x, y, c.traj_offsets, eps)
        np.testing.assert_array_equal(keep, ref)
        assert nk == int(ref.sum())
