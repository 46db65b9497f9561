"""GPU parity of kde_snap, the paper's own pipeline (NEXT-F1: Eqs. 5-6, Alg. 3, Eqs. 12-13,
Eq. 7), against oracle/snap.py: M_D bit-exact, the Eq. 7 matrix within 1e-5 * max."""
import numpy as np
import pytest

import aisgen
from oracle import snap

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-5


def _labels(cloud):
    return np.repeat(np.arange(len(cloud.traj_offsets) - 1, dtype=np.int32), np.diff(cloud.traj_offsets))


def _kde(W, H, hpx, kernel=6, cutoff=4.0):
    from paper_2004_13653_b200 import KDE
    return KDE(0.0, 0.0, 1.0, W, H, hpx, kernel=kernel, cutoff=cutoff)


def _run(k, x, y, lab, W, H, device=True):
    cnt = torch.zeros(H * W, dtype=torch.int32, device="cuda")
    if device:
        tx, ty = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        tl = torch.from_numpy(lab).cuda() if lab is not None else None
    else:
        tx, ty, tl = torch.from_numpy(x), torch.from_numpy(y), (torch.from_numpy(lab) if lab is not None else None)
    out = k.snap(tx, ty, tl, counts=cnt)
    torch.cuda.synchronize()
    return cnt.cpu().numpy().reshape(H, W).astype(np.int64), out.cpu().numpy()


@pytest.mark.parametrize("kernel", range(8))
def test_snap_small_all_kernels_with_interpolation(kernel):
    cloud = aisgen.generate("estuary", 20_000, 11)
    lab = _labels(cloud)
    W, H, hpx = 256, 192, 3.0
    cut = 4.0 if kernel == 6 else 1.0
    M, ref = snap.snapped_kde(cloud.x, cloud.y, lab, W, H, kernel, hpx, cut)
    cnt, out = _run(_kde(W, H, hpx, kernel, cut), cloud.x, cloud.y, lab, W, H)
    np.testing.assert_array_equal(cnt, M)                 # bit-exact (integer)
    assert np.abs(out - ref).max() <= TOL * ref.max()


@pytest.mark.parametrize("hpx", [1.0, 2.5, 12.0])
def test_snap_edge_cases_host_inputs_and_no_labels(hpx):
    rng = np.random.default_rng(5)
    n = 5000
    x = np.cumsum(rng.normal(0, 40, n)) + 1.35e7
    y = np.cumsum(rng.normal(0, 40, n)) + 3.6e6
    x[::97] = np.nan                                      # breaks interpolation chains
    y[5::131] = np.inf
    lab = (np.arange(n) // 300).astype(np.int32)
    W, H = 181, 97                                        # ragged vs 256/32/64 tiles
    k = _kde(W, H, hpx)
    for L in (lab, None):
        M, ref = snap.snapped_kde(x, y, L, W, H, 6, hpx, 4.0)
        c_dev, o_dev = _run(k, x, y, L, W, H, device=True)
        c_host, o_host = _run(k, x, y, L, W, H, device=False)
        np.testing.assert_array_equal(c_dev, M)
        np.testing.assert_array_equal(c_host, M)
        np.testing.assert_array_equal(o_dev.view(np.uint32), o_host.view(np.uint32))  # deterministic
        assert np.abs(o_dev - ref).max() <= TOL * ref.max()


def test_snap_empty_and_degenerate():
    k = _kde(40, 30, 2.0)
    e = np.zeros(0)
    cnt, out = _run(k, e, e, None, 40, 30)
    assert not cnt.any() and not out.any()
    x = np.full(7, 5.0)                                   # x_max = x_min: every x~ = 1
    y = np.linspace(0.0, 1.0, 7)
    M, ref = snap.snapped_kde(x, y, None, 40, 30, 6, 2.0, 4.0)
    cnt, out = _run(k, x, y, None, 40, 30)
    np.testing.assert_array_equal(cnt, M)
    assert cnt[:, 0].sum() == 7
    assert np.abs(out - ref).max() <= TOL * ref.max()


def test_snap_full_size_C2_sampled():
    """2M estuary points with trajectory labels on 2048^2: the no-interpolation M_D
    bit-exact (vectorised Eqs. 5-6), the interpolated mass = n + sum(c_max - 1), and Eq. 7
    at sampled pixels from the oracle's own M_D."""
    cloud = aisgen.generate("estuary", 2_000_000, aisgen.SEED_BASE + 1)
    lab = _labels(cloud)
    W = H = 2048
    hpx = 4.0
    k = _kde(W, H, hpx)
    xt, yt = snap.project(cloud.x, cloud.y, W, H)
    M0 = np.zeros((H, W), np.int64)
    np.add.at(M0, (yt - 1, xt - 1), 1)
    cnt0, out0 = _run(k, cloud.x, cloud.y, None, W, H)
    np.testing.assert_array_equal(cnt0, M0)
    cnt, out = _run(k, cloud.x, cloud.y, lab, W, H)
    same = lab[:-1] == lab[1:]
    cmax = np.maximum(np.abs(np.diff(xt)), np.abs(np.diff(yt)))[same]
    assert cnt.sum() == len(cloud.x) + int(np.maximum(cmax - 1, 0).sum())
    assert (cnt >= cnt0).all()
    # Eq. 7 per sampled pixel from the GPU's (now verified) M_D, fp64
    a = snap.window_a(6, hpx, 4.0)
    w = np.array([snap.k1(6, s / hpx) for s in range(-a, a + 1)])
    rng = np.random.default_rng(1)
    iy = np.concatenate([rng.integers(0, H, 1500), [int(np.argmax(out) // W)]])
    ix = np.concatenate([rng.integers(0, W, 1500), [int(np.argmax(out) % W)]])
    Mp = np.pad(cnt.astype(np.float64), a)
    ref = np.array([w @ Mp[j:j + 2 * a + 1, i:i + 2 * a + 1][::-1, ::-1] @ w for j, i in zip(iy, ix)])
    assert np.abs(out[iy, ix] - ref).max() <= TOL * ref.max()


def test_snap_errors():
    from paper_2004_13653_b200 import KDE, KdeError, _lib
    x = torch.zeros(4, dtype=torch.float64, device="cuda")
    k = KDE(0.0, 0.0, 1.0, 32, 32, 2.0, kernel=6 | 0x100)      # radial: not separable
    with pytest.raises(KdeError) as e:
        k.snap(x, x)
    assert e.value.code == _lib.KDE_EUNSUPPORTED
    k = KDE(0.0, 0.0, 1.0, 32, 32, 2.0, rows=(0, 16))          # banded context
    with pytest.raises(KdeError) as e:
        k.snap(x, x)
    assert e.value.code == _lib.KDE_EUNSUPPORTED
    k = KDE(0.0, 0.0, 1.0, 32, 32, 2.0)
    with pytest.raises(KdeError) as e:                          # mixed host / device inputs
        k.snap(x, torch.zeros(4, dtype=torch.float64))
    assert e.value.code == _lib.KDE_EINVAL
