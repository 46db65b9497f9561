"""C5 at full size (BASELINE.json configs[4]): Zhoushan-shaped 50M points on a 16384^2 raster
(1 GiB fp32), Gaussian, bandwidth sweep h = 1, 4, 32 px (cutoff 4h), direct and tensor-core
paths, in the bench's launch configuration.  Sampled pixels (the hottest 16x16 tile, 256
seeded pixels, the GPU argmax +- 2) against the fp64 oracle.

The oracle is called on the points that can reach the sampled pixels (every point whose
support box, widened by 2 px, contains a sampled pixel: the exact support test S of the
oracle then runs on that superset), and its density -- normalised by the
subset's n -- is rescaled by n_subset / n_all (density = sum / (n h^2), exact in fp64 up to
one rounding).  Bars: direct 1e-5 * max, tensor 2e-3 * max (north star)."""
import numpy as np
import pytest
import torch

import aisgen
import oracle
from tests.gpu_cases import THREADS, sample_pixels

pytestmark = pytest.mark.gpu

W = 16384
N = 50_000_000
_CLOUD = {}


def _cloud():
    if "c" not in _CLOUD:
        c = aisgen.generate("islands", N, aisgen.SEED_BASE + 4)
        x0, y0, res = aisgen.grid_for("islands", W)
        u = (c.x - x0) / res
        v = (c.y - y0) / res
        cell = 64  # coarse cells for the prefilter (index of every point by cell)
        cu = np.clip(np.floor(u / cell), -1, W // cell).astype(np.int64) + 1
        cv = np.clip(np.floor(v / cell), -1, W // cell).astype(np.int64) + 1
        key = cv * (W // cell + 2) + cu
        order = np.argsort(key, kind="stable")
        starts = np.searchsorted(key[order], np.arange((W // cell + 2) ** 2 + 1))
        _CLOUD["c"] = (c, x0, y0, res, order, starts, cell)
    return _CLOUD["c"]


def _reaching(pi, pj, R, pre):
    """Indices of the points whose support (box of half-width R + 2 px) may contain a pixel."""
    c, x0, y0, res, order, starts, cell = pre
    nc = W // cell + 2
    reach = int(np.ceil(R + 2.0))
    cells = set()
    for i, j in zip(pi.tolist(), pj.tolist()):
        for cj in range((j - reach) // cell, (j + reach) // cell + 1):
            for ci in range((i - reach) // cell, (i + reach) // cell + 1):
                cu, cv = min(max(ci, -1), W // cell) + 1, min(max(cj, -1), W // cell) + 1
                cells.add(cv * nc + cu)
    idx = np.concatenate([order[starts[k]:starts[k + 1]] for k in sorted(cells)])
    return np.sort(idx)


@pytest.mark.parametrize("hpx", [1.0, 4.0, 32.0])
def test_C5_full_size_sampled(hpx):
    from paper_2004_13653_b200 import KDE
    pre = _cloud()
    c, x0, y0, res = pre[:4]
    k = KDE(x0, y0, res, W, W, hpx * res, kernel="gaussian", cutoff=4.0)
    k.load(torch.from_numpy(c.x).cuda(), torch.from_numpy(c.y).cuda())
    st = k.stats()
    assert st["n_finite"] == N
    g = oracle.Grid(x0, y0, res, W, W, hpx * res, 6, 4.0)
    R = oracle.r_px(g)
    ref = None
    for path, tol in (("direct", 1e-5), ("tensor", 2e-3)):
        out = k.eval(path)
        am = int(torch.argmax(out).item())
        if ref is None:
            # hottest 16x16 tile (of the point histogram), 256 seeded pixels, GPU argmax +- 2
            u = np.floor((c.x - x0) / res)
            v = np.floor((c.y - y0) / res)
            ok = (u >= 0) & (u < W) & (v >= 0) & (v < W)
            hist = np.bincount(((v[ok] // 16) * (W // 16) + u[ok] // 16).astype(np.int64))
            t = int(np.argmax(hist))
            tiles = [((t % (W // 16)) * 16, (t // (W // 16)) * 16, 16, 16)]
            gm = np.zeros((1, W), np.float32)
            pi, pj = sample_pixels(W, W, (0, W), tiles=tiles, n_random=256, seed=11)
            j0, i0 = divmod(am, W)
            extra = [(i0 + di, j0 + dj) for dj in range(-2, 3) for di in range(-2, 3)
                     if 0 <= i0 + di < W and 0 <= j0 + dj < W]
            pi = np.concatenate([pi, np.array([e[0] for e in extra], np.int32)])
            pj = np.concatenate([pj, np.array([e[1] for e in extra], np.int32)])
            sel = _reaching(pi, pj, R, pre)
            val, nsub = oracle.kde_pixels(g, c.x[sel], c.y[sel], pi, pj, threads=THREADS)
            ref = val * (nsub / N)
            del gm
        got = out[torch.from_numpy(pj.astype(np.int64)).cuda(), torch.from_numpy(pi.astype(np.int64)).cuda()]
        got = got.double().cpu().numpy()
        err = np.abs(got - ref).max() / ref.max()
        assert err <= tol, (path, hpx, err)
        assert ref.max() >= 0.5 * float(out.max())  # the sample holds the peak region
        del out
        torch.cuda.empty_cache()
    k.close()
