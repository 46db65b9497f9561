"""GPU tests of the asynchronous runtime around the kernels: host-input
staging on the copy stream, lazy per-path plans, asynchronous stats, the executed-MMA
flop count, and the per-load segment size under band sharding.

Every expected value comes from the oracle or from a fresh context evaluating the same
input (bitwise), never from the path under test itself.
"""
import numpy as np
import pytest
import torch

import oracle
from tests.gpu_cases import THREADS, case

pytestmark = pytest.mark.gpu


def _kde(c, rows=None):
    from paper_2004_13653_b200 import KDE
    return KDE(c["x0"], c["y0"], c["res"], c["W"], c["H"], c["h"], kernel=c.get("kernel", 6),
               cutoff=c.get("cutoff", 4.0), rows=rows)


def _fresh(c, path, rows=None):
    k = _kde(c, rows)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    out = k.eval(path).cpu().numpy()
    k.close()
    return out


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_loads_back_to_back_use_both_staging_buffers(pinned):
    """load(A); load(B); eval == fresh(B); then load(A); eval == fresh(A): the two
    staging buffers and the copy stream never mix the point sets."""
    a = case("estuary", 60_000, 256, 3.0, seed=31)
    b = case("islands", 45_000, 256, 3.0, seed=32)
    b.update(x0=a["x0"], y0=a["y0"], res=a["res"], h=a["h"])  # same grid
    b["x"] = a["x0"] + (b["x"] - b["x"].min()) / (np.ptp(b["x"]) + 1) * 256 * a["res"]
    b["y"] = a["y0"] + (b["y"] - b["y"].min()) / (np.ptp(b["y"]) + 1) * 256 * a["res"]

    def host(v):
        t = torch.from_numpy(v)
        return t.pin_memory() if pinned else v

    k = _kde(a)
    ha, hb = (host(a["x"]), host(a["y"])), (host(b["x"]), host(b["y"]))
    k.load(*ha)
    k.load(*hb)
    rb = k.eval("tensor").cpu().numpy()
    k.load(*ha)
    ra = k.eval("tensor").cpu().numpy()
    k.load(*hb)
    rb2 = k.eval("direct").cpu().numpy()
    np.testing.assert_array_equal(_bits(rb), _bits(_fresh(b, "tensor")))
    np.testing.assert_array_equal(_bits(ra), _bits(_fresh(a, "tensor")))
    np.testing.assert_array_equal(_bits(rb2), _bits(_fresh(b, "direct")))
    k.close()


def test_interleaved_paths_and_loads_plan_lazily():
    """Plans are built per path on first use after each load; any interleaving of loads
    and evaluations gives the fresh-context result."""
    a = case("estuary", 80_000, 320, 4.0, seed=41)
    b = case("estuary", 50_000, 320, 4.0, seed=42)
    k = _kde(a)
    dev = lambda c: (torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    k.load(*dev(a))
    d1 = k.eval("direct").cpu().numpy()
    t1 = k.eval("tensor").cpu().numpy()
    d1b = k.eval("direct").cpu().numpy()  # cached plan
    k.load(*dev(b))
    t2 = k.eval("tensor").cpu().numpy()
    d2 = k.eval("direct").cpu().numpy()
    np.testing.assert_array_equal(_bits(d1), _bits(_fresh(a, "direct")))
    np.testing.assert_array_equal(_bits(d1b), _bits(d1))
    np.testing.assert_array_equal(_bits(t1), _bits(_fresh(a, "tensor")))
    np.testing.assert_array_equal(_bits(t2), _bits(_fresh(b, "tensor")))
    np.testing.assert_array_equal(_bits(d2), _bits(_fresh(b, "direct")))
    k.close()


def test_stats_arrive_without_an_eval():
    """kde_get_stats waits for the load's asynchronous readback; the counts equal the
    binning oracle's."""
    c = case("promontory", 40_000, 200, 2.0, seed=51)
    c["x"][::97] = np.nan
    k = _kde(c)
    k.load(c["x"], c["y"])
    st = k.stats()
    ref = oracle.bin_points(oracle.Grid(c["x0"], c["y0"], c["res"], c["W"], c["H"], c["h"], 6, 4.0),
                            st["bucket"], c["x"], c["y"], stack=st["stack"])["stats"]
    for f in ("n_finite", "n_binned", "n_outside", "useful_pairs"):
        assert st[f] == ref[f], f
    assert st["tc_mma_flops"] == 0  # no tensor-core evaluation yet
    k.close()


def test_tc_mma_flops_counts_the_executed_contraction():
    c = case("estuary", 120_000, 384, 4.0, seed=61)
    k = _kde(c)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    k.eval("tensor")
    st = k.stats()
    W_win = st["bucket"] + 2 * int(np.floor(4.0 * 4.0 + 0.5))  # B + 2F, F = floor(R + 1/2)
    N = (W_win + 15) // 16 * 16
    M = st["tc_m"]  # 64: the window (B + 2F rows per bucket stack) fits M = 64 tiles
    assert M == (64 if W_win <= 48 and (64 - (W_win - st["bucket"])) // st["bucket"] >= 1 else 128)
    per_mma = 2 * M * N * 16
    f = st["tc_mma_flops"]
    assert f > 0 and f % per_mma == 0
    # every kept point sits in one chunk of 32: chunks >= n_binned / 32, and each chunk
    # holds at least one point; the contraction covers every useful pair
    chunks = f // (2 * per_mma)
    assert st["n_binned"] / 32 <= chunks <= st["n_binned"]
    assert f >= 2 * st["useful_pairs"]
    k.close()


@pytest.mark.parametrize("path", ["direct", "tensor"])
def test_large_segments_band_sharding_bitwise(path):
    """2.5 M points: the per-load segment size is above its minimum; the plan depends on
    the global point count only, so bands still concatenate bitwise to the full raster."""
    c = case("estuary", 2_500_000, 512, 4.0, seed=71)
    full = _fresh(c, path)
    parts = [_fresh(c, path, rows=r) for r in ((0, 96), (96, 300), (300, 512))]
    np.testing.assert_array_equal(_bits(np.concatenate(parts)), _bits(full))
    # and the raster is right: sampled pixels against the oracle
    rng = np.random.default_rng(0)
    pi = rng.integers(0, 512, 256).astype(np.int32)
    pj = rng.integers(0, 512, 256).astype(np.int32)
    hot = np.unravel_index(np.argmax(full), full.shape)
    pi = np.append(pi, np.int32(hot[1]))
    pj = np.append(pj, np.int32(hot[0]))
    ref, _ = oracle.kde_pixels(oracle.Grid(c["x0"], c["y0"], c["res"], 512, 512, c["h"], 6, 4.0),
                               c["x"], c["y"], pi, pj, threads=THREADS)
    tol = 1e-5 if path == "direct" else 2e-3
    assert np.abs(full[pj, pi] - ref).max() <= tol * ref.max()
