"""Row-band sharding host logic on CPU: world_size-2 gloo process group.

The band planner and the all-gather assembly of paper_2004_13653_b200/dist.py are run
in two processes; each rank evaluates its band with the oracle (test infrastructure, the
GPU is not available here) and the assembled raster must equal the full-raster oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _load_dist():
    # dist.py only needs torch; load it without importing the package (no libkde.so here)
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_kde_dist", os.path.join(ROOT, "paper_2004_13653_b200", "dist.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_plan_bands_cover_and_align():
    d = _load_dist()
    for H, world, tile in [(2048, 8, 256), (2048, 3, 256), (256, 8, 256), (1000, 4, 64), (70, 2, 256)]:
        bands = d.plan_bands(H, world, tile)
        assert len(bands) == world
        assert bands[0][0] == 0 and max(b[1] for b in bands) == H
        for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
            assert a1 == b0 or (b0 == b1 == H)
        for rb, re in bands[:-1]:
            if re < H:
                assert re % 64 == 0  # tile aligned


def _worker(rank, world, port, H, W, seed, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = _load_dist()
    rng = np.random.default_rng(seed)
    x = rng.uniform(-3, W + 3, 400)
    y = rng.uniform(-3, H + 3, 400)
    bands = d.plan_bands(H, world, tile=64)
    rb, re = bands[rank]
    maxr = max(b - a for a, b in bands)
    band = torch.zeros((maxr, W), dtype=torch.float64)
    if re > rb:
        g = oracle.Grid(0.0, 0.0, 1.0, W, H, 2.5, 6, 4.0, rb, re)
        r, _ = oracle.kde_raster(g, x, y)
        band[: re - rb] = torch.from_numpy(r)
    full = d.assemble(band, bands, H, W)
    if rank == 0:
        g = oracle.Grid(0.0, 0.0, 1.0, W, H, 2.5, 6, 4.0)
        ref, _ = oracle.kde_raster(g, x, y)
        q.put(float(np.abs(full.numpy() - ref).max()))
    dist.destroy_process_group()


@pytest.mark.parametrize("H", [130, 200])
def test_two_rank_band_assembly_equals_full_raster(H):
    world, W = 2, 48
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) == 0.0


def test_row_workload_is_the_support_convolution():
    d = _load_dist()
    H, R = 50, 3.2
    counts = np.zeros(H)
    counts[10] = 5
    counts[49] = 2
    w = d.row_workload(counts, H, R)
    r = 4  # ceil(R)
    expect = np.zeros(H)
    expect[10 - r:10 + r + 1] += 5
    expect[49 - r:] += 2
    np.testing.assert_array_equal(w, expect)


def test_plan_bands_balanced_cuts_equal_work():
    d = _load_dist()
    rng = np.random.default_rng(3)
    H = 2048
    # lane-skewed rows: most points in two narrow lanes
    rows = np.concatenate([rng.normal(300, 10, 80_000), rng.normal(1500, 30, 40_000), rng.uniform(0, H, 10_000)])
    counts = np.bincount(np.clip(rows.astype(int), 0, H - 1), minlength=H)
    work = d.row_workload(counts, H, 16.0)
    for world in (2, 3, 4, 8):
        bands = d.plan_bands_balanced(work, world, tile=32)
        assert len(bands) == world and bands[0][0] == 0
        live = [b for b in bands if b[1] > b[0]]
        assert live[-1][1] == H
        assert all(a[1] == b[0] for a, b in zip(live, live[1:]))
        assert all(rb % 32 == 0 for rb, _ in live)
        shares = [work[rb:re].sum() / work.sum() for rb, re in live]
        # each cut lands within one 32-row tile of the exact quantile: the largest share is
        # bounded by 1/world plus the heaviest 32-row window on each side
        cs = np.concatenate([[0], np.cumsum(work)])
        heaviest = max(cs[i + 32] - cs[i] for i in range(H - 32)) / work.sum()
        assert max(shares) <= 1.0 / world + 2 * heaviest + 1e-12, (world, shares)
    eq = d.plan_bands(H, 8, 256)  # equal bands would give the lane band most of the work
    assert max(work[rb:re].sum() for rb, re in eq) / work.sum() > 0.5


def _worker_points(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = _load_dist()
    x = torch.arange(11, dtype=torch.float64)
    y = -torch.arange(11, dtype=torch.float64)
    xs, ys = d.shard_points(x, y, rank, world)
    gx, gy = d.gather_points(xs, ys)
    keep = torch.isfinite(gx)
    ok = bool(torch.equal(gx[keep], x) and torch.equal(gy[keep], y))  # order preserved, NaN padding only
    # gather of the padded bands to rank 0
    H, W = 7, 3
    rows = [(0, 4), (4, 7)]
    band = torch.full((4, W), float(rank + 1))
    full = d.gather_to_root(band, rows, H, W)
    if rank == 0:
        ok = ok and bool(torch.equal(full[:4], torch.full((4, W), 1.0)) and torch.equal(full[4:], torch.full((3, W), 2.0)))
    else:
        ok = ok and full is None
    q.put((rank, ok))
    dist.destroy_process_group()


def test_two_rank_point_sharding_and_root_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_points, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert res == {0: True, 1: True}
