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
