"""Row-band sharding of the raster across ranks (step a6).

One process per GPU.  Each rank owns a tile-aligned band of rows [rb, re), bins the
(replicated) point set with the band's home-bucket halo filter inside libkde, evaluates
its band, and an all-gather over the process group (NCCL over NVLink on B200; gloo in
the CPU tests) assembles the H x W heatmap.  Bands are aligned to the evaluation tiles,
so every tile is computed by exactly one rank and the assembled raster is bitwise equal
to the unsharded one (tests/test_gpu_parity.py, tests/test_dist_gloo.py).
"""
from __future__ import annotations

import math


def plan_bands(H: int, world: int, tile: int = 256, min_tile: int = 64):
    """Equal tile-aligned row bands [(rb, re)] * world; trailing ranks may get (H, H)."""
    if world < 1 or H < 1:
        raise ValueError("world and H must be >= 1")
    t = tile
    while t > min_tile and math.ceil(H / t) < world:
        t //= 2
    per = math.ceil(math.ceil(H / t) / world) * t
    return [(min(r * per, H), min((r + 1) * per, H)) for r in range(world)]


def assemble(band, rows, H, W, group=None):
    """All-gather equal-height band buffers and stitch the full (H, W) raster.

    band: this rank's (max_rows, W) tensor (rows beyond its band are ignored);
    rows: the list from plan_bands.  Returns the full raster on every rank.
    """
    import torch
    import torch.distributed as dist
    world = len(rows)
    maxr = max(re - rb for rb, re in rows)
    if band.shape[0] != maxr:
        raise ValueError(f"band buffer must have {maxr} rows (padded), got {band.shape[0]}")
    buf = torch.empty((world * maxr, W), dtype=band.dtype, device=band.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, band.contiguous(), group=group)
    else:  # gloo (CPU tests, or several ranks sharing one GPU): list all-gather
        dist.all_gather(list(buf.chunk(world)), band.contiguous(), group=group)
    out = torch.empty((H, W), dtype=band.dtype, device=band.device)
    for r, (rb, re) in enumerate(rows):
        if re > rb:
            out[rb:re] = buf[r * maxr:r * maxr + (re - rb)]
    return out


class ShardedKDE:
    """A KDE whose raster is split in row bands over the ranks of a process group."""

    def __init__(self, x0, y0, res, width, height, h, kernel="gaussian", cutoff=4.0,
                 radial=False, device=0, group=None, tile=256):
        import torch.distributed as dist

        from . import KDE
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.rows = plan_bands(height, self.world, tile)
        self.H, self.W = int(height), int(width)
        self.device = device
        rb, re = self.rows[self.rank]
        self.kde = None
        if re > rb:
            self.kde = KDE(x0, y0, res, width, height, h, kernel=kernel, cutoff=cutoff,
                           radial=radial, rows=(rb, re), device=device)

    def load(self, x, y):
        if self.kde is not None:
            self.kde.load(x, y)
        return self

    def eval(self, path="direct"):
        import torch
        maxr = max(re - rb for rb, re in self.rows)
        band = torch.zeros((maxr, self.W), dtype=torch.float32,
                           device=torch.device("cuda", self.device))
        if self.kde is not None:
            rb, re = self.rows[self.rank]
            self.kde.eval(path, out=band[: re - rb])
        return assemble(band, self.rows, self.H, self.W, self.group)
