"""Row-band sharding of the raster across ranks (step a6).

One process per GPU.  The work decomposition:

* **bands** -- each rank owns rows [rb, re) of the raster.  ``plan_bands_balanced`` cuts the
  bands at equal shares of the useful-pair workload: per raster row, the number of points
  whose support reaches it (a per-row point histogram convolved with the (2R+1)-row
  support), so lane-skewed AIS data does not leave one rank with the shipping lanes.  Any
  row boundary is exact: every tile is computed by exactly one rank and the assembled raster
  is bitwise equal to the unsharded one (tests/test_gpu_parity.py, tests/test_dist_gloo.py).
* **points** -- each rank holds 1/P of the points (``shard_points``: a contiguous slice,
  padded to equal length with NaN -- non-finite points are dropped and not counted by the
  library, R4) and ``gather_points`` replicates the set with one all-gather over
  NVLink; the banded context then compacts the points whose home-bucket row lies within the
  band's reach (the cutoff-width halo) before it sorts them (csrc/bin.cu), so a rank sorts
  ~n/P + halo keys.
* **raster** -- ``gather_to_root`` gathers the padded band rasters to rank 0 only (NCCL
  gather over NVLink on the B200 box, gloo in the CPU tests); ``assemble`` (all-gather) is
  kept for callers that need the map on every rank.
"""
from __future__ import annotations

import math

import numpy as np


def plan_bands(H: int, world: int, tile: int = 256, min_tile: int = 64):
    """Equal tile-aligned row bands [(rb, re)] * world; trailing ranks may get (H, H)."""
    if world < 1 or H < 1:
        raise ValueError("world and H must be >= 1")
    t = tile
    while t > min_tile and math.ceil(H / t) < world:
        t //= 2
    per = math.ceil(math.ceil(H / t) / world) * t
    return [(min(r * per, H), min((r + 1) * per, H)) for r in range(world)]


def row_workload(row_counts, H: int, R: float):
    """Useful pairs per raster row (up to the constant 2R+1 columns): row j's work is the
    number of points whose support [v - 1/2 - R, v - 1/2 + R] contains j -- the per-row
    point histogram (rows of the home pixel, clipped to [0, H)) convolved with a box of
    2*ceil(R) + 1 rows."""
    c = np.asarray(row_counts, np.float64)
    if c.shape[0] != H:
        raise ValueError("row_counts must have H entries")
    r = int(math.ceil(R))
    cs = np.concatenate([[0.0], np.cumsum(c)])
    lo = np.clip(np.arange(H) - r, 0, H)
    hi = np.clip(np.arange(H) + r + 1, 0, H)
    return cs[hi] - cs[lo]


def plan_bands_balanced(work, world: int, tile: int = 32):
    """Bands [(rb, re)] * world cutting the cumulative per-row work at k/world, boundaries
    rounded to multiples of `tile` rows; deterministic (every rank computes the same bands
    from the same all-reduced histogram).  Ranks beyond the rows get empty (H, H) bands."""
    w = np.asarray(work, np.float64)
    H = w.shape[0]
    if world < 1 or H < 1:
        raise ValueError("world and H must be >= 1")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for k in range(1, world):
        if total > 0:
            j = int(np.searchsorted(cum, total * k / world, side="left"))
        else:
            j = (H * k) // world
        j = int(round(j / tile)) * tile
        j = min(max(j, cuts[-1]), H)
        cuts.append(j)
    cuts.append(H)
    return [(cuts[k], cuts[k + 1]) if cuts[k + 1] > cuts[k] else (H, H) for k in range(world)]


def balanced_bands_for(y, y0: float, res: float, H: int, R: float, world: int, group=None, tile: int = 32):
    """Balanced bands from this rank's point shard: per-row histogram of the home rows
    (torch.bincount on the shard's device), summed over ranks (all-reduce), then
    plan_bands_balanced on the host (the same result on every rank)."""
    import torch
    import torch.distributed as dist
    v = torch.floor((y - y0) / res)
    v = v[torch.isfinite(v)].clamp_(0, H - 1).to(torch.int64)
    hist = torch.bincount(v, minlength=H).to(torch.float64)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, group=group)
    return plan_bands_balanced(row_workload(hist.cpu().numpy(), H, R), world, tile)


def shard_points(x, y, rank: int, world: int):
    """Rank's contiguous 1/world slice of (x, y), NaN-padded to ceil(n/world) points."""
    import torch
    n = int(x.shape[0])
    per = (n + world - 1) // world
    a, b = min(rank * per, n), min((rank + 1) * per, n)
    xs = torch.full((per,), float("nan"), dtype=x.dtype, device=x.device)
    ys = torch.full((per,), float("nan"), dtype=y.dtype, device=y.device)
    xs[: b - a] = x[a:b]
    ys[: b - a] = y[a:b]
    return xs, ys


def gather_points(xs, ys, group=None):
    """All-gather the equal-length point shards: every rank gets the full (padded) set."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = int(xs.shape[0])
    xy = torch.stack([xs, ys])  # one collective for both coordinates
    out = torch.empty((world, 2, per), dtype=xs.dtype, device=xs.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, xy.contiguous(), group=group)
    else:
        dist.all_gather(list(out.unbind(0)), xy.contiguous(), group=group)
    return out[:, 0].reshape(-1), out[:, 1].reshape(-1)


def _stitch(buf, rows, maxr, H, W, dtype, device):
    import torch
    out = torch.empty((H, W), dtype=dtype, device=device)
    for r, (rb, re) in enumerate(rows):
        if re > rb:
            out[rb:re] = buf[r * maxr:r * maxr + (re - rb)]
    return out


def assemble(band, rows, H, W, group=None):
    """All-gather equal-height band buffers and stitch the full (H, W) raster on every rank.

    band: this rank's (max_rows, W) tensor (rows beyond its band are ignored);
    rows: the band list.  Returns the full raster on every rank.
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
    return _stitch(buf, rows, maxr, H, W, band.dtype, band.device)


def gather_to_root(band, rows, H, W, group=None, root: int = 0):
    """Gather the padded band buffers to `root` only and stitch the (H, W) raster there;
    other ranks return None (rank 0 receives (P-1)/P of the raster, nobody else does)."""
    import torch
    import torch.distributed as dist
    world = len(rows)
    maxr = max(re - rb for rb, re in rows)
    if band.shape[0] != maxr:
        raise ValueError(f"band buffer must have {maxr} rows (padded), got {band.shape[0]}")
    rank = dist.get_rank(group)
    if rank == root:
        buf = torch.empty((world * maxr, W), dtype=band.dtype, device=band.device)
        dist.gather(band.contiguous(), list(buf.chunk(world)), dst=root, group=group)
        return _stitch(buf, rows, maxr, H, W, band.dtype, band.device)
    dist.gather(band.contiguous(), None, dst=root, group=group)
    return None


class PeerRaster:
    """NEXT-F4, fused band assembly: rank 0's (H, W) raster mapped into every rank's address
    space (CUDA IPC through libkde: kde_ipc_export / kde_ipc_open; over NVLink P2P between
    GPUs), so each rank's kde_eval writes its band straight into rank 0's memory from the
    combine kernel's epilogue -- no separate gather.  ``complete()``: stream sync + barrier,
    after which rank 0's ``full`` holds the whole raster."""

    def __init__(self, H, W, device=0, group=None):
        import torch
        import torch.distributed as dist

        from . import kde_ipc_export, kde_ipc_open
        self.group = group
        self.rank = dist.get_rank(group)
        self.H, self.W, self.device = int(H), int(W), int(device)
        dev = torch.device("cuda", self.device)
        payload = torch.zeros(72, dtype=torch.uint8)
        self.full = None
        if self.rank == 0:
            self.full = torch.zeros((self.H, self.W), dtype=torch.float32, device=dev)
            handle, off = kde_ipc_export(self.full.data_ptr())
            payload[:64] = torch.frombuffer(bytearray(handle), dtype=torch.uint8)
            payload[64:] = torch.frombuffer(bytearray(int(off).to_bytes(8, "little", signed=True)),
                                            dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            pd = payload.to(dev)
            dist.broadcast(pd, src=0, group=group)
            payload = pd.cpu()
        else:
            dist.broadcast(payload, src=0, group=group)
        raw = bytes(payload.tolist())
        off = int.from_bytes(raw[64:], "little", signed=True)
        self._mapped = None
        if self.rank == 0:
            self.base = self.full.data_ptr()
        else:
            self._mapped = kde_ipc_open(raw[:64], self.device)
            self.base = self._mapped + off

    def band_ptr(self, rb):
        """Device address of row rb of rank 0's raster (kde_eval_ptr's `out`)."""
        return self.base + 4 * rb * self.W

    def complete(self):
        import torch
        import torch.distributed as dist
        torch.cuda.current_stream(torch.device("cuda", self.device)).synchronize()
        dist.barrier(group=self.group)
        return self.full

    def close(self):
        from . import kde_ipc_close
        if self._mapped:
            kde_ipc_close(self._mapped, self.device)
            self._mapped = None


class ShardedKDE:
    """A KDE whose raster is split in row bands over the ranks of a process group.

    ``load(xs, ys)`` takes this rank's point shard (``shard_points``), all-gathers the set,
    plans work-balanced bands on the first load (or uses `rows`), and bins it in the band's
    context; ``eval(path)`` returns the full raster on rank 0 (None elsewhere), or on every
    rank with ``everywhere=True``.
    """

    def __init__(self, x0, y0, res, width, height, h, kernel="gaussian", cutoff=4.0,
                 radial=False, device=0, group=None, rows=None, tile=32):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.args = dict(x0=x0, y0=y0, res=res, width=width, height=height, h=h, kernel=kernel,
                         cutoff=cutoff, radial=radial, device=device)
        self.H, self.W = int(height), int(width)
        self.device = device
        self.tile = tile
        self.rows = rows
        self.kde = None
        if rows is not None:
            self._make()

    def _support_px(self):
        a = self.args
        kid = a["kernel"] if isinstance(a["kernel"], int) else None
        gauss = (kid == 6) if kid is not None else (a["kernel"] == "gaussian")
        ceff = a["cutoff"] if gauss else min(a["cutoff"], 1.0)
        return ceff * a["h"] / a["res"]

    def _make(self):
        from . import KDE
        rb, re = self.rows[self.rank]
        if re > rb:
            a = self.args
            self.kde = KDE(a["x0"], a["y0"], a["res"], a["width"], a["height"], a["h"], kernel=a["kernel"],
                           cutoff=a["cutoff"], radial=a["radial"], rows=(rb, re), device=a["device"])

    def load(self, xs, ys):
        if self.rows is None:
            self.rows = balanced_bands_for(ys, self.args["y0"], self.args["res"], self.H, self._support_px(),
                                           self.world, self.group, self.tile)
            self._make()
        x, y = gather_points(xs, ys, self.group)
        if self.kde is not None:
            self.kde.load(x, y)
        return self

    def eval(self, path="direct", everywhere=False, peer: "PeerRaster | None" = None):
        """The full raster on rank 0 (None elsewhere): gathered over the process group, or --
        with `peer` (NEXT-F4) -- written by every rank's combine straight into rank 0's
        memory."""
        import torch
        if peer is not None:
            from . import _PATHS, kde_eval_ptr
            if self.kde is not None:
                rb, _ = self.rows[self.rank]
                p = _PATHS[path] if isinstance(path, str) else int(path)
                stream = torch.cuda.current_stream(torch.device("cuda", self.device)).cuda_stream
                kde_eval_ptr(self.kde.ctx, p, peer.band_ptr(rb), stream)
            return peer.complete()
        maxr = max(re - rb for rb, re in self.rows)
        band = torch.zeros((maxr, self.W), dtype=torch.float32, device=torch.device("cuda", self.device))
        if self.kde is not None:
            rb, re = self.rows[self.rank]
            self.kde.eval(path, out=band[: re - rb])
        if everywhere:
            return assemble(band, self.rows, self.H, self.W, self.group)
        return gather_to_root(band, self.rows, self.H, self.W, self.group)
