"""Per-rank work of the row-band split, measured one band at a time on ONE B200.

    python tools/band_projection.py [--config C4] [--path tensor] [--ranks 2 4 8]

For N ranks, the work-balanced bands (paper_2004_13653_b200.dist.plan_bands_balanced) are
evaluated one after the other on the same GPU, each in its own banded context on the full
(replicated) point set: load (band compaction + binning) + eval, device time by CUDA events
(median of 5 after 3 warm-ups).  The max over bands is the compute part of an N-GPU step;
the collectives (point all-gather, raster gather over NVLink) are not included -- this box
has one GPU.  Prints one JSON line per N.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2004_13653_b200 import KDE  # noqa: E402
from paper_2004_13653_b200 import dist as kdist  # noqa: E402


def timed(fn, reps=5, warm=3):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--path", default="tensor")
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    cloud, x0, y0, res = bench._gen(cfg)
    W = H = cfg["W"]
    h = cfg["hpx"] * res
    xd, yd = torch.from_numpy(cloud.x).cuda(), torch.from_numpy(cloud.y).cuda()
    R = cfg["cutoff"] * cfg["hpx"]
    v = np.clip(np.floor((cloud.y - y0) / res), 0, H - 1).astype(np.int64)
    work = kdist.row_workload(np.bincount(v, minlength=H), H, R)
    for n in args.ranks:
        bands = kdist.plan_bands_balanced(work, n) if n > 1 else [(0, H)]
        per, phases = [], []
        for rb, re in bands:
            if re <= rb:
                per.append(0.0)
                continue
            k = KDE(x0, y0, res, W, H, h, kernel=cfg["kernel"], cutoff=cfg["cutoff"],
                    rows=(rb, re) if n > 1 else None)
            out = torch.empty((re - rb, W), dtype=torch.float32, device="cuda")

            def step():
                k.load(xd, yd)
                k.eval(args.path, out)
            per.append(timed(step))
            k.set_timing(True)
            step()
            torch.cuda.synchronize()
            phases.append({kk: round(vv, 4) for kk, vv in k.timing().items()})
            k.set_timing(False)
            k.close()
        print(json.dumps({"config": args.config, "path": args.path, "ranks": n, "bands": bands,
                          "band_ms": [round(t, 4) for t in per], "max_band_ms": round(max(per), 4),
                          "phases_of_max_band": phases[int(np.argmax(per))] if phases else None,
                          "note": "one band at a time on one B200; collectives excluded"}), flush=True)


if __name__ == "__main__":
    main()
