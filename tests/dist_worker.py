"""torchrun worker for tests/test_dist_gpu.py: row-band sharded KDE on the GPU(s).

Every rank takes its 1/P shard of the same synthetic points (NaN-padded), the ShardedKDE
all-gathers the set, plans work-balanced bands from the all-reduced row histogram, bins the
band's compacted points, evaluates its band and gathers the heatmap to rank 0, which compares
it with an unsharded KDE, bitwise, and writes the verdict to argv[1].  With one GPU both ranks share cuda:0 and the collective runs on
gloo (NCCL refuses two ranks on one device); on a multi-GPU box use nccl.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2004_13653_b200 import KDE  # noqa: E402
from paper_2004_13653_b200.dist import PeerRaster, ShardedKDE, shard_points  # noqa: E402
from tests.gpu_cases import case  # noqa: E402


def main():
    out_path, backend = sys.argv[1], sys.argv[2]
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = int(os.environ.get("LOCAL_RANK", "0")) % ngpu
    torch.cuda.set_device(dev)
    dist.init_process_group(backend)
    res = {}
    for path in ("direct", "tensor"):
        c = case("estuary", 150_000, 640, 4.0, seed=33, H=600)
        sk = ShardedKDE(c["x0"], c["y0"], c["res"], c["W"], c["H"], c["h"], device=dev, tile=32)
        xs, ys = shard_points(torch.from_numpy(c["x"]).cuda(dev), torch.from_numpy(c["y"]).cuda(dev), rank, world)
        sk.load(xs, ys)
        full = sk.eval(path)
        full = full.cpu().numpy() if full is not None else None
        peer = PeerRaster(c["H"], c["W"], device=dev)  # NEXT-F4: bands written into rank 0's raster
        fused = sk.eval(path, peer=peer)
        fused = fused.cpu().numpy() if fused is not None else None
        peer.close()
        if rank == 0:
            ref = KDE(c["x0"], c["y0"], c["res"], c["W"], c["H"], c["h"], device=dev)
            ref.load(torch.from_numpy(c["x"]).cuda(dev), torch.from_numpy(c["y"]).cuda(dev))
            r = ref.eval(path).cpu().numpy()
            res[path] = bool(np.array_equal(full.view(np.uint32), r.view(np.uint32)))
            res[path + "_fused"] = bool(np.array_equal(fused.view(np.uint32), r.view(np.uint32)))
            res["bands"] = sk.rows
            res["n_finite"] = sk.kde.stats()["n_finite"] == ref.stats()["n_finite"]
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(res, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
