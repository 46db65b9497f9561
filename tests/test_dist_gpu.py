"""Row-band sharding on the GPU through torchrun (a6): 2 ranks, assembled == unsharded bitwise."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_row_bands_bitwise(tmp_path):
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    out = tmp_path / "verdict.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), str(out), backend]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    v = json.loads(out.read_text())
    assert v["direct"] and v["tensor"] and v["n_finite"], v
    assert v["direct_fused"] and v["tensor_fused"], v  # NEXT-F4 peer-memory assembly
    bands = v["bands"]
    assert bands[0][0] == 0 and bands[-1][1] == 600 and all(a[1] == b[0] for a, b in zip(bands, bands[1:]))


def test_bench_two_ranks_prints_one_line():
    """bench.py's N > 1 path (row bands + all-gather, max over ranks) end to end; gloo when
    the box has one GPU (both ranks share it)."""
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "C1", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--dist-backend", backend]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "row-bands x2"
    assert d["useful_pairs"] > 0 and d["roofline"]["frac"] > 0


@pytest.mark.parametrize("fused", [False, True])
def test_bench_gpus_flag_spawns_ranks_itself(fused):
    """`bench.py --gpus 2` without torchrun launches its own 2 ranks (rank 0 prints); with
    --fused the bands go into rank 0's raster through peer memory (NEXT-F4)."""
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "C1",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--dist-backend", backend] + (["--fused"] if fused else [])
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "row-bands x2" + (" fused-peer" if fused else "")
