"""bench.py host logic on CPU: the reference arm (the oracle) and the `--gpus N` self-spawn
(torch.distributed.run with N ranks; rank 0 alone prints one JSON line)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "1"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "evals/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_gpus_flag_spawns_ranks_and_rank0_prints_once():
    d = _run(["--impl", "reference", "--gpus", "2", "--config", "C1", "--steps", "1", "--warmup", "1"])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


def test_default_config_is_the_metric_config():
    sys.path.insert(0, ROOT)
    import bench
    import argparse  # noqa: F401
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--config", default="C4"' in src
    c = bench.CONFIGS["C4"]
    assert (c["preset"], c["n"], c["W"], c["hpx"], c["kernel"]) == ("islands", 20_000_000, 8192, 4.0, "gaussian")
