#!/usr/bin/env python
"""Benchmark of the gridded-KDE hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--dp-eps E]
                    [--path auto|direct|tensor|tensor_split|snap]
    python bench.py --impl reference ...      # the fp64 CPU oracle on the host cores

Default workload: C4, the config BASELINE.json's metric is quoted on (Zhoushan-Islands-
shaped 20M raw points, 8192^2, Gaussian h = 4 px, cutoff 4h); --dp-eps 0.5|1|5 evaluates
the same trajectories Douglas-Peucker-compressed by the library's kde_dp (PAPER.md
Table 4 thresholds).  `--gpus N` outside torchrun spawns N ranks itself.

A step is one pass of the whole hot path over one batch of synthetic input that is
already resident in HBM: kde_load_points (a1 convert/keys, a2 stable counting sort +
gather, plan) followed by kde_eval (a3 direct or a4 tensor-core evaluation, a5 scale +
store).  Under torchrun (N > 1) each rank owns a tile-aligned row band of the raster,
bins the replicated point set with the band's halo filter, evaluates its band, and an
NCCL all-gather assembles the heatmap (a6) inside the timed step.

Metric (BASELINE.json): kernel evaluations per second = useful (pixel, point) pairs
inside the support (kde_stats.useful_pairs, summed over bands) / step time; heatmap
pixels/s is reported beside it.  Timing: W untimed warm-ups, then K steps, each
preceded by an L2 flush (a 512 MiB write) outside its CUDA-event bracket; barrier +
synchronize around the whole timed region; max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# BASELINE.json configs -> concrete synthetic inputs
CONFIGS = {
    "C1": dict(preset="estuary", n=10_000, W=256, hpx=2.0, kernel="gaussian", cutoff=4.0, idx=0),
    "C2": dict(preset="estuary", n=2_000_000, W=2048, hpx=4.0, kernel="gaussian", cutoff=4.0, idx=1),
    "C3": dict(preset="promontory", n=5_000_000, W=4096, hpx=8.0, kernel="gaussian", cutoff=4.0, idx=2),
    "C4": dict(preset="islands", n=20_000_000, W=8192, hpx=4.0, kernel="gaussian", cutoff=4.0, idx=3),
    # bandwidth sweep h = 1..32 px (--hpx); 16384^2 = 1 GiB fp32 raster
    "C5": dict(preset="islands", n=50_000_000, W=16384, hpx=8.0, kernel="gaussian", cutoff=4.0, idx=4),
}
WORKLOAD = {
    "C2": "South-Channel-Yangtze-Estuary-shaped 2M points, 2048x2048, Gaussian h=4px cutoff 4h",
    "C1": "10k estuary points, 256x256, Gaussian h=2px cutoff 4h",
    "C3": "Chengshan-Jiao-Promontory-shaped 5M points, 4096x4096, h=8px",
    "C4": "Zhoushan-Islands-shaped 20M points, 8192x8192, Gaussian h=4px",
    "C5": "Zhoushan-Islands-shaped 50M points, 16384x16384, Gaussian, bandwidth sweep h=1-32px",
}
METRIC = "kernel evals/sec (useful pixel-point pairs) and heatmap pixels/sec"
UNIT = "evals/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


def _traffic(key):
    """dram read+write bytes per launch of the dominant kernel, from the committed ncu
    capture of exactly this workload (profiles/traffic.json, keyed "<config>/<path>/<kernel>"
    by profiles/summarize.py); None when no capture of this workload exists."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def _workload_key(args):
    """The traffic/profile key of this run: config (+ bandwidth, kernel, form, DP eps)."""
    cfg = args.cfg
    k = args.config
    if args.hpx is not None:
        k += f"-h{cfg['hpx']:g}"
    if args.kernel is not None:
        k += f"-{cfg['kernel']}"
    if cfg["radial"]:
        k += "-radial"
    if args.dp_eps is not None:
        k += f"-dp{args.dp_eps:g}"
    return k


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every ~2 ms during the timed
    region (nvidia-smi's 50 ms floor gave only a couple of samples per region)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, dev, period=0.002):
        self.dev = dev
        self.period = period
        self.rows = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def _nvml_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.dev < len(ids) and ids[self.dev].isdigit():
                return int(ids[self.dev])
        return self.dev

    def _poll(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        if self.t is not None:
            time.sleep(self.period)
            self._stop.set()
            self.t.join(1.0)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for _, rs in self.rows for k, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml, 2 ms period"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class _Cloud:
    def __init__(self, x, y, traj_offsets):
        self.x, self.y, self.traj_offsets = x, y, traj_offsets


def _gen(cfg, dp_eps=None, device=None):
    """The config's seeded synthetic input; with dp_eps, the same trajectories compressed by
    the library's own GPU Douglas-Peucker (kde_dp) at that threshold (in
    metres) -- input preparation, outside every timed region."""
    import aisgen
    cloud = aisgen.generate(cfg["preset"], cfg["n"], aisgen.SEED_BASE + cfg["idx"])
    x0, y0, res = aisgen.grid_for(cfg["preset"], cfg["W"])
    if dp_eps is not None and device == "oracle":
        # reference arm (CPU): the serial oracle DP, which the GPU kde_dp matches bit for bit
        import oracle
        keep = oracle.dp_compress(cloud.x, cloud.y, cloud.traj_offsets, float(dp_eps)).astype(bool)
        kc = np.concatenate([[0], np.cumsum(keep.astype(np.int64))])
        cloud = _Cloud(cloud.x[keep], cloud.y[keep], kc[np.asarray(cloud.traj_offsets, np.int64)])
    elif dp_eps is not None:
        import torch

        from paper_2004_13653_b200 import kde_dp
        dev = device if device is not None else torch.device("cuda", 0)
        offs = np.asarray(cloud.traj_offsets, np.int64)
        xd, yd, od = (torch.from_numpy(a).to(dev) for a in (cloud.x, cloud.y, offs))
        keep, nk, _ = kde_dp(xd, yd, od, float(dp_eps), device=dev.index or 0)
        keep = keep.bool()
        x, y = xd[keep].cpu().numpy(), yd[keep].cpu().numpy()
        kc = np.concatenate([[0], np.cumsum(keep.cpu().numpy().astype(np.int64))])
        cloud = _Cloud(x, y, kc[offs])
        assert len(x) == nk
    return cloud, x0, y0, res


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2004_13653_b200 import KDE, KdeError

    ws, rank, local = _dist()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # validation of the N > 1 code path with several ranks on one GPU
            dist.init_process_group(args.dist_backend)
    cfg = args.cfg
    W = H = cfg["W"]
    cloud, x0, y0, res = _gen(cfg, args.dp_eps, dev)
    n_pts = len(cloud.x)
    from paper_2004_13653_b200 import dist as kdist
    xfull = torch.from_numpy(cloud.x).to(dev)
    yfull = torch.from_numpy(cloud.y).to(dev)
    if ws > 1:
        # a6: every rank holds 1/P of the points (NaN-padded shard) and the
        # step all-gathers them over NVLink; the bands are cut at equal shares of the useful-pair
        # workload (the all-reduced per-row histogram convolved with the support), once
        xs, ys = kdist.shard_points(xfull, yfull, rank, ws)
        R = (cfg["cutoff"] if cfg["kernel"] == "gaussian" else min(cfg["cutoff"], 1.0)) * cfg["hpx"]
        bands = kdist.balanced_bands_for(ys, y0, res, H, R, ws)
        del xfull, yfull
    else:
        xs, ys, bands = xfull, yfull, [(0, H)]
    rows = bands[rank]
    nrows = max(re - rb for rb, re in bands)
    k = KDE(x0, y0, res, W, H, cfg["hpx"] * res, kernel=cfg["kernel"], cutoff=cfg["cutoff"],
            radial=cfg["radial"], rows=rows if ws > 1 else None, device=local) if rows[1] > rows[0] else None
    out = torch.zeros((nrows, W), dtype=torch.float32, device=dev)
    myrows = rows[1] - rows[0]

    def points(xa, ya):
        return kdist.gather_points(xa, ya) if ws > 1 else (xa, ya)

    peer = kdist.PeerRaster(H, W, device=local) if (ws > 1 and args.fused) else None

    def assemble(o):
        if peer is not None:  # NEXT-F4: the bands are already in rank 0's raster
            return peer.complete()
        return kdist.gather_to_root(o, bands, H, W) if ws > 1 else o  # a6: NCCL gather to rank 0

    def evaluate(o):
        if peer is not None:
            from paper_2004_13653_b200 import _PATHS, kde_eval_ptr
            kde_eval_ptr(k.ctx, _PATHS[path], peer.band_ptr(rows[0]), stream.cuda_stream)
        else:
            k.eval(path, o[:myrows])
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    path = args.path
    if path == "auto":
        path = "tensor" if (not cfg["radial"]) else "direct"  # the tensor path takes product kernels

    def step():
        x, y = points(xs, ys)
        if k is not None:
            k.load(x, y)
            evaluate(out)
        return assemble(out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = k.stats() if k is not None else {"useful_pairs": 0, "kernel_launches": 0, "tc_mma_flops": 0}
    kstats = (lambda: k.stats()) if k is not None else (lambda: st)

    # --- timed region: K steps, L2 flushed before each, events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = kstats()["kernel_launches"]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = kstats()["kernel_launches"] - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / len(step_ms)
    step_stats = {"mean": round(ms, 4), "median": round(statistics.median(step_ms), 4),
                  "min": round(min(step_ms), 4)}

    # --- per-phase device times (CUDA events recorded by libkde on the streams its
    # kernels run on), for the dominant kernel's roofline
    ph = {"bin_ms": [], "plan_ms": [], "main_ms": [], "combine_ms": []}
    if k is not None:
        xg, yg = points(xs, ys)
        k.set_timing(True)
        for i in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            k.load(xg, yg)
            k.eval(path, out[:myrows])
            t = k.timing()
            for key in ph:
                ph[key].append(t[key])
        k.set_timing(False)
        del xg, yg
    phases = {key: round(sum(v) / len(v), 4) if v else 0.0 for key, v in ph.items()}
    eval_ms = phases["main_ms"]

    # --- e2e: the same step through the public API with HOST buffers (pinned): every step
    # copies its points host->device (inside kde_load_points) and reads its raster back
    # device->host.  Steps are pipelined the way a user streaming batches would: step i's
    # D2H runs on a side stream (double-buffered raster) while step i+1 uploads and bins,
    # so the two PCIe directions overlap.
    # N > 1: each rank uploads only its 1/P shard of the points, then the all-gather
    xh = xs.cpu().pin_memory()
    yh = ys.cpu().pin_memory()
    xsd, ysd = torch.empty_like(xs), torch.empty_like(ys)
    fullh = [torch.empty((H, W), dtype=torch.float32).pin_memory() for _ in range(2)]
    outs = [torch.zeros((nrows, W), dtype=torch.float32, device=dev) for _ in range(2)]
    d2h = torch.cuda.Stream(dev)
    done_ev = [torch.cuda.Event() for _ in range(2)]

    def step_e2e(i):
        o = outs[i % 2]
        done_ev[i % 2].synchronize()  # the D2H that last read this buffer has finished
        if ws > 1:
            xsd.copy_(xh, non_blocking=True)
            ysd.copy_(yh, non_blocking=True)
            x, y = points(xsd, ysd)
            if k is not None:
                k.load(x, y)
        elif k is not None:
            k.load(xh, yh)  # host buffers straight through the C ABI (H2D inside kde_load_points)
        if k is not None:
            evaluate(o)
        full = assemble(o)
        ready = torch.cuda.Event()
        ready.record(stream)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ready)
            if rank == 0:
                fullh[i % 2].copy_(full, non_blocking=True)
            done_ev[i % 2].record(d2h)

    for i in range(max(1, args.warmup // 2)):
        step_e2e(i)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        step_e2e(i)
    torch.cuda.synchronize()
    e2e = (time.perf_counter() - t0) * 1e3 / args.steps
    # context for e2e: the raw pinned host->device copy of the same 16 B/point, alone
    dx_ = torch.empty_like(xs)
    dy_ = torch.empty_like(ys)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dx_.copy_(xh, non_blocking=True)
    torch.cuda.synchronize()
    h0.record(stream)
    for _ in range(5):
        dx_.copy_(xh, non_blocking=True)
        dy_.copy_(yh, non_blocking=True)
    h1.record(stream)
    torch.cuda.synchronize()
    h2d_ms = h0.elapsed_time(h1) / 5
    del dx_, dy_

    # --- max over ranks; sum of units over ranks
    useful = st["useful_pairs"]
    vals = torch.tensor([ms, eval_ms, e2e, float(useful)], dtype=torch.float64, device=dev)
    if ws > 1:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, eval_ms, e2e = float(mx[0]), float(mx[1]), float(mx[2])
        useful = int(sm[3])
    if rank != 0:
        dist.destroy_process_group()
        return

    peaks, peak_src = _peaks()
    clocks = clk.summary()
    clk = peaks.get("sm_max_mhz", 1965.0) * 1e6
    if path == "direct" and cfg["radial"]:
        # radial forms evaluate K per pair: Gaussian / Triangular /
        # Tricube need one MUFU op per pair (ex2 or sqrt: XU pipe, 16/clk/SM), Cosine two
        # (sqrt + cos: 8/clk/SM); the polynomial ones ~4 FMA-pipe ops (s^2+t^2, clamp, poly)
        kname = cfg["kernel"]
        if kname in ("gaussian", "triangular", "tricube", "cosine"):
            per_clk = 8 if kname == "cosine" else 16
            bound, src = "xu", f"derived: 148 SMs x {per_clk} MUFU pair-evals/clk x sm_max_mhz"
        else:
            per_clk, bound, src = 32, "alu", "derived: 148 SMs x 128 FP32 ops/clk / 4 ops per pair x sm_max_mhz"
        peak = 148 * per_clk * clk / 1e9
        roof = {"bound": bound, "kernel": "splat_kernel",
                "achieved": st["useful_pairs"] / (eval_ms * 1e-3) / 1e9,
                "peak": round(peak, 1), "unit": "Gevals/s", "peak_source": f"{src} ({peak_src})"}
    elif path == "direct":
        # ALU-bound: 1 FFMA (2 flops) per useful pair; FP32 peak = 148 SMs x 128 FFMA/clk
        # x 2 flops x max SM clock
        peak = 148 * 128 * 2 * clk / 1e12
        roof = {"bound": "alu", "kernel": "splat_kernel",
                "achieved": 2.0 * st["useful_pairs"] / (eval_ms * 1e-3) / 1e12,
                "peak": round(peak, 2), "unit": "TFLOP/s",
                "peak_source": "derived: 148 SMs x 128 FP32 FMA/clk x 2 x sm_max_mhz (%s)" % peak_src}
    else:
        # tensor-pipe bound.  achieved = the METHOD's work: 2 flops per
        # useful (pixel, point) pair per kernel time, against the dense fp16 peak (fp16 dense
        # = bf16 dense rate, the guide's nominal ratio 1).  The executed MMA flops
        # (kde_stats.tc_mma_flops: chunks x 2 x 128 x N x 16 x 2, zero padding included) and
        # their tensor-pipe share are reported beside it.
        peak = peaks["bf16_tflops"]
        mma = st["tc_mma_flops"] * (3 if path == "tensor_split" else 1)  # split: 3 MMAs / K step
        useful_tf = 2.0 * st["useful_pairs"] / (eval_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "kernel": {3: "tc5_kernel"}.get(st.get("main_kernel"), "tc_splat_kernel"),
                "achieved": useful_tf,
                "peak": peak, "unit": "TFLOP/s",
                "peak_source": f"{peak_src} bf16_tflops (fp16 dense rate = bf16)",
                "achieved_counts": "2 flops per useful pair (kde_stats.useful_pairs)",
                "executed_mma_flops_per_launch": mma,
                "executed_mma_tflops": round(mma / (eval_ms * 1e-3) / 1e12, 3),
                "executed_frac": float(f"{mma / (eval_ms * 1e-3) / 1e12 / peak:.4g}"),
                "useful_share_of_mma": round(2.0 * st["useful_pairs"] / max(mma, 1), 4),
                # context for BASELINE's north star, which names a tf32 path: the same useful
                # TFLOP/s against the tf32 dense rate (1.1 of 2.25 PFLOP/s nominal: x 0.489 of
                # the measured bf16 peak; B200_PROFILING.md)
                "frac_vs_tf32_peak": float(f"{useful_tf / (peak * 1.1 / 2.25):.4g}")}
    roof["frac"] = float(f"{roof['achieved'] / roof['peak']:.4g}")
    roof["achieved"] = float(f"{roof['achieved']:.6g}")
    roof["traffic"] = _traffic(f"{_workload_key(args)}/{path}/{roof['kernel']}")
    roof["traffic_key"] = f"{_workload_key(args)}/{path}/{roof['kernel']}"
    roof["kernel_ms"] = round(eval_ms, 4)

    line = {
        "metric": METRIC, "value": useful / (ms * 1e-3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None, "dtype": {"direct": "f32", "tensor": "f16xf16->f32",
                                        "tensor_split": "(f16+f16)x(f16+f16)->f32"}[path],
        "data": "synthetic (aisgen, seeded)",
        "config": {"workload": _workload_name(args, n_pts), "config": args.config, "path": path,
                   "n_points": n_pts, "grid": f"{W}x{H}", "h_px": cfg["hpx"],
                   "dp_eps_m": args.dp_eps,
                   "dp_compression_pct": (round(100.0 * (1 - n_pts / cfg["n"]), 2)
                                          if args.dp_eps is not None else None),
                   "cutoff": cfg["cutoff"], "kernel": cfg["kernel"],
                   "form": "radial" if cfg["radial"] else "product",
                   "parallelism": (f"row-bands x{ws}" + (" fused-peer" if args.fused else "")) if ws > 1 else "single",
                   "bands": bands if ws > 1 else None,
                   "l2": "flushed (512 MiB write) before every timed step"},
        "pixels_per_s": W * H / (ms * 1e-3),
        "useful_pairs": useful,
        "step_ms_rank0": step_stats,
        "e2e": {"value": useful / (e2e * 1e-3), "unit": UNIT, "ms_per_step": round(e2e, 4),
                "h2d_bytes_per_step": 16 * int(xs.shape[0]),
                "d2h_bytes_per_step": 4 * W * H,
                "note": "pinned host buffers; step i's D2H overlaps step i+1's H2D (pipelined)",
                "h2d_alone_ms": round(h2d_ms, 4),
                "h2d_alone_gbs": round(16 * int(xs.shape[0]) / (h2d_ms * 1e-3) / 1e9, 1)},
        "gpu_launches": int(launches),
        "phases_ms": phases,
        "clocks": clocks,
        "roofline": roof,
    }
    if not args.no_cpu_baseline and ws == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, cloud, x0, y0, res, args.cpu_seconds)
    if ws > 1:
        dist.destroy_process_group()
    print(json.dumps(line), flush=True)


def _workload_name(args, n_pts):
    w = WORKLOAD[args.config]
    if args.hpx is not None:
        w += f" at h={args.cfg['hpx']:g}px"
    if args.dp_eps is not None:
        w += f", Douglas-Peucker-compressed at eps={args.dp_eps:g} m ({n_pts} points kept)"
    return w


def run_snap(args):
    """--path snap: the paper's own pipeline (kde_snap: Eqs. 5-6 projection, Alg. 3 density
    matrix with Eqs. 12-13 interpolation along the trajectories, Eq. 7 separable
    convolution) on the config's points and grid, one GPU (other ranks exit)."""
    import torch

    from paper_2004_13653_b200 import KDE
    ws, rank, local = _dist()
    if rank != 0:
        return
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    cfg = args.cfg
    W = H = cfg["W"]
    cloud, x0, y0, res = _gen(cfg)
    lab = np.repeat(np.arange(len(cloud.traj_offsets) - 1, dtype=np.int32), np.diff(cloud.traj_offsets))
    k = KDE(x0, y0, res, W, H, cfg["hpx"] * res, kernel=cfg["kernel"], cutoff=cfg["cutoff"], device=0)
    xd, yd, ld = (torch.from_numpy(a).to(dev) for a in (cloud.x, cloud.y, lab))
    out = torch.empty((H, W), dtype=torch.float32, device=dev)
    cnt = torch.empty((H, W), dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        k.snap(xd, yd, ld, out=out, counts=cnt)
    torch.cuda.synchronize()
    launches0 = k.stats()["kernel_launches"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(0) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            k.snap(xd, yd, ld, out=out, counts=cnt)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = k.stats()["kernel_launches"] - launches0
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    # e2e: host inputs (pinned), the Eq. 7 matrix read back every step
    xh, yh, lh = (torch.from_numpy(a).pin_memory() for a in (cloud.x, cloud.y, lab))
    outh = torch.empty((H, W), dtype=torch.float32).pin_memory()
    k.snap(xh, yh, lh, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        k.snap(xh, yh, lh, out=out)
        outh.copy_(out)
    torch.cuda.synchronize()
    e2e = (time.perf_counter() - t0) * 1e3 / args.steps
    a = int(np.floor((cfg["cutoff"] if cfg["kernel"] == "gaussian" else min(cfg["cutoff"], 1.0)) * cfg["hpx"]))
    taps = W * H * (2 * a + 1) ** 2  # Eq. 7's multiply-adds (the separable form does 2(2a+1))
    n = len(cloud.x)
    mass = int(cnt.sum())
    # HBM-bound: 20 B per point in (x, y, label) + per pixel M_D zero, read; tmp write, read;
    # out write (20 B/px), plus one atomic per counted cell (interpolated cells included)
    algo = 20 * n + 20 * W * H + 4 * mass
    peaks, peak_src = _peaks()
    line = {
        "metric": "Eq. 7 kernel taps/sec of the paper's snapped pipeline (and heatmap pixels/sec)",
        "value": taps / (ms * 1e-3), "unit": "taps/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 counts, f32 convolution",
        "data": "synthetic (aisgen, seeded; trajectory labels from the generator)",
        "config": {"workload": WORKLOAD[args.config] + " - snapped pipeline (Alg. 3 + Eq. 7)",
                   "config": args.config, "path": "snap", "n_points": n, "grid": f"{W}x{H}",
                   "h_px": cfg["hpx"], "window_a": a, "kernel": cfg["kernel"],
                   "interpolated_cells": mass - n, "parallelism": "single",
                   "l2": "flushed (512 MiB write) before every timed step"},
        "pixels_per_s": W * H / (ms * 1e-3),
        "e2e": {"value": taps / (e2e * 1e-3), "unit": "taps/s", "ms_per_step": round(e2e, 4),
                "h2d_bytes_per_step": 20 * n, "d2h_bytes_per_step": 4 * W * H},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "kernel": "kde_snap (whole call)",
                     "achieved": round(algo / (ms * 1e-3) / 1e9, 1), "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": round(algo / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                     "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes": algo},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, cloud, x0, y0, res, seconds=15.0):
    """The oracle as it stands, timed on the host cores on a bounded sample: random (seeded)
    row pieces of L pixels (whole rows while W*n is small; L ~ 2e10/n at C4/C5 so a piece
    stays ~1 s of fp64 double loop), so the useful pairs in the sample are exact."""
    import oracle
    W = cfg["W"]
    kid = oracle.KERNELS.index(cfg["kernel"]) | (0x100 if cfg.get("radial") else 0)
    g = oracle.Grid(x0, y0, res, W, W, cfg["hpx"] * res, kid, cfg["cutoff"])
    cores = os.cpu_count() or 1
    n = len(cloud.x)
    L = int(min(W, max(64, 2e10 // max(n, 1))))
    b = oracle.bin_points(g, 32, cloud.x, cloud.y)
    rng_ = b["ranges"].astype(np.int64)
    rs = np.random.default_rng(7)
    npiece = W * ((W + L - 1) // L)
    order = rs.permutation(npiece)
    done, pairs, t_used = 0, 0, 0.0
    while t_used < seconds and done < npiece:
        take = order[done:done + max(1, cores)]
        pis, pjs = [], []
        for q in take:
            j, i0 = int(q % W), int(q // W) * L
            pis.append(np.arange(i0, min(i0 + L, W)))
            pjs.append(np.full(len(pis[-1]), j))
        pi = np.concatenate(pis).astype(np.int32)
        pj = np.concatenate(pjs).astype(np.int32)
        t0 = time.perf_counter()
        oracle.kde_pixels(g, cloud.x, cloud.y, pi, pj, threads=cores)
        t_used += time.perf_counter() - t0
        for q in take:
            j, i0 = int(q % W), int(q // W) * L
            i1 = min(i0 + L, W) - 1
            sel = (rng_[:, 2] <= j) & (rng_[:, 3] >= j)
            pairs += int(np.clip(np.minimum(rng_[sel, 1], i1) - np.maximum(rng_[sel, 0], i0) + 1,
                                 0, None).sum())
        done += len(take)
    return {"value": pairs / t_used, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{done} random row pieces of {L} px (of a {W}x{W} raster) over all "
                      f"{n} points ({t_used:.1f} s, fp64 double loop)",
            "seconds": round(t_used, 2)}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle
    cfg = args.cfg
    cloud, x0, y0, res = _gen(cfg, args.dp_eps, "oracle")
    per = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    import oracle
    oracle.build()
    for _ in range(args.warmup):
        cpu_baseline(cfg, cloud, x0, y0, res, seconds=per / 4)
    vals = [cpu_baseline(cfg, cloud, x0, y0, res, seconds=per) for _ in range(args.steps)]
    v = statistics.mean(x["value"] for x in vals)
    W = cfg["W"]
    ms = statistics.mean(x["seconds"] for x in vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (aisgen, seeded)",
        "config": {"workload": _workload_name(args, len(cloud.x)), "config": args.config,
                   "n_points": len(cloud.x), "grid": f"{W}x{W}", "h_px": cfg["hpx"],
                   "dp_eps_m": args.dp_eps,
                   "cutoff": cfg["cutoff"], "kernel": cfg["kernel"],
                   "form": "radial" if cfg["radial"] else "product", "parallelism": "host threads"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[0]["cores"], "kind": "oracle",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _spawn(args):
    """`bench.py --gpus N` outside torchrun: launch N ranks of this script on this node
    (one process per GPU, rendezvous on 127.0.0.1), rank 0 prints the JSON line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # C4 (Zhoushan-shaped 20M points, 8192^2, Gaussian h = 4 px) is the config BASELINE's
    # metric is quoted on
    ap.add_argument("--config", default="C4", choices=list(CONFIGS))
    ap.add_argument("--path", default="auto", choices=["auto", "direct", "tensor", "tensor_split", "snap"])
    ap.add_argument("--kernel", default=None, help="Table-1 kernel name (default: the config's)")
    ap.add_argument("--radial", action="store_true", help="radial form K(||.||/h) (DESIGN.md R1)")
    ap.add_argument("--hpx", type=float, default=None, help="bandwidth in pixels (C5 sweep)")
    ap.add_argument("--dp-eps", type=float, default=None,
                    help="Douglas-Peucker threshold in metres: evaluate the DP-compressed input "
                         "(C4: 0.5, 1.0, 5.0 -- PAPER.md Table 4 thresholds)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--fused", action="store_true",
                    help="N > 1: bands written into rank 0's raster through peer memory (NEXT-F4) "
                         "instead of the NCCL gather")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.kernel is not None:
        cfg["kernel"] = args.kernel
    if args.hpx is not None:
        cfg["hpx"] = args.hpx
    cfg["radial"] = bool(args.radial)
    args.cfg = cfg
    if args.impl == "reference":
        run_reference(args)
    elif args.path == "snap":
        run_snap(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
