"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bars (BASELINE.json north_star):
  * binning, indices, stats: bit-exact;
  * direct fp32 path: max |gpu - oracle| <= 1e-5 * max(oracle) over the evaluated set;
  * tensor-core path: <= 2e-3 * max(oracle).
Radial parity excludes pixels the oracle flags as fp32 near-ties of the disk
test (R3).
"""
import numpy as np
import pytest
import torch

import oracle
from tests.gpu_cases import (CONFIGS, THREADS, adversarial, case, hottest_bucket_tile,
                             sample_pixels)

pytestmark = pytest.mark.gpu

TOL_DIRECT = 1e-5
TOL_TENSOR = 2e-3


def _kde(c, kernel=None, rows=None, cutoff=None):
    from paper_2004_13653_b200 import KDE
    k = c.get("kernel", 6) if kernel is None else kernel
    cut = c.get("cutoff", 4.0) if cutoff is None else cutoff
    return KDE(c["x0"], c["y0"], c["res"], c["W"], c["H"], c["h"], kernel=k, cutoff=cut, rows=rows)


def _grid(c, kernel=None, rows=None, cutoff=None):
    rb, re = (0, 0) if rows is None else rows
    return oracle.Grid(c["x0"], c["y0"], c["res"], c["W"], c["H"], c["h"],
                       c.get("kernel", 6) if kernel is None else kernel,
                       c.get("cutoff", 4.0) if cutoff is None else cutoff, rb, re)


def _err(gpu, ref, ties=None):
    d = np.abs(gpu.astype(np.float64) - ref)
    if ties is not None:
        d = np.where(ties.astype(bool), 0.0, d)
    return d.max() / max(ref.max(), 1e-300)


# --- binning: bit-exact ------------------------------------------------------------
BIN_CASES = {
    "C1": lambda: case("estuary", 10_000, 256, 2.0, seed=CONFIGS["C1"][6]),
    "adversarial": lambda: adversarial(),
    "islands_ragged": lambda: case("islands", 50_000, 300, 3.0, seed=4, H=170),
    "big_h": lambda: case("promontory", 30_000, 512, 20.0, seed=5),
}


@pytest.mark.parametrize("name", list(BIN_CASES))
@pytest.mark.parametrize("rows", [None, (64, 150)])
def test_binning_bit_exact(name, rows):
    c = BIN_CASES[name]()
    if rows is not None and rows[1] > c["H"]:
        rows = (rows[0], c["H"])
    k = _kde(c, rows=rows)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    got = k.bins()
    want = oracle.bin_points(_grid(c, rows=rows), got["stats"]["bucket"], c["x"], c["y"],
                             stack=got["stats"]["stack"])
    for f in ("n_in", "n_finite", "n_binned", "n_outside", "useful_pairs"):
        assert got["stats"][f] == want["stats"][f], f
    np.testing.assert_array_equal(got["offsets"], want["offsets"])
    np.testing.assert_array_equal(got["perm"], want["perm"])
    np.testing.assert_array_equal(got["ranges"], want["ranges"])
    np.testing.assert_array_equal(got["lx"].view(np.uint32), want["lx"].view(np.uint32))
    np.testing.assert_array_equal(got["ly"].view(np.uint32), want["ly"].view(np.uint32))
    assert got["stats"]["reach_px"] == oracle.reach_px(_grid(c))
    # every kept window lies inside its group's window [bx*B - F, bx*B + B - 1 + F]
    # (the splat pass relies on it; F = floor(R + 1/2))
    B = got["stats"]["bucket"]
    F = int(np.floor(oracle.r_px(_grid(c)) + 0.5))
    keys = np.repeat(np.arange(len(got["offsets"]) - 1), np.diff(got["offsets"]))
    bx, by = keys // got["stats"]["nby"], keys % got["stats"]["nby"]  # column-major keys
    r = got["ranges"]
    assert np.all(r[:, 0] >= bx * B - F) and np.all(r[:, 1] <= bx * B + B - 1 + F)
    assert np.all(r[:, 2] >= by * B - F) and np.all(r[:, 3] <= by * B + B - 1 + F)


def test_binning_host_and_device_inputs_identical():
    c = BIN_CASES["adversarial"]()
    a = _kde(c).load(torch.from_numpy(c["x"]), torch.from_numpy(c["y"]))
    b = _kde(c).load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    ra, rb = a.eval().cpu().numpy(), b.eval().cpu().numpy()
    np.testing.assert_array_equal(ra.view(np.uint32), rb.view(np.uint32))
    assert a.stats() == b.stats()


# --- direct path: full raster, all kernels x forms -----------------------------------
@pytest.mark.parametrize("kernel", [k | f for f in (0, 0x100) for k in range(8)])
def test_direct_C1_full_raster(kernel):
    preset, n, W, hpx, _, cut, seed = CONFIGS["C1"]
    c = case(preset, n, W, hpx, seed=seed)
    k = _kde(c, kernel=kernel)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("direct").cpu().numpy()
    ref, nf, ties = oracle.kde_raster(_grid(c, kernel=kernel), c["x"], c["y"], threads=THREADS,
                                      want_ties=True)
    assert nf == k.stats()["n_finite"]
    assert _err(gpu, ref, ties if kernel & 0x100 else None) <= TOL_DIRECT


@pytest.mark.parametrize("kernel", [0, 2, 5, 6, 7, 6 | 0x100, 1 | 0x100])
@pytest.mark.parametrize("cutoff", [4.0, 0.6])
def test_direct_adversarial_ragged(kernel, cutoff):
    c = adversarial()
    k = _kde(c, kernel=kernel, cutoff=cutoff)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("direct").cpu().numpy()
    ref, _, ties = oracle.kde_raster(_grid(c, kernel=kernel, cutoff=cutoff), c["x"], c["y"],
                                     threads=THREADS, want_ties=True)
    assert _err(gpu, ref, ties if kernel & 0x100 else None) <= TOL_DIRECT


def test_direct_hot_pixel_split_k():
    """All points in (nearly) one pixel: m ~ 6e4 contributions per pixel, forces split-K."""
    rng = np.random.default_rng(3)
    n = 60_000
    res = 10.0
    c = dict(x=1e6 + (40.3 + rng.normal(0, 0.2, n)) * res, y=2e6 + (21.7 + rng.normal(0, 0.2, n)) * res,
             x0=1e6, y0=2e6, res=res, W=90, H=50, h=3.0 * res, kernel=6, cutoff=4.0)
    k = _kde(c)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("direct").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_DIRECT


def test_direct_empty_and_all_nan():
    c = adversarial()
    k = _kde(c)
    k.load(torch.zeros(0, dtype=torch.float64), torch.zeros(0, dtype=torch.float64))
    assert not k.eval().any()
    k.load(torch.full((10,), float("nan"), dtype=torch.float64), torch.zeros(10, dtype=torch.float64))
    assert not k.eval().any()
    assert k.stats()["n_finite"] == 0


def test_direct_deterministic_and_band_sharding_bitwise():
    c = case("estuary", 200_000, 512, 4.0, seed=21)
    full = _kde(c).load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    a = full.eval().cpu().numpy()
    b = full.eval().cpu().numpy()
    np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
    parts = []
    bands = [(0, 64), (64, 200), (200, 448), (448, 512)]
    for rb, re in bands:
        kb = _kde(c, rows=(rb, re)).load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
        parts.append(kb.eval().cpu().numpy())
        assert kb.stats()["n_finite"] == full.stats()["n_finite"]
    cat = np.concatenate(parts, axis=0)
    np.testing.assert_array_equal(cat.view(np.uint32), a.view(np.uint32))


@pytest.mark.parametrize("cfg", ["C2"])
@pytest.mark.parametrize("kernel", [6, 2])
def test_direct_full_size_sampled(cfg, kernel):
    """BASELINE config at full size, in the bench's launch configuration, on sampled pixels."""
    preset, n, W, hpx, _, cut, seed = CONFIGS[cfg]
    c = case(preset, n, W, hpx, seed=seed)
    k = _kde(c, kernel=kernel)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("direct").cpu().numpy()
    hx, hy = hottest_bucket_tile(c["x"], c["y"], c["x0"], c["y0"], c["res"], W, W)
    tiles = [(hx, hy, 64, 64), (0, 0, 16, 16), (W - 16, W - 16, 16, 16)]
    pi, pj = sample_pixels(W, W, (0, W), gpu=gpu, tiles=tiles, n_random=2048, seed=seed)
    ref, _ = oracle.kde_pixels(_grid(c, kernel=kernel), c["x"], c["y"], pi, pj, threads=THREADS)
    got = gpu[pj, pi]
    assert np.abs(got - ref).max() <= TOL_DIRECT * ref.max()
    assert ref.max() >= 0.5 * gpu.max()  # the sample contains the peak region


def test_error_paths_on_device():
    from paper_2004_13653_b200 import KdeError, _lib
    c = adversarial()
    k = _kde(c, kernel=6 | 0x100)
    with pytest.raises(KdeError) as e:
        k.eval()
    assert e.value.code == _lib.KDE_ESTATE
    k.load(torch.from_numpy(c["x"]), torch.from_numpy(c["y"]))
    with pytest.raises(KdeError) as e:
        k.eval("tensor")
    assert e.value.code == _lib.KDE_EUNSUPPORTED
    # the binding checks the caller's raster buffer (the ABI takes a plain pointer)
    with pytest.raises(ValueError):
        k.eval("direct", out=torch.empty(c["W"] * c["H"] - 1, dtype=torch.float32, device="cuda"))
    with pytest.raises(TypeError):
        k.eval("direct", out=torch.empty(c["W"] * c["H"], dtype=torch.float64, device="cuda"))


# --- tensor-core Gaussian path (a4): 2e-3 * max -----------------------------------------
def _tc(c, rows=None, cutoff=None):
    k = _kde(c, kernel=6, rows=rows, cutoff=cutoff)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    return k


def test_tensor_C1_full_raster():
    preset, n, W, hpx, _, cut, seed = CONFIGS["C1"]
    c = case(preset, n, W, hpx, seed=seed)
    k = _tc(c)
    gpu = k.eval("tensor").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=6), c["x"], c["y"], threads=THREADS)
    err = _err(gpu, ref)
    assert err <= TOL_TENSOR, err
    d = k.eval("direct").cpu().numpy()
    assert np.abs(gpu - d).max() <= TOL_TENSOR * d.max()  # O11: TC vs direct


@pytest.mark.parametrize("cutoff", [4.0, 2.5])
@pytest.mark.parametrize("hpx", [1.5, 3.0, 6.0])
def test_tensor_adversarial_ragged(cutoff, hpx):
    c = adversarial(hpx=hpx)
    k = _tc(c, cutoff=cutoff)
    gpu = k.eval("tensor").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=6, cutoff=cutoff), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_TENSOR


def test_tensor_hot_pixel_split_and_sharding_bitwise():
    rng = np.random.default_rng(3)
    n = 60_000
    res = 10.0
    c = dict(x=1e6 + (40.3 + rng.normal(0, 3, n)) * res, y=2e6 + (61.7 + rng.normal(0, 5, n)) * res,
             x0=1e6, y0=2e6, res=res, W=90, H=150, h=3.0 * res, kernel=6, cutoff=4.0)
    full = _tc(c)
    a = full.eval("tensor").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c), c["x"], c["y"], threads=THREADS)
    assert _err(a, ref) <= TOL_TENSOR
    b = full.eval("tensor").cpu().numpy()
    np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
    parts = [_tc(c, rows=r).eval("tensor").cpu().numpy() for r in ((0, 40), (40, 100), (100, 150))]
    np.testing.assert_array_equal(np.concatenate(parts).view(np.uint32), a.view(np.uint32))


def test_tensor_full_size_sampled_C2():
    preset, n, W, hpx, _, cut, seed = CONFIGS["C2"]
    c = case(preset, n, W, hpx, seed=seed)
    k = _tc(c)
    gpu = k.eval("tensor").cpu().numpy()
    hx, hy = hottest_bucket_tile(c["x"], c["y"], c["x0"], c["y0"], c["res"], W, W)
    pi, pj = sample_pixels(W, W, (0, W), gpu=gpu, tiles=[(hx, hy, 64, 64)], n_random=2048, seed=seed)
    ref, _ = oracle.kde_pixels(_grid(c, kernel=6), c["x"], c["y"], pi, pj, threads=THREADS)
    assert np.abs(gpu[pj, pi] - ref).max() <= TOL_TENSOR * ref.max()


@pytest.mark.parametrize("hpx,cutoff", [(20.0, 4.0), (36.0, 4.0), (14.0, 4.5)])
def test_tensor_large_support_subwindows(hpx, cutoff):
    """Windows wider than the 128 TMEM lanes (C5 at h >= 16 px): nsubx x nsuby MMA tiles."""
    c = adversarial(W=260, H=230, n=4000, hpx=hpx)
    k = _tc(c, cutoff=cutoff)
    gpu = k.eval("tensor").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=6, cutoff=cutoff), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_TENSOR
    d = k.eval("direct").cpu().numpy()
    assert np.abs(gpu - d).max() <= TOL_TENSOR * d.max()  # O11


# --- all eight product kernels on the tensor-core path (NEXT-F2) ----------------------------
@pytest.mark.parametrize("kernel", range(8))
def test_tensor_all_kernels_C1_full_raster(kernel):
    preset, n, W, hpx, _, cut, seed = CONFIGS["C1"]
    c = case(preset, n, W, hpx, seed=seed)
    k = _kde(c, kernel=kernel)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("tensor").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=kernel), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_TENSOR


@pytest.mark.parametrize("kernel", [0, 1, 5, 7])
@pytest.mark.parametrize("hpx", [1.5, 6.0, 40.0])
def test_tensor_all_kernels_adversarial(kernel, hpx):
    """Ragged grid, halo points, NaN/Inf, boundary ties; compact kernels (c_eff = 1) and
    the sub-window geometry at h = 40 px."""
    c = adversarial(W=180 if hpx > 10 else 100, H=150 if hpx > 10 else 70, hpx=hpx)
    k = _kde(c, kernel=kernel)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("tensor").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=kernel), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_TENSOR


# --- C3 / C4 at full size, in the bench's configuration, on sampled pixels ------------------
_BIG = {}


def _big(cfg):
    if cfg not in _BIG:
        preset, n, W, hpx, _, cut, seed = CONFIGS[cfg]
        _BIG.clear()
        _BIG[cfg] = case(preset, n, W, hpx, seed=seed)
    return _BIG[cfg]


def _sampled_check(c, kernel, path, tol, n_random=768, cutoff=None):
    from paper_2004_13653_b200 import KDE
    W = c["W"]
    cut = c.get("cutoff", 4.0) if cutoff is None else cutoff
    k = KDE(c["x0"], c["y0"], c["res"], W, W, c["h"], kernel=kernel, cutoff=cut)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval(path).cpu().numpy()
    hx, hy = hottest_bucket_tile(c["x"], c["y"], c["x0"], c["y0"], c["res"], W, W)
    pi, pj = sample_pixels(W, W, (0, W), gpu=gpu, tiles=[(hx, hy, 24, 24)], n_random=n_random, seed=7)
    g = oracle.Grid(c["x0"], c["y0"], c["res"], W, W, c["h"], kernel, cut)
    ref, nf, ties = oracle.kde_pixels(g, c["x"], c["y"], pi, pj, threads=THREADS, want_ties=True)
    assert nf == k.stats()["n_finite"]
    d = np.abs(gpu[pj, pi].astype(np.float64) - ref)
    if kernel & 0x100:
        d = np.where(ties.astype(bool), 0.0, d)
    assert d.max() <= tol * ref.max(), (d.max() / ref.max())
    assert ref.max() >= 0.5 * gpu.max()
    return k


@pytest.mark.parametrize("kernel", list(range(8)) + [2 | 0x100, 6 | 0x100])
def test_C3_all_kernels_direct_sampled(kernel):
    """Chengshan-Jiao-shaped 5M points, 4096^2, h = 8 px: all 8 Table-1 kernels."""
    _sampled_check(_big("C3"), kernel, "direct", TOL_DIRECT)


@pytest.mark.parametrize("kernel", range(8))
def test_C3_all_kernels_tensor_sampled(kernel):
    _sampled_check(_big("C3"), kernel, "tensor", TOL_TENSOR)


@pytest.mark.parametrize("eps", [None, 0.5, 1.0, 5.0])
def test_C4_raw_and_dp_compressed(eps):
    """Zhoushan-shaped 20M points at 8192^2, raw and Douglas-Peucker-compressed (oracle DP,
    PAPER.md:116-129) at the Table-4 thresholds; direct and tensor paths."""
    c = dict(_big("C4"))
    if eps is not None:
        keep = oracle.dp_compress(c["x"], c["y"], c["cloud"].traj_offsets, eps).astype(bool)
        c["x"], c["y"] = c["x"][keep], c["y"][keep]
        assert 0 < keep.sum() < keep.size
    _sampled_check(c, 6, "direct", TOL_DIRECT, n_random=384)
    _sampled_check(c, 6, "tensor", TOL_TENSOR, n_random=384)


# --- split-fp16 tensor-core accuracy mode (NEXT-F4): the DIRECT path's 1e-5 bar ---------------
@pytest.mark.parametrize("kernel", [6, 2, 5, 7])
def test_tensor_split_C1_full_raster(kernel):
    preset, n, W, hpx, _, cut, seed = CONFIGS["C1"]
    c = case(preset, n, W, hpx, seed=seed)
    k = _kde(c, kernel=kernel)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("tensor_split").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=kernel), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_DIRECT


@pytest.mark.parametrize("hpx", [1.5, 6.0, 36.0])
def test_tensor_split_adversarial(hpx):
    c = adversarial(W=260 if hpx > 10 else 100, H=230 if hpx > 10 else 70, hpx=hpx)
    k = _tc(c)
    gpu = k.eval("tensor_split").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=6), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_DIRECT
    # deterministic, and the plain tensor path's plan is shared
    np.testing.assert_array_equal(gpu.view(np.uint32), k.eval("tensor_split").cpu().numpy().view(np.uint32))
    assert _err(k.eval("tensor").cpu().numpy(), ref) <= TOL_TENSOR


def test_tensor_split_full_size_sampled_C2():
    preset, n, W, hpx, _, cut, seed = CONFIGS["C2"]
    c = case(preset, n, W, hpx, seed=seed)
    k = _tc(c)
    gpu = k.eval("tensor_split").cpu().numpy()
    hx, hy = hottest_bucket_tile(c["x"], c["y"], c["x0"], c["y0"], c["res"], W, W)
    pi, pj = sample_pixels(W, W, (0, W), gpu=gpu, tiles=[(hx, hy, 64, 64)], n_random=2048, seed=seed)
    ref, _ = oracle.kde_pixels(_grid(c, kernel=6), c["x"], c["y"], pi, pj, threads=THREADS)
    assert np.abs(gpu[pj, pi] - ref).max() <= TOL_DIRECT * ref.max()


# --- fp16 operand range (R11): a cutoff far past fp16's normal range -----------------
@pytest.mark.parametrize("hpx", [1.5, 4.0])
def test_tensor_fp16_range_cutoff9(hpx):
    """The tensor path rounds 1-D factors exp(-s^2/2) to fp16.  At cutoff 9 the smallest kept
    factor is exp(-40.5) = 2.6e-18, far below fp16's smallest subnormal (6e-8): such factors
    flush to 0 (or a subnormal).  Each lost product is < 6e-8 of the peak pair (1 x 1), so the
    2e-3 * max bar holds unless ~3e4 far-tail pairs outweigh the peak pixel -- checked here on
    an estuary cloud (hot lanes + sparse tails) at h = 1.5 px (the per-factor exp2 branch of
    the recurrence guard) and 4 px."""
    c = case("estuary", 100_000, 300, hpx, seed=31, H=260)
    k = _tc(c, cutoff=9.0)
    gpu = k.eval("tensor").cpu().numpy()
    ref, _ = oracle.kde_raster(_grid(c, kernel=6, cutoff=9.0), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_TENSOR
    d = k.eval("direct").cpu().numpy()
    assert _err(d, ref) <= TOL_DIRECT


@pytest.mark.parametrize("m64", ["1", "0"])
@pytest.mark.parametrize("kernel", [6, 2])
def test_tensor_tile_shapes_M64_and_M128(monkeypatch, m64, kernel):
    """The tensor-core path's two tile shapes: M = 64 tiles (4-bucket stacks, two
    accumulators per TMEM column slice, 16 workers) and M = 128 tiles (KDE_TC_M64=0: 12-bucket
    stacks, 10 workers) on the same ragged, clustered input -- each against the oracle, and the
    reported M matches the geometry."""
    monkeypatch.setenv("KDE_TC_M64", m64)
    c = case("estuary", 40_000, 200, 4.0, seed=83, H=170)
    k = _kde(c, kernel=kernel)
    k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
    gpu = k.eval("tensor").cpu().numpy()
    st = k.stats()
    k.close()
    assert st["tc_m"] == (64 if m64 == "1" else 128)
    assert st["main_kernel"] == 3  # the per-warp kernel (eval_tc5.cu) for both shapes
    ref, _ = oracle.kde_raster(_grid(c, kernel=kernel), c["x"], c["y"], threads=THREADS)
    assert _err(gpu, ref) <= TOL_TENSOR


@pytest.mark.parametrize("path", ["tensor", "direct"])
def test_strip_combine_bitwise_equals_tile_combine(monkeypatch, path):
    """The strip combine (8-column strips, warp-uniform block skipping) adds the same blocks in
    the same order as the 32 x 32-tile combine: bitwise-identical rasters on a clustered input
    with ragged raster edges (combine pass round 2)."""
    c = case("estuary", 60_000, 260, 4.0, seed=91, H=230)

    def run(strip):
        monkeypatch.setenv("KDE_COMBINE_STRIP", strip)
        k = _kde(c, kernel=6)
        k.load(torch.from_numpy(c["x"]).cuda(), torch.from_numpy(c["y"]).cuda())
        out = k.eval(path).cpu().numpy()
        k.close()
        return out

    a, b = run("1"), run("0")
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert a.max() > 0
