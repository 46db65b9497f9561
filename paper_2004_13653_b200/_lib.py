"""Thin ctypes binding of libkde.so (include/kde.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
converts torch tensors / numpy arrays to pointers and return codes to
exceptions.  There is no CPU fallback: if libkde.so is missing or cannot be
loaded, importing the package raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libkde.so")

KDE_UNIFORM, KDE_TRIANGULAR, KDE_EPANECHNIKOV, KDE_QUARTIC = 0, 1, 2, 3
KDE_TRIWEIGHT, KDE_TRICUBE, KDE_GAUSSIAN, KDE_COSINE = 4, 5, 6, 7
KDE_RADIAL = 0x100
KERNEL_NAMES = ["uniform", "triangular", "epanechnikov", "quartic", "triweight", "tricube",
                "gaussian", "cosine"]
KDE_PATH_DIRECT, KDE_PATH_TENSOR, KDE_PATH_TENSOR_SPLIT = 0, 1, 2
KDE_OK, KDE_EINVAL, KDE_ENOMEM, KDE_ECUDA, KDE_EUNSUPPORTED, KDE_ESTATE = 0, -1, -2, -3, -4, -5
_CODES = {KDE_EINVAL: "EINVAL", KDE_ENOMEM: "ENOMEM", KDE_ECUDA: "ECUDA",
          KDE_EUNSUPPORTED: "EUNSUPPORTED", KDE_ESTATE: "ESTATE"}

EXPORTS = ("kde_create", "kde_load_points", "kde_eval", "kde_get_stats", "kde_get_bins",
           "kde_set_timing", "kde_get_timing", "kde_snap", "kde_dp", "kde_ipc_export", "kde_ipc_open",
           "kde_ipc_close", "kde_last_error", "kde_free")


class kde_params(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("y0", ctypes.c_double), ("res", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("h", ctypes.c_double),
                ("kernel", ctypes.c_int32), ("cutoff", ctypes.c_double),
                ("row_begin", ctypes.c_int32), ("row_end", ctypes.c_int32),
                ("device", ctypes.c_int32)]


class kde_stats(ctypes.Structure):
    _fields_ = [("n_in", ctypes.c_int64), ("n_finite", ctypes.c_int64),
                ("n_binned", ctypes.c_int64), ("n_outside", ctypes.c_int64),
                ("useful_pairs", ctypes.c_int64), ("bucket", ctypes.c_int32),
                ("nbx", ctypes.c_int32), ("nby", ctypes.c_int32), ("reach_px", ctypes.c_int32),
                ("stack", ctypes.c_int32), ("band_lo", ctypes.c_int32), ("band_hi", ctypes.c_int32),
                ("kernel_launches", ctypes.c_int64), ("tc_mma_flops", ctypes.c_int64),
                ("main_kernel", ctypes.c_int32), ("tc_m", ctypes.c_int32)]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class kde_timing(ctypes.Structure):
    _fields_ = [("bin_ms", ctypes.c_float), ("plan_ms", ctypes.c_float),
                ("main_ms", ctypes.c_float), ("combine_ms", ctypes.c_float)]


class KdeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_2004_13653_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    P = ctypes.POINTER
    L.kde_create.argtypes = [P(kde_params), P(vp)]
    L.kde_load_points.argtypes = [vp, vp, vp, ctypes.c_int64]
    L.kde_eval.argtypes = [vp, ctypes.c_int32, vp, vp]
    L.kde_get_stats.argtypes = [vp, P(kde_stats)]
    L.kde_get_bins.argtypes = [vp, vp, vp, vp, vp, vp]
    L.kde_last_error.restype = ctypes.c_char_p
    L.kde_last_error.argtypes = []
    L.kde_set_timing.argtypes = [vp, ctypes.c_int]
    L.kde_get_timing.argtypes = [vp, P(kde_timing)]
    L.kde_snap.argtypes = [vp, vp, vp, vp, ctypes.c_int64, vp, vp, vp]
    L.kde_dp.argtypes = [vp, vp, vp, ctypes.c_int64, ctypes.c_double, vp, ctypes.c_int32, vp,
                         P(ctypes.c_int64), P(ctypes.c_int64)]
    L.kde_ipc_export.argtypes = [vp, vp, P(ctypes.c_int64)]
    L.kde_ipc_open.argtypes = [vp, ctypes.c_int32, P(vp)]
    L.kde_ipc_close.argtypes = [vp, ctypes.c_int32]
    L.kde_free.argtypes = [vp]
    L.kde_free.restype = None
    for f in ("kde_create", "kde_load_points", "kde_eval", "kde_get_stats", "kde_get_bins",
              "kde_set_timing", "kde_get_timing", "kde_snap", "kde_dp", "kde_ipc_export", "kde_ipc_open",
              "kde_ipc_close"):
        getattr(L, f).restype = ctypes.c_int
    return L


_L = _load()


def _check(rc):
    if rc != KDE_OK:
        raise KdeError(rc, _L.kde_last_error().decode(errors="replace"))


def kde_last_error() -> str:
    return _L.kde_last_error().decode(errors="replace")


def _ptr(a):
    """(pointer, device?) of a contiguous torch tensor or numpy array."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return a.data_ptr()


# ctx handle -> (band rows, raster rows H, width, device): the sizes the C calls write into
# caller buffers, so the binding can check them (the ABI takes plain pointers)
_SHAPES: dict = {}


def kde_create(params: kde_params) -> int:
    h = ctypes.c_void_p()
    _check(_L.kde_create(ctypes.byref(params), ctypes.byref(h)))
    rb, re = int(params.row_begin), int(params.row_end)
    if rb == 0 and re == 0:
        re = int(params.height)
    _SHAPES[h.value] = (re - rb, int(params.height), int(params.width), int(params.device))
    return h.value


def _check_out(ctx, t, numel, what, dtypes=("torch.float32",)):
    if str(t.dtype) not in dtypes or not getattr(t, "is_cuda", False):
        raise TypeError(f"{what} must be a CUDA tensor of dtype {' or '.join(dtypes)}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    shp = _SHAPES.get(ctx)
    if shp is not None and t.device.index != shp[3]:
        raise ValueError(f"{what} is on cuda:{t.device.index}, the context on cuda:{shp[3]}")
    if t.numel() < numel:
        raise ValueError(f"{what} holds {t.numel()} elements, needs {numel}")


def kde_load_points(ctx: int, x, y) -> None:
    """x, y: float64 torch tensors (host or on the context's device) or numpy arrays."""
    n = int(x.shape[0])
    if int(y.shape[0]) != n:
        raise ValueError("x and y lengths differ")
    for a in (x, y):
        dt = a.dtype
        if (isinstance(a, np.ndarray) and dt != np.float64) or (not isinstance(a, np.ndarray)
                                                                and str(dt) != "torch.float64"):
            raise TypeError("coordinates must be float64")
    _check(_L.kde_load_points(ctx, _ptr(x) if n else None, _ptr(y) if n else None, n))


def kde_eval(ctx: int, path: int, out, stream: int | None = None) -> None:
    """out: float32 CUDA tensor of band_rows*W; stream: raw cudaStream_t handle."""
    shp = _SHAPES.get(ctx)
    _check_out(ctx, out, shp[0] * shp[2] if shp else 0, "out")
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(out.device).cuda_stream
    _check(_L.kde_eval(ctx, int(path), _ptr(out), stream))


def kde_eval_ptr(ctx: int, path: int, out_ptr: int, stream: int) -> None:
    """kde_eval into a raw device pointer (e.g. a peer's raster mapped with kde_ipc_open, at
    the band's first row): the caller guarantees (row_end-row_begin)*W fp32 behind it."""
    _check(_L.kde_eval(ctx, int(path), ctypes.c_void_p(out_ptr), stream))


def kde_snap(ctx: int, x, y, label, out, counts=None, stream: int | None = None) -> None:
    """The paper's snapped pipeline (include/kde.h kde_snap).  x, y: float64, label: int32
    or None (torch tensors on the context's device, or host tensors / numpy arrays);
    out: float32 CUDA tensor of H*W; counts: None or an int32/uint32 CUDA tensor of H*W."""
    n = int(x.shape[0])
    if int(y.shape[0]) != n or (label is not None and int(label.shape[0]) != n):
        raise ValueError("x, y and label lengths differ")
    shp = _SHAPES.get(ctx)
    npx = shp[0] * shp[2] if shp else 0  # (a banded context is rejected by the C call itself)
    _check_out(ctx, out, npx, "out")
    if counts is not None:
        _check_out(ctx, counts, npx, "counts", ("torch.int32", "torch.uint32"))
    if label is not None and str(label.dtype) not in ("int32", "torch.int32"):
        raise TypeError("labels must be int32")
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(out.device).cuda_stream
    _check(_L.kde_snap(ctx, _ptr(x) if n else None, _ptr(y) if n else None,
                       _ptr(label) if (label is not None and n) else None, n,
                       _ptr(counts) if counts is not None else None, _ptr(out), stream))


def kde_dp(x, y, traj_offsets, eps: float, keep=None, device: int = 0, stream: int | None = None):
    """GPU Douglas-Peucker (include/kde.h kde_dp).  x, y float64 and traj_offsets int64:
    CUDA tensors on `device` (keep: a uint8 CUDA tensor, allocated if None) or host
    arrays/tensors (keep: a host uint8 array).  Returns (keep, n_kept, rounds)."""
    n = int(x.shape[0])
    ntraj = int(traj_offsets.shape[0]) - 1
    dev = not isinstance(x, np.ndarray) and x.is_cuda
    # the C call reads n from traj_offsets[ntraj]: check the offsets against the buffers
    # (a mismatch would index x, y, keep out of bounds)
    if ntraj < 0:
        raise ValueError("traj_offsets must hold at least one entry")
    offs = traj_offsets.cpu().numpy() if hasattr(traj_offsets, "cpu") else np.asarray(traj_offsets)
    if str(offs.dtype) != "int64":
        raise TypeError("traj_offsets must be int64")
    if offs[0] != 0 or np.any(np.diff(offs) < 0) or int(offs[-1]) != n or int(y.shape[0]) != n:
        raise ValueError("traj_offsets must start at 0, be nondecreasing and end at len(x) == len(y)")
    if keep is not None and int(keep.shape[0]) < n:
        raise ValueError("keep is shorter than x")
    for a in (y, traj_offsets) + ((keep,) if keep is not None else ()):
        adev = not isinstance(a, np.ndarray) and a.is_cuda
        if adev != dev or (dev and a.device != x.device):
            raise ValueError("x, y, traj_offsets and keep must all be on the same device (or host)")
    if keep is None:
        if dev:
            import torch
            keep = torch.empty(n, dtype=torch.uint8, device=x.device)
        else:
            keep = np.zeros(n, np.uint8)
    if stream is None and dev:
        import torch
        stream = torch.cuda.current_stream(x.device).cuda_stream
    nk, rounds = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(_L.kde_dp(_ptr(x) if n else None, _ptr(y) if n else None, _ptr(traj_offsets), ntraj,
                     float(eps), _ptr(keep) if n else None, int(device), stream,
                     ctypes.byref(nk), ctypes.byref(rounds)))
    return keep, nk.value, rounds.value


def kde_get_stats(ctx: int) -> dict:
    s = kde_stats()
    _check(_L.kde_get_stats(ctx, ctypes.byref(s)))
    return s.as_dict()


def kde_get_bins(ctx: int) -> dict:
    st = kde_get_stats(ctx)
    nb = st["nbx"] * st["nby"]
    m = st["n_binned"]
    off = np.zeros(nb + 1, np.int64)
    perm = np.zeros(max(m, 1), np.int64)
    lx = np.zeros(max(m, 1), np.float32)
    ly = np.zeros(max(m, 1), np.float32)
    rng = np.zeros((max(m, 1), 4), np.int32)
    _check(_L.kde_get_bins(ctx, off.ctypes.data, perm.ctypes.data, lx.ctypes.data,
                           ly.ctypes.data, rng.ctypes.data))
    return dict(offsets=off, perm=perm[:m], lx=lx[:m], ly=ly[:m], ranges=rng[:m], stats=st)


def kde_set_timing(ctx: int, enable: bool) -> None:
    _check(_L.kde_set_timing(ctx, 1 if enable else 0))


def kde_get_timing(ctx: int) -> dict:
    t = kde_timing()
    _check(_L.kde_get_timing(ctx, ctypes.byref(t)))
    return {f: float(getattr(t, f)) for f, _ in t._fields_}


def kde_ipc_export(dev_ptr: int):
    """(64-byte handle, byte offset) of the device allocation holding dev_ptr."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _check(_L.kde_ipc_export(ctypes.c_void_p(dev_ptr), h, ctypes.byref(off)))
    return h.raw, off.value


def kde_ipc_open(handle: bytes, device: int) -> int:
    """Map another process's exported allocation; returns its base device pointer."""
    if len(handle) != 64:
        raise ValueError("an IPC handle is 64 bytes")
    p = ctypes.c_void_p()
    _check(_L.kde_ipc_open(ctypes.create_string_buffer(handle, 64), int(device), ctypes.byref(p)))
    return p.value


def kde_ipc_close(dev_ptr: int, device: int) -> None:
    _check(_L.kde_ipc_close(ctypes.c_void_p(dev_ptr), int(device)))


def kde_free(ctx: int | None) -> None:
    if ctx:
        _SHAPES.pop(ctx, None)
        _L.kde_free(ctx)
