"""B200-native gridded KDE of arxiv 2004.13653's trajectory-visualisation hot path.

The product is ``libkde.so`` (C ABI in ``include/kde.h``, sm_100a CUDA in
``csrc/``); this package is its thin Python face:

* ``kde_create / kde_load_points / kde_eval / kde_get_stats / kde_get_bins /
  kde_last_error / kde_free`` -- the C calls with the same names (``_lib.py``);
* ``KDE`` -- a small owner object over one context;
* ``dist`` -- row-band sharding over ``torch.distributed`` ranks.

PyTorch is used only for device memory, streams and process groups.
"""
from __future__ import annotations

from . import _lib
from ._lib import (KDE_COSINE, KDE_EPANECHNIKOV, KDE_GAUSSIAN, KDE_PATH_DIRECT,
                   KDE_PATH_TENSOR, KDE_PATH_TENSOR_SPLIT, KDE_QUARTIC, KDE_RADIAL, KDE_TRIANGULAR, KDE_TRICUBE,
                   KDE_TRIWEIGHT, KDE_UNIFORM, KERNEL_NAMES, KdeError, kde_create, kde_eval,
                   kde_free, kde_get_bins, kde_get_stats, kde_get_timing, kde_last_error,
                   kde_load_points, kde_params, kde_set_timing, kde_snap, kde_dp,
                   kde_eval_ptr, kde_ipc_close, kde_ipc_export, kde_ipc_open)

__all__ = ["KDE", "KdeError", "kde_params", "kde_create", "kde_load_points", "kde_eval",
           "kde_get_stats", "kde_get_bins", "kde_set_timing", "kde_get_timing", "kde_snap", "kde_dp", "kde_last_error",
           "kde_free", "kde_eval_ptr", "kde_ipc_export", "kde_ipc_open", "kde_ipc_close", "KERNEL_NAMES",
           "KDE_PATH_DIRECT", "KDE_PATH_TENSOR", "KDE_PATH_TENSOR_SPLIT", "KDE_RADIAL", "kernel_id"]


_PATHS = {"direct": KDE_PATH_DIRECT, "tensor": KDE_PATH_TENSOR, "tensor_split": KDE_PATH_TENSOR_SPLIT}


def kernel_id(name: str, radial: bool = False) -> int:
    return KERNEL_NAMES.index(name) | (KDE_RADIAL if radial else 0)


class KDE:
    """One libkde context: grid + kernel fixed at construction, points replaceable.

    ``KDE(x0, y0, res, W, H, h, kernel="gaussian", cutoff=4.0, radial=False,
    rows=None, device=0)``; ``load(x, y)`` bins (host or device float64 tensors);
    ``eval(path="direct"|"tensor"|"tensor_split", out=None)`` returns the (rows, W) float32 raster.
    """

    def __init__(self, x0, y0, res, width, height, h, kernel="gaussian", cutoff=4.0,
                 radial=False, rows=None, device=0):
        kid = kernel if isinstance(kernel, int) else kernel_id(kernel, radial)
        rb, re = (0, 0) if rows is None else rows
        self.params = kde_params(float(x0), float(y0), float(res), int(width), int(height),
                                 float(h), int(kid), float(cutoff), int(rb), int(re), int(device))
        self.rows = (0, int(height)) if rows is None else (int(rb), int(re))
        self.width = int(width)
        self.device = int(device)
        self.ctx = kde_create(self.params)

    def load(self, x, y):
        kde_load_points(self.ctx, x, y)
        return self

    def snap(self, x, y, label=None, out=None, counts=None, stream=None):
        """The paper's own pipeline (Eqs. 5-6 projection, Alg. 3 density matrix with
        Eqs. 12-13 interpolation, Eq. 7 convolution): returns the (H, W) Eq. 7 matrix."""
        import torch
        if out is None:
            out = torch.empty((self.rows[1] - self.rows[0], self.width), dtype=torch.float32,
                              device=torch.device("cuda", self.device))
        kde_snap(self.ctx, x, y, label, out, counts, stream)
        return out

    def eval(self, path="direct", out=None, stream=None):
        import torch
        p = _PATHS[path] if isinstance(path, str) else int(path)
        nr = self.rows[1] - self.rows[0]
        if out is None:
            out = torch.empty((nr, self.width), dtype=torch.float32,
                              device=torch.device("cuda", self.device))
        kde_eval(self.ctx, p, out, stream)
        return out

    def stats(self):
        return kde_get_stats(self.ctx)

    def bins(self):
        return kde_get_bins(self.ctx)

    def set_timing(self, enable=True):
        kde_set_timing(self.ctx, enable)

    def timing(self):
        return kde_get_timing(self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            kde_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
