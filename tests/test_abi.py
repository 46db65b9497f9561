"""Host-side checks of the C-ABI boundary (no GPU needed).

libkde.so must load and export every symbol include/kde.h declares; argument
validation that needs no device must answer EINVAL; with no device at all the
library must fail loudly (ECUDA), never fall back to the CPU.
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "kde.h")).read()
    return re.findall(r"KDE_API\s+[\w\s\*]+?\b(kde_\w+)\s*\(", src)


def test_header_declares_the_boundary():
    names = set(_declared())
    assert {"kde_create", "kde_load_points", "kde_eval", "kde_free", "kde_get_stats",
            "kde_last_error", "kde_get_bins"} <= names


def test_library_exports_every_declared_symbol():
    from paper_2004_13653_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_lib.EXPORTS) == set(_declared())


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirrors == the C compiler's layout of include/kde.h (sizes and offsets)."""
    import subprocess
    from paper_2004_13653_b200 import _lib
    fields = {"kde_params": _lib.kde_params, "kde_stats": _lib.kde_stats, "kde_timing": _lib.kde_timing}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "kde.h"', "int main(void){"]
    for st, cls in fields.items():
        lines.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.split("\n") if l)
    for st, cls in fields.items():
        assert int(out[st]) == ctypes.sizeof(cls), st
        for f, _ in cls._fields_:
            assert int(out[f"{st}.{f}"]) == getattr(cls, f).offset, (st, f)


def test_enum_values_match_header(tmp_path):
    """The binding's constants == the header's enums (compiled with gcc)."""
    import subprocess
    from paper_2004_13653_b200 import _lib
    names = ["KDE_PATH_DIRECT", "KDE_PATH_TENSOR", "KDE_PATH_TENSOR_SPLIT", "KDE_RADIAL", "KDE_OK",
             "KDE_EINVAL", "KDE_ENOMEM", "KDE_ECUDA", "KDE_EUNSUPPORTED", "KDE_ESTATE",
             "KDE_UNIFORM", "KDE_GAUSSIAN", "KDE_COSINE"]
    lines = ['#include <stdio.h>', '#include "kde.h"', "int main(void){"]
    lines += [f'printf("{n} %d\\n", (int){n});' for n in names] + ["return 0;}"]
    src = tmp_path / "enums.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "enums"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.split("\n") if l)
    for n in names:
        assert int(out[n]) == getattr(_lib, n), n


def _params(**kw):
    from paper_2004_13653_b200 import _lib
    p = dict(x0=0.0, y0=0.0, res=1.0, width=64, height=64, h=2.0, kernel=6, cutoff=4.0,
             row_begin=0, row_end=0, device=0)
    p.update(kw)
    return _lib.kde_params(**p)


@pytest.mark.parametrize("bad", [dict(res=0.0), dict(res=float("nan")), dict(h=-1.0),
                                 dict(cutoff=float("inf")), dict(width=0), dict(height=40000),
                                 dict(kernel=8), dict(kernel=0x200 | 6), dict(row_begin=5, row_end=5),
                                 dict(row_begin=0, row_end=65), dict(x0=float("nan"))])
def test_create_rejects_bad_params(bad):
    from paper_2004_13653_b200 import _lib
    with pytest.raises(_lib.KdeError) as e:
        _lib.kde_create(_params(**bad))
    assert e.value.code == _lib.KDE_EINVAL
    assert _lib.kde_last_error()


def test_null_arguments_are_einval():
    from paper_2004_13653_b200 import _lib
    L = _lib._L
    assert L.kde_create(None, None) == _lib.KDE_EINVAL
    assert L.kde_load_points(None, None, None, 0) == _lib.KDE_EINVAL
    assert L.kde_eval(None, 0, None, None) == _lib.KDE_EINVAL
    assert L.kde_get_stats(None, None) == _lib.KDE_EINVAL
    assert L.kde_get_bins(None, None, None, None, None, None) == _lib.KDE_EINVAL
    assert L.kde_snap(None, None, None, None, 0, None, None, None) == _lib.KDE_EINVAL
    assert L.kde_dp(None, None, None, 0, 1.0, None, 0, None, None, None) == _lib.KDE_EINVAL
    assert L.kde_dp(None, None, None, -1, 1.0, None, 0, None, None, None) == _lib.KDE_EINVAL
    L.kde_free(None)  # NULL-safe


def test_no_device_fails_loudly_without_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2004_13653_b200 import _lib
    with pytest.raises(_lib.KdeError) as e:
        _lib.kde_create(_params())
    assert e.value.code == _lib.KDE_ECUDA
    x = np.linspace(0.0, 1.0, 8)
    with pytest.raises(_lib.KdeError) as e:  # the GPU Douglas-Peucker has no CPU fallback either
        _lib.kde_dp(x, x, np.array([0, 8], np.int64), 0.1)
    assert e.value.code == _lib.KDE_ECUDA
