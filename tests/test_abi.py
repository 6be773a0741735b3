"""CPU tests of the boundary: the C-ABI library loads, exports every symbol
include/fde.h declares, and its host-side validation answers without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "fde.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fde_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for n in ("fde_create", "fde_destroy", "fde_matvec", "fde_tau_apply", "fde_pcg", "fde_gmres",
              "fde_status_str", "fde_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1912_13304_b200 import fde
    for name in _declared_functions():
        assert hasattr(fde.lib, name), name


def test_status_strings():
    from paper_1912_13304_b200 import fde
    assert fde.fde_status_str(0) == "FDE_OK"
    assert fde.fde_status_str(9) == "FDE_ERR_NOT_CONVERGED"
    assert fde.fde_status_str(1234) == "FDE_ERR_UNKNOWN"


def _create(**kw):
    from paper_1912_13304_b200 import fde
    d = fde.fde_desc()
    base = dict(n=127, dims=1, batch=1, stencil=1, alpha=1.5, beta=1.5, nu=0.1, dp=1.0, dm=1.0, ep=1.0, em=1.0,
                prec=1, cx=1.0, cy=1.0, ywt=1.0)
    base.update(kw)
    for k, v in base.items():
        setattr(d, k, v)
    h = ctypes.c_void_p()
    st = fde.lib.fde_create(ctypes.byref(d), ctypes.byref(h))
    if st == 0:
        fde.lib.fde_destroy(h)
    return st


@pytest.mark.parametrize("kw", [
    dict(alpha=1.0), dict(alpha=2.0), dict(alpha=float("nan")), dict(dims=2, beta=2.5), dict(dims=3),
    dict(n=0), dict(batch=0), dict(batch=9), dict(nu=-1.0), dict(nu=float("inf")), dict(dp=-1.0),
    dict(prec=7), dict(stencil=3), dict(cx=float("nan")), dict(dims=2, prec=4),
])
def test_create_rejects_invalid(kw):
    assert _create(**kw) == 1   # FDE_ERR_INVALID_ARG, decided before any CUDA call


@pytest.mark.parametrize("n", [8191, 5000, 2049, 16383])
def test_create_unsupported_sizes(n):
    # FDE_ERR_UNSUPPORTED: n+1 not a power of two in [32, 4096] (FFT path) and
    # n > 2048 (direct path); decided before any CUDA call
    assert _create(n=n) == 2


def test_null_handle_and_args():
    from paper_1912_13304_b200 import fde
    assert fde.lib.fde_create(None, None) == 1
    assert fde.lib.fde_matvec(None, None, None) == 1
    assert fde.lib.fde_tau_apply(None, None, None) == 1
    assert fde.lib.fde_pcg(None, None, None, 1e-10, 10, None) == 1
    assert fde.lib.fde_gmres(None, None, None, 1e-10, 30, 10, 0, None) == 1
    fde.lib.fde_destroy(None)   # NULL-safe
    assert fde.lib.fde_last_error(None) == b"NULL handle"
    assert fde.lib.fde_kernel_launches(None) == 0


def test_binding_rejects_bad_arrays():
    from paper_1912_13304_b200 import fde
    with pytest.raises(TypeError):
        fde._ptr(np.zeros(4, dtype=np.float32))
    with pytest.raises(TypeError):
        fde._ptr(np.zeros((4, 4))[:, 1])
    # the library reads/writes batch·N elements behind every vector pointer:
    # a short (or long) array is refused before any call into libfde
    with pytest.raises(ValueError):
        fde._ptr(np.zeros(10), numel=11)
    with pytest.raises(ValueError):
        fde._ptr(np.zeros((2, 6)), numel=11)
    assert fde._ptr(np.zeros((1, 11)), numel=11) != 0
