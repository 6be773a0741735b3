"""Thin ctypes binding of libfde.so (include/fde.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module
only converts arguments. There is no CPU fallback: if the shared library is
missing, importing this module raises.

Vectors may be CUDA float64 torch tensors (device pointers, asynchronous on
the handle's stream) or C-contiguous float64 numpy arrays (host pointers,
staged by the library; the call synchronises).
"""
from __future__ import annotations

import ctypes
import os
import sys
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDE_LIB") or os.path.join(_HERE, "libfde.so")

FDE_OK = 0
FDE_ERR_INVALID_ARG = 1
FDE_ERR_UNSUPPORTED = 2
FDE_ERR_OUT_OF_MEMORY = 3
FDE_ERR_CUDA = 4
FDE_ERR_SINGULAR = 5
FDE_ERR_NOT_SPD = 6
FDE_ERR_BREAKDOWN = 7
FDE_ERR_NONFINITE = 8
FDE_ERR_NOT_CONVERGED = 9

FDE_PREC_NONE, FDE_PREC_TAU, FDE_PREC_TAU_D, FDE_PREC_TAU_DSYM, FDE_PREC_TILDE, FDE_PREC_TRI = 0, 1, 2, 3, 4, 5


class fde_desc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("dims", ctypes.c_int32), ("batch", ctypes.c_int32), ("stencil", ctypes.c_int32),
        ("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("nu", ctypes.c_double),
        ("dp", ctypes.c_double), ("dm", ctypes.c_double), ("ep", ctypes.c_double), ("em", ctypes.c_double),
        ("dp_field", ctypes.c_void_p), ("dm_field", ctypes.c_void_p),
        ("ep_field", ctypes.c_void_p), ("em_field", ctypes.c_void_p),
        ("prec", ctypes.c_int32),
        ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("ywt", ctypes.c_double),
        ("stream", ctypes.c_void_p),
    ]


class fde_stats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("restarts", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("status", ctypes.c_int32), ("rel_res", ctypes.c_double)]


if not os.path.exists(LIB_PATH):
    raise ImportError("libfde.so not built at %s — run `python __graft_entry__.py build` "
                      "(there is no CPU fallback)" % LIB_PATH)

lib = ctypes.CDLL(LIB_PATH)
_H = ctypes.c_void_p
_P = ctypes.c_void_p
lib.fde_create.argtypes = [ctypes.POINTER(fde_desc), ctypes.POINTER(_H)]
lib.fde_create.restype = ctypes.c_int
lib.fde_destroy.argtypes = [_H]
lib.fde_destroy.restype = None
lib.fde_matvec.argtypes = [_H, _P, _P]
lib.fde_matvec.restype = ctypes.c_int
lib.fde_tau_apply.argtypes = [_H, _P, _P]
lib.fde_tau_apply.restype = ctypes.c_int
lib.fde_pcg.argtypes = [_H, _P, _P, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(fde_stats)]
lib.fde_pcg.restype = ctypes.c_int
lib.fde_gmres.argtypes = [_H, _P, _P, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                          ctypes.POINTER(fde_stats)]
lib.fde_gmres.restype = ctypes.c_int
lib.fde_status_str.argtypes = [ctypes.c_int]
lib.fde_status_str.restype = ctypes.c_char_p
lib.fde_last_error.argtypes = [_H]
lib.fde_last_error.restype = ctypes.c_char_p
lib.fde_kernel_launches.argtypes = [_H]
lib.fde_kernel_launches.restype = ctypes.c_int64
lib.fde_profile_unit.argtypes = [_H, _P, _P, _P, ctypes.c_int32, _P, ctypes.c_int64, ctypes.c_int32,
                                 ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_char_p)]
lib.fde_profile_unit.restype = ctypes.c_int
lib.fde_profile_solve.argtypes = [_H, _P, _P, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                  ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(fde_stats)]
lib.fde_profile_solve.restype = ctypes.c_int
lib.fde_measure_fp64_peak.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]
lib.fde_measure_fp64_peak.restype = ctypes.c_int


def measure_fp64_peak(reps: int = 5) -> float:
    """fde_measure_fp64_peak: DFMA throughput of the current device, TFLOP/s."""
    v = ctypes.c_double(0.0)
    st = lib.fde_measure_fp64_peak(int(reps), ctypes.byref(v))
    if st != FDE_OK:
        raise FdeError(st, "fde_measure_fp64_peak")
    return v.value


def fde_status_str(s: int) -> str:
    return lib.fde_status_str(int(s)).decode()


class FdeError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__("%s: %s" % (fde_status_str(status), msg))
        self.status = status


def _ptr(a, numel: Optional[int] = None, device: Optional[int] = None) -> int:
    """Raw pointer of a float64 C-contiguous torch tensor or numpy array.
    With `numel`, the array must hold exactly that many elements (the library
    reads/writes batch·N values behind the pointer); with `device`, a CUDA
    tensor must live on that device (the handle's)."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
            raise TypeError("numpy arrays must be C-contiguous float64")
        if numel is not None and a.size != numel:
            raise ValueError("array has %d elements, the handle needs batch*N = %d" % (a.size, numel))
        return a.ctypes.data
    # torch tensor (imported lazily: torch is plumbing, not a dependency of the binding)
    if getattr(a, "dtype", None) is None or str(a.dtype) != "torch.float64":
        raise TypeError("tensors must be float64")
    if not a.is_contiguous():
        raise TypeError("tensors must be contiguous")
    if numel is not None and a.numel() != numel:
        raise ValueError("tensor has %d elements, the handle needs batch*N = %d" % (a.numel(), numel))
    if device is not None and a.is_cuda and a.device.index != device:
        raise ValueError("tensor is on cuda:%d, the handle on cuda:%d" % (a.device.index, device))
    return a.data_ptr()


def _field(v, N: int):
    """A coefficient field (length N, copied by fde_create)."""
    if v is None:
        return None, None
    if isinstance(v, np.ndarray):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return v, _ptr(v, N)
    return v, _ptr(v, N)


class Fde:
    """Handle over fde_create/... with the ABI's names (fde_matvec -> matvec, ...)."""

    def __init__(self, n: int, dims: int, alpha: float, beta: float = 1.5, nu: float = 0.0,
                 dp: float = 1.0, dm: float = 1.0, ep: float = 1.0, em: float = 1.0,
                 dp_field=None, dm_field=None, ep_field=None, em_field=None,
                 prec: int = FDE_PREC_TAU, cx: float = 1.0, cy: float = 1.0, ywt: float = 1.0,
                 batch: int = 1, stencil: int = 1, stream: Optional[int] = None):
        d = fde_desc()
        d.n, d.dims, d.batch, d.stencil = n, dims, batch, stencil
        d.alpha, d.beta, d.nu = alpha, beta, nu
        d.dp, d.dm, d.ep, d.em = dp, dm, ep, em
        keep = []
        for name, v in (("dp_field", dp_field), ("dm_field", dm_field), ("ep_field", ep_field), ("em_field", em_field)):
            obj, p = _field(v, n ** dims)
            keep.append(obj)
            setattr(d, name, p)
        d.prec, d.cx, d.cy, d.ywt = prec, cx, cy, ywt
        d.stream = stream
        self.desc = d
        self.n, self.dims, self.batch = n, dims, batch
        self.N = n ** dims
        self.numel = batch * self.N
        # the library creates the handle on the calling thread's current device
        self.device = None
        torch = sys.modules.get("torch")
        if torch is not None and torch.cuda.is_available():
            self.device = torch.cuda.current_device()
        self._h = _H()
        st = lib.fde_create(ctypes.byref(d), ctypes.byref(self._h))
        if st != FDE_OK:
            raise FdeError(st, "fde_create")

    @classmethod
    def from_problem(cls, p, stream: Optional[int] = None):
        """Build from a workloads.Problem (seeded synthetic config)."""
        return cls(p.n, p.dims, p.alpha, p.beta if p.dims == 2 else 1.5, p.nu, p.dp, p.dm, p.ep, p.em,
                   p.dp_field, p.dm_field, p.ep_field, p.em_field, p.prec, p.cx, p.cy, 1.0,
                   p.batch, p.stencil, stream)

    def _v(self, a) -> int:
        """Pointer of a length batch·N vector argument (size and device checked)."""
        return _ptr(a, self.numel, self.device)

    def _check(self, st):
        if st != FDE_OK and st != FDE_ERR_NOT_CONVERGED:
            raise FdeError(st, lib.fde_last_error(self._h).decode())
        return st

    def matvec(self, x, y):
        return self._check(lib.fde_matvec(self._h, self._v(x), self._v(y)))

    def tau_apply(self, r, z):
        return self._check(lib.fde_tau_apply(self._h, self._v(r), self._v(z)))

    def pcg(self, b, x, rtol: float = 1e-10, maxit: int = 5000):
        stats = (fde_stats * self.batch)()
        st = self._check(lib.fde_pcg(self._h, self._v(b), self._v(x), rtol, maxit, stats))
        return st, [dict(iters=s.iters, restarts=s.restarts, converged=bool(s.converged), status=s.status,
                         rel_res=s.rel_res) for s in stats]

    def gmres(self, b, x, rtol: float = 1e-10, restart: int = 30, maxit: int = 20000, left: bool = False):
        stats = (fde_stats * self.batch)()
        st = self._check(lib.fde_gmres(self._h, self._v(b), self._v(x), rtol, restart, maxit, int(left), stats))
        return st, [dict(iters=s.iters, restarts=s.restarts, converged=bool(s.converged), status=s.status,
                         rel_res=s.rel_res) for s in stats]

    def kernel_launches(self) -> int:
        return int(lib.fde_kernel_launches(self._h))

    def profile_unit(self, x, y, z, reps: int = 20, flush=None):
        """fde_profile_unit: per-kernel mean device µs of one unit
        (matvec x->y + τ-solve x->z), each launch after an L2 flush of the
        device buffer `flush` (a uint8 CUDA tensor) if given. Returns
        [(name, µs), ...] in launch order."""
        MAXK = 16
        us = (ctypes.c_double * MAXK)()
        names = (ctypes.c_char_p * MAXK)()
        cnt = ctypes.c_int32(0)
        fp = 0 if flush is None else flush.data_ptr()
        fb = 0 if flush is None else flush.numel() * flush.element_size()
        self._check(lib.fde_profile_unit(self._h, self._v(x), self._v(y), self._v(z), reps, fp or None, fb, MAXK,
                                         ctypes.byref(cnt), us, names))
        return [(names[i].decode(), us[i]) for i in range(min(cnt.value, MAXK))]

    def profile_solve(self, b, x, solver: str = "pcg", rtol: float = 1e-10, maxit: int = 5000, restart: int = 30):
        """fde_profile_solve: one solve whose loop body carries CUDA events;
        returns ([(name, µs of the last loop body)], stats)."""
        MAXK = 256
        us = (ctypes.c_double * MAXK)()
        names = (ctypes.c_char_p * MAXK)()
        cnt = ctypes.c_int32(0)
        stats = (fde_stats * self.batch)()
        self._check(lib.fde_profile_solve(self._h, self._v(b), self._v(x), rtol, maxit, 0 if solver == "pcg" else 1,
                                          restart, MAXK, ctypes.byref(cnt), us, names, stats))
        return ([(names[i].decode(), us[i]) for i in range(min(cnt.value, MAXK))],
                [dict(iters=s.iters, converged=bool(s.converged)) for s in stats])

    def close(self):
        if self._h:
            lib.fde_destroy(self._h)
            self._h = _H()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
