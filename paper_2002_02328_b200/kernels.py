"""Drop-in for the reference's backend switch ``bd3mg.kernels``
(pkg/src/bd3mg/kernels.py:14-32).

The reference binds ``depthvar_correlate[_adjoint]`` from its Cython core or
a SciPy fallback at import time.  Here there is exactly one backend: the
sm_100a library, called through its host-buffer C entry points
(``bd3mg_depthvar_correlate[_adjoint]_host_f64``) with the Cython
functions' contract -- C-contiguous float64 fragment (nzf, ny, nx) and
kernel stack (nz, kz, ky, kx), global depth coordinates, a new
(out_hi-out_lo+1, ny, nx) float64 result.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

USING_COMPILED = True


def backend_name() -> str:
    return "cuda-sm100a"


def _buffer(a, ndim: int, what: str) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.float64:
        raise ValueError(f"Buffer dtype mismatch for {what}: expected 'double' but got '{a.dtype}'")
    if a.ndim != ndim:
        raise ValueError(f"Buffer has wrong number of dimensions for {what} (expected {ndim}, got {a.ndim})")
    if not a.flags.c_contiguous:
        raise ValueError(f"{what} is not C-contiguous")
    return a


def _call(fn, frag, kernels, frag_z0, out_lo, out_hi):
    frag = _buffer(frag, 3, "frag")
    kernels = _buffer(kernels, 4, "kernels")
    nzf, ny, nx = frag.shape
    nzk, kz, ky, kx = kernels.shape
    nout = out_hi - out_lo + 1
    if nout < 0:
        raise ValueError("negative dimensions are not allowed")
    out = np.empty((nout, ny, nx))
    if nout == 0:
        return out
    N.check(fn(frag.ctypes.data, nzf, ny, nx, kernels.ctypes.data, nzk, kz, ky, kx,
               int(frag_z0), int(out_lo), int(out_hi), out.ctypes.data))
    return out


def depthvar_correlate(frag, kernels, frag_z0, out_lo, out_hi) -> np.ndarray:
    """H rows (reference _core.pyx:17-53)."""
    return _call(N.lib.bd3mg_depthvar_correlate_host_f64, frag, kernels, frag_z0, out_lo, out_hi)


def depthvar_correlate_adjoint(frag, kernels, frag_z0, out_lo, out_hi) -> np.ndarray:
    """H^T rows (reference _core.pyx:56-96)."""
    return _call(N.lib.bd3mg_depthvar_correlate_adjoint_host_f64, frag, kernels, frag_z0, out_lo, out_hi)
