"""ctypes binding of libbd3mg_b200.so for the reference package.

This is the file a maintainer drops into the reference as
``pkg/src/bd3mg/_b200.py``.  With the two-line
switch in ``bd3mg/kernels.py`` (``BD3MG_B200=1``) every caller of the native
core -- blur.apply_H/Ht[_rows], objective._grad_rows, MajorantOperator.apply,
eval_f, rho_hth_estimate -- runs on the B200 unchanged.

Contract (reference src/_core.pyx:17-18, :56-57): ``fn(frag, kernels,
frag_z0, out_lo, out_hi)`` with ``frag`` a C-contiguous writable float64
(nzf, ny, nx) buffer, ``kernels`` a C-contiguous writable float64
(nz, kz, ky, kx) buffer; returns a new float64 (out_hi-out_lo+1, ny, nx)
array.  Buffer errors are raised exactly as the Cython typed memoryviews
raise them (same exception type, same message, same check order: buffer
acquisition -- contiguity, writability -- then rank, then dtype; fragment
before kernels).  Row ranges the reference leaves undefined
(``boundscheck=False`` reads out of bounds) are a ValueError here.
The foreign call releases the GIL (ctypes), as the Cython loops do.
"""

import ctypes
import os

import numpy as np

_lib = ctypes.CDLL(os.environ.get("BD3MG_B200_LIB", "libbd3mg_b200.so"))
_i64, _vp = ctypes.c_int64, ctypes.c_void_p
for _name in ("bd3mg_depthvar_correlate_host_f64", "bd3mg_depthvar_correlate_adjoint_host_f64"):
    getattr(_lib, _name).argtypes = [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64,
                                     _i64, _i64, _i64, _vp]
    getattr(_lib, _name).restype = ctypes.c_int
_lib.bd3mg_last_error.restype = ctypes.c_char_p

# struct-module format codes -> the C type names Cython reports
_CNAMES = {"b": "signed char", "B": "unsigned char", "h": "short", "H": "unsigned short", "i": "int",
           "I": "unsigned int", "l": "long", "L": "unsigned long", "q": "long long",
           "Q": "unsigned long long", "f": "float", "g": "long double", "?": "bool",
           "Zf": "complex float", "Zd": "complex double", "Zg": "complex long double"}


def _buffer(a, ndim):
    """A double[:, ..., ::1] memoryview acquisition, Cython's way."""
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("ndarray is not C-contiguous")
        if not a.flags.writeable:
            raise ValueError("buffer source array is read-only")
    try:
        m = memoryview(a)
    except TypeError:
        raise TypeError(f"a bytes-like object is required, not '{type(a).__name__}'") from None
    if m.readonly:
        raise BufferError("Object is not writable.")
    if not m.c_contiguous:
        raise ValueError("ndarray is not C-contiguous")
    if m.ndim != ndim:
        raise ValueError(f"Buffer has wrong number of dimensions (expected {ndim}, got {m.ndim})")
    fmt = m.format
    if fmt[:1] in (">", "!"):
        raise ValueError("Big-endian buffer not supported on little-endian compiler")
    fmt = fmt.lstrip("<=@")
    if fmt != "d":
        name = _CNAMES.get(fmt)
        if name is None:
            raise ValueError(f"Does not understand character buffer dtype format string ('{fmt}')")
        raise ValueError(f"Buffer dtype mismatch, expected 'double' but got '{name}'")
    return np.asarray(a)


def _call(fn, frag, kernels, frag_z0, out_lo, out_hi):
    frag = _buffer(frag, 3)
    kernels = _buffer(kernels, 4)
    nzf, ny, nx = frag.shape
    nzk, kz, ky, kx = kernels.shape
    out = np.zeros((out_hi - out_lo + 1, ny, nx))  # negative extent: numpy's ValueError, as in _core.pyx:28
    if out.shape[0] == 0:
        return out
    rc = fn(frag.ctypes.data, nzf, ny, nx, kernels.ctypes.data, nzk, kz, ky, kx,
            frag_z0, out_lo, out_hi, out.ctypes.data)
    if rc:
        raise ValueError(_lib.bd3mg_last_error().decode())
    return out


def depthvar_correlate(frag, kernels, frag_z0, out_lo, out_hi):
    return _call(_lib.bd3mg_depthvar_correlate_host_f64, frag, kernels, frag_z0, out_lo, out_hi)


def depthvar_correlate_adjoint(frag, kernels, frag_z0, out_lo, out_hi):
    return _call(_lib.bd3mg_depthvar_correlate_adjoint_host_f64, frag, kernels, frag_z0, out_lo, out_hi)
