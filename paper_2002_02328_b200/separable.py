"""Separable-PSF fast path: H / Hᵀ for kernel stacks
whose every plane is rank one, K[zo] = u_zo ⊗ v_zo ⊗ w_zo.

The BASELINE PSF family (axis-aligned Gaussians, reference blur.py:100-124
with φ = θ = 0) is rank one up to rounding, so the depth-variant
correlation costs kz + ky + kx FMAs per voxel instead of kz·ky·kx and is
memory-bound.  Detection happens once, on the host, when the stack is
factored: the depth / y / x marginals of a unit-sum rank-one kernel are its
factors, so ``u ⊗ v ⊗ w`` reproducing K to ``tol`` decides it.  The result
agrees with the dense kernels to rounding (different summation order); the
dense graded kernels stay the default everywhere, and this path is reported
against HBM bandwidth, never against the FMA roofline.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import device as D
from .blur import PsfStack, _check_dims, _dtype_of


def factor_stack(psf: PsfStack, tol: float = 1e-13):
    """(u, v, w) with K[z] = u[z] ⊗ v[z] ⊗ w[z] to ``tol`` · max|K[z]| for
    every plane, or None if some plane is not rank one."""
    k = psf.kernels
    u = k.sum(axis=(2, 3))  # (nz, kz)
    v = k.sum(axis=(1, 3))  # (nz, ky)
    w = k.sum(axis=(1, 2))  # (nz, kx)
    rec = u[:, :, None, None] * v[:, None, :, None] * w[:, None, None, :]
    err = np.abs(rec - k).reshape(k.shape[0], -1).max(axis=1)
    scale = np.abs(k).reshape(k.shape[0], -1).max(axis=1)
    if np.any(err > tol * scale):
        return None
    return u, v, w


@dataclass
class SeparableStack:
    """Rank-one factors of a PSF stack, uploaded once per (dtype, device)."""

    psf: PsfStack
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    _dev: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    @classmethod
    def from_psf(cls, psf: PsfStack, tol: float = 1e-13) -> "SeparableStack":
        kx, ky, kz = psf.kdims
        if kx != ky or kx not in (3, 5, 7, 9):
            raise ValueError(f"separable path needs kx == ky in (3, 5, 7, 9), got {psf.kdims}")
        f = factor_stack(psf, tol)
        if f is None:
            raise ValueError("PSF stack is not separable (some plane is not rank one)")
        return cls(psf, *f)

    def factors(self, dtype: torch.dtype, device=None):
        dev = torch.device(device) if device is not None else D.default_device()
        key = (dtype, dev.index if dev.index is not None else torch.cuda.current_device())
        t = self._dev.get(key)
        if t is None:
            t = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype) for a in (self.u, self.v, self.w))
            self._dev[key] = t
        return t

    def correlate_rows(self, frag, frag_z0: int, out_lo: int, out_hi: int, adjoint: bool = False, out=None):
        """H (or Hᵀ) rows [out_lo, out_hi] of a fragment whose plane 0 is depth
        frag_z0 — the contract of blur.correlate_rows / _core (zero outside
        the fragment), on device tensors (float64 or float32)."""
        dt = _dtype_of(frag)
        f = D.to_device(frag, dt)
        nzf, ny, nx = f.shape
        kx, ky, kz = self.psf.kdims
        nout = out_hi - out_lo + 1
        if out is None:
            out = torch.empty((max(nout, 0), ny, nx), dtype=dt, device=f.device)
        u, v, w = self.factors(dt, f.device)
        fn = N.lib.bd3mg_sep_correlate_f64 if dt == torch.float64 else N.lib.bd3mg_sep_correlate_f32
        with torch.cuda.device(f.device):
            N.check(fn(f.data_ptr(), nzf, ny, nx, u.data_ptr(), v.data_ptr(), w.data_ptr(), self.psf.dims.nz, kz,
                       ky, kx, frag_z0, out_lo, out_hi, out.data_ptr(), int(adjoint),
                       torch.cuda.current_stream(f.device).cuda_stream))
        return out

    def apply_H(self, x):
        _check_dims(self.psf, x)
        r = self.correlate_rows(x, 0, 0, self.psf.dims.nz - 1)
        return r if D.is_tensor(x) else r.double().cpu().numpy()

    def apply_Ht(self, v):
        _check_dims(self.psf, v)
        r = self.correlate_rows(v, 0, 0, self.psf.dims.nz - 1, adjoint=True)
        return r if D.is_tensor(v) else r.double().cpu().numpy()


def bytes_H(dims, dtype_bytes: int) -> int:
    """Algorithmic HBM bytes of one full separable H: every plane read once
    and written once."""
    return 2 * dims[0] * dims[1] * dims[2] * dtype_bytes
