"""Host-buffer entry points: the GPU as the reference's worker pool.

``HostProblem`` owns a C-ABI problem handle (kernels and observation
uploaded once) and serves the two host-level contracts of the reference:

* ``mg_direction(x_slab, slab_z0, block, d_mem)`` -- a worker step on a
  TaskMessage snapshot, returning the UpdateMessage increment
  (reference runtime.py:92-105, scheduler.py:36-57);
* ``jacobi_sweep(x, dmem, blocks)`` -- one bp3mg barrier cycle over the given
  blocks (runtime.py:244-292) on host arrays, updated in place.

Both go through ``bd3mg_problem_*_host`` (include/bd3mg_b200.h); pass pinned
host memory (``pinned_empty``) for full PCIe bandwidth.  Calls on one handle are
serialised by the library (one stream and buffer set per handle); worker
threads that should overlap each open their own ``HostProblem``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from . import device as D
from .objective import Objective
from .volume import SliceBlock


class _PinnedArray(np.ndarray):
    """ndarray view that keeps its pinned torch allocation alive."""

    _owner = None


def pinned_empty(shape) -> np.ndarray:
    """Page-locked float64 host array (numpy view of a pinned torch tensor)."""
    import torch
    t = torch.empty(tuple(shape), dtype=torch.float64, pin_memory=True)
    arr = t.numpy().view(_PinnedArray)
    arr._owner = t
    return arr


class HostProblem:
    def __init__(self, obj: Objective, dtype: str = "f64", device: int = 0):
        self.obj = obj
        d = obj.dims
        kx, ky, kz = obj.psf.kdims
        self.geom = N.Geom(d.nx, d.ny, d.nz, kx, ky, kz, N.BD3MG_F64 if dtype == "f64" else N.BD3MG_F32)
        self.h = C.c_void_p()
        N.check(N.lib.bd3mg_problem_create(C.byref(self.geom), C.byref(D.reg(obj.params)),
                                           obj.psf.kernels.ctypes.data, obj.y.ctypes.data, device, C.byref(self.h)))

    def close(self) -> None:
        if self.h:
            N.lib.bd3mg_problem_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def mg_direction(self, x_slab: np.ndarray, slab_z0: int, block: SliceBlock, d_mem=None,
                     info: np.ndarray | None = None) -> np.ndarray:
        xs = np.ascontiguousarray(x_slab, dtype=np.float64)
        n = block.count(self.obj.dims)
        dm = None if d_mem is None else np.ascontiguousarray(d_mem, dtype=np.float64).reshape(-1)
        if dm is not None and dm.size != n:
            raise ValueError(f"memory direction has {dm.size} entries, expected {n}")
        inc = np.empty(n)
        N.check(N.lib.bd3mg_problem_mg_direction_host(self.h, xs.ctypes.data, slab_z0, xs.shape[0], block.z_lo,
                                                      block.z_hi, None if dm is None else dm.ctypes.data,
                                                      inc.ctypes.data, None if info is None else info.ctypes.data))
        return inc

    def jacobi_sweep(self, x: np.ndarray, dmem: np.ndarray | None, blocks, frag_z0: int = 0,
                     terms: np.ndarray | None = None, info: np.ndarray | None = None) -> np.ndarray:
        """In place on C-contiguous float64 x / dmem; returns the anchor's
        recorder terms [data, box, tv, axial, f, 0, 0].  dmem=None keeps the
        memory store on the device between calls (session mode)."""
        for a in (x, dmem):
            if a is not None and (a.dtype != np.float64 or not a.flags.c_contiguous):
                raise ValueError("x and dmem must be C-contiguous float64")
        barr = (C.c_int64 * (2 * len(blocks)))(*[v for b in blocks for v in (b.z_lo, b.z_hi)])
        if terms is None:
            terms = np.zeros(N.EVAL_DOUBLES)
        N.check(N.lib.bd3mg_problem_jacobi_sweep_host(self.h, x.ctypes.data, None if dmem is None else dmem.ctypes.data,
                                                      frag_z0, x.shape[0],
                                                      barr, len(blocks), terms.ctypes.data,
                                                      None if info is None else info.ctypes.data))
        return terms
