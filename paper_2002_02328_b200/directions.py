"""Worker-side step kernels (drop-in for ``bd3mg.directions``,
reference pkg/src/bd3mg/directions.py).

``mg_direction`` -- the north-star block step -- runs fused on the GPU via
``bd3mg_mg_steps``: H rows -> residual -> H^T + regulariser epilogue (the
gradient), the forward-only 2x2 Gram <H b_i, H b_j> + regulariser terms for
D = [-g, d_mem], the pruned pseudo-inverse solve and the increment, without
a host round trip.  ``subspace_step``/``pinv_sym`` keep the reference's
generic seam (metric passed as a callable) for the ablation kernels.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import device as D
from .objective import MajorantOperator, Objective, _check_slab, _dtype_of, grad_block
from .volume import SliceBlock

PRUNE_TOL = 1e-14   # directions.py:19
PINV_TOL = 1e-12    # directions.py:22


class MmSolveWarning(UserWarning):
    """The inner linear solve stopped before reaching its residual target."""


@dataclass
class StepInfo:
    """Diagnostics of one subspace solve (reference directions.py:29-40)."""

    increment: object
    gram: np.ndarray
    rhs: np.ndarray
    coeffs: np.ndarray
    ncols: int


def pinv_sym(gram, tol_rel: float = PINV_TOL) -> np.ndarray:
    """Pseudo-inverse of a small symmetric matrix (directions.py:43-54)."""
    m = np.asarray(gram, dtype=np.float64)
    if m.size == 0:
        return m.copy()
    w, vecs = np.linalg.eigh(m)
    amax = float(np.abs(w).max())
    if amax == 0.0:
        return np.zeros_like(m)
    inv = np.where(np.abs(w) > tol_rel * amax, np.divide(1.0, w, where=w != 0), 0.0)
    return (vecs * inv) @ vecs.T


def _vec(a):
    return a.reshape(-1) if D.is_tensor(a) else np.asarray(a, dtype=np.float64).ravel()


def _dot(a, b) -> float:
    if D.is_tensor(a):
        return float(torch.dot(a.double(), b.double()).item())
    return float(a @ b)


def subspace_step(g, d_mem, apply_metric) -> StepInfo:
    """Minimise <g,w> + 1/2 <w, A w> over span{-g, d_mem}
    (directions.py:57-86), generic in the metric."""
    g = _vec(g)
    is_t = D.is_tensor(g)
    finite = bool(torch.isfinite(g).all()) if is_t else bool(np.isfinite(g).all())
    if not finite:
        raise ValueError("non-finite gradient")
    zeros = torch.zeros_like(g) if is_t else np.zeros_like(g)
    zero = StepInfo(zeros, np.zeros((0, 0)), np.zeros(0), np.zeros(0), 0)
    if not (bool(g.any()) if is_t else g.any()):
        return zero
    gnorm = _dot(g, g) ** 0.5
    cols = []
    if gnorm > PRUNE_TOL * (1.0 + gnorm):
        cols.append(-g)
    if d_mem is not None:
        d_mem = _vec(d_mem)
        if is_t and not D.is_tensor(d_mem):
            d_mem = torch.as_tensor(d_mem, dtype=g.dtype, device=g.device)
        if _dot(d_mem, d_mem) ** 0.5 > PRUNE_TOL * (1.0 + gnorm):
            cols.append(d_mem)
    if not cols:
        return zero
    mcols = [apply_metric(c) for c in cols]
    k = len(cols)
    gram = np.array([[_dot(cols[i], mcols[j]) for j in range(k)] for i in range(k)])
    gram = 0.5 * (gram + gram.T)
    rhs = np.array([_dot(c, g) for c in cols])
    coeffs = -pinv_sym(gram) @ rhs
    inc = cols[0] * float(coeffs[0])
    for c, u in zip(cols[1:], coeffs[1:]):
        inc = inc + c * float(u)
    return StepInfo(inc, gram, rhs, coeffs, k)


# ---------------------------------------------------------------------------
def info_to_step(info: np.ndarray, increment) -> StepInfo:
    """StepInfo from the device record (layout: include/bd3mg_b200.h)."""
    k = int(info[7])
    if k == 2:
        gram = np.array([[info[0], info[1]], [info[1], info[2]]])
    elif k == 1:
        gram = np.array([[info[0]]])
    else:
        gram = np.zeros((0, 0))
    return StepInfo(increment, gram, np.asarray(info[3:3 + k]), np.asarray(info[5:5 + k]), k)


_WS_CACHE: dict = {}


def _ws_bytes_cached(g: N.Geom, arr, n: int) -> int:
    """bd3mg_mg_steps_ws_bytes memoised on what it depends on: the geometry,
    each task's rows and which of its pointers are set, and whether the
    tasks share one fragment (the per-update host cost of the runtime's
    schedules)."""
    frag0 = arr[0].frag if n else None
    key = (g.nx, g.ny, g.nz, g.kx, g.ky, g.kz, g.dtype, n,
           all(arr[i].frag == frag0 and arr[i].frag_z0 == arr[0].frag_z0 and arr[i].nzf == arr[0].nzf
               for i in range(n)),
           tuple((t.frag_z0, t.nzf, t.z_lo, t.z_hi, bool(t.d_mem), bool(t.inc_out), bool(t.x_rows),
                  bool(t.dmem_rows)) for t in arr[:n]))
    nbytes = _WS_CACHE.get(key)
    if nbytes is None:
        nbytes = N.ws_bytes(N.lib.bd3mg_mg_steps_ws_bytes(D.byref(g), arr, n))
        if len(_WS_CACHE) > 4096:
            _WS_CACHE.clear()
        _WS_CACHE[key] = nbytes
    return nbytes


def mg_steps_device(obj: Objective, tasks: list[N.Task], dtype: torch.dtype,
                    info: torch.Tensor | None = None, stream=None, mirrors=None) -> torch.Tensor:
    """Launch the fused block steps for `tasks` (device pointers) on the
    current stream; returns the device info tensor (ntasks x 16).
    ``mirrors`` (a list of N.Mirror): updated rows also stored there
    (bd3mg_mg_steps_mirrored; the asynchronous mode's peer halo rings)."""
    n = len(tasks)
    arr = (N.Task * max(n, 1))(*tasks)
    g = obj.geom(dtype)
    nbytes = _ws_bytes_cached(g, arr, n)
    ws = D.workspace(nbytes, stream)
    dev = torch.device("cuda", torch.cuda.current_device())
    if info is None:
        info = torch.empty((n, N.INFO_DOUBLES), dtype=torch.float64, device=dev)
    k = obj.psf.device_kernels(dtype, dev)
    if mirrors:
        marr = (N.Mirror * len(mirrors))(*mirrors)
        N.check(N.lib.bd3mg_mg_steps_mirrored(D.byref(g), D.byref(D.reg(obj.params)), k.data_ptr(),
                                              obj.device_y(dtype, dev).data_ptr(), arr, n, marr, len(mirrors),
                                              info.data_ptr(), ws.data_ptr(), nbytes, D.stream_handle(stream)))
        return info
    N.check(N.lib.bd3mg_mg_steps(D.byref(g), D.byref(D.reg(obj.params)), k.data_ptr(),
                                 obj.device_y(dtype, dev).data_ptr(), arr, n, info.data_ptr(),
                                 ws.data_ptr(), nbytes, D.stream_handle(stream)))
    return info


def mg_step(obj: Objective, x_slab, slab_z0: int, block: SliceBlock, d_mem) -> StepInfo:
    """Fused mg_direction returning the full StepInfo (device increment for
    tensor inputs, numpy otherwise)."""
    _check_slab(obj, x_slab, slab_z0, block)
    dt = _dtype_of(x_slab)
    xt = D.to_device(x_slab, dt)
    n = block.count(obj.dims)
    dt_mem = None
    if d_mem is not None:
        dt_mem = D.to_device(d_mem, dt).reshape(-1)
        if dt_mem.numel() != n:
            raise ValueError(f"memory direction has {dt_mem.numel()} entries, expected {n}")
    inc = torch.empty(n, dtype=dt, device=xt.device)
    task = N.Task(xt.data_ptr(), slab_z0, xt.shape[0], block.z_lo, block.z_hi,
                  D.ptr(dt_mem), inc.data_ptr(), None, None)
    info = mg_steps_device(obj, [task], dt)
    rec = info[0].cpu().numpy()
    if rec[8] == 1.0:
        raise ValueError("non-finite gradient")
    if rec[8] != 0.0:  # overflowed solve: the reference returns the non-finite increment
        inc = torch.full_like(inc, float("nan"))
    return info_to_step(rec, inc if D.is_tensor(x_slab) else D.to_host(inc))


def mg_direction(obj: Objective, x_slab, slab_z0: int, block: SliceBlock, d_mem):
    """Memory-gradient increment with the full curvature metric A_S(x)
    (directions.py:89-94)."""
    return mg_step(obj, x_slab, slab_z0, block, d_mem).increment


# -- ablation kernels (directions.py:97-168) ---------------------------------
def gd_direction(obj: Objective, x_slab, slab_z0: int, block: SliceBlock, L: float):
    """Scaled steepest descent -g / L."""
    if L <= 0:
        raise ValueError("L must be strictly positive")
    g = grad_block(obj, x_slab, block, slab_z0)
    finite = bool(torch.isfinite(g).all()) if D.is_tensor(g) else bool(np.isfinite(g).all())
    if not finite:
        raise ValueError("non-finite gradient")
    return -g / L


def cg_direction(obj: Objective, x_slab, slab_z0: int, block: SliceBlock, d_mem, L: float):
    """Memory-gradient step with the scalar metric L*Id."""
    if L <= 0:
        raise ValueError("L must be strictly positive")
    g = grad_block(obj, x_slab, block, slab_z0)
    return subspace_step(g, d_mem, lambda v: L * v).increment


def cg_solve(apply_A, b, tol: float, maxit: int):
    """Conjugate gradients for SPD A; best iterate on breakdown/budget
    (reference directions.py:117-149).  When A is a block majorant
    (``MajorantOperator.apply``) the whole solve runs on the device
    (bd3mg_cg_solve); any other callable runs this host-driven loop."""
    maj = getattr(apply_A, "__self__", None)
    if isinstance(maj, MajorantOperator) and getattr(apply_A, "__func__", None) is MajorantOperator.apply:
        return maj.solve_cg(b, tol, maxit)
    b = _vec(b)
    x = b * 0
    b_norm = _dot(b, b) ** 0.5
    if b_norm == 0.0:
        return x, True, 0, 0.0
    r = b.clone() if D.is_tensor(b) else b.copy()
    p = r.clone() if D.is_tensor(r) else r.copy()
    rs = _dot(r, r)
    best, best_res = (x.clone() if D.is_tensor(x) else x.copy()), b_norm
    it = 0
    for it in range(1, maxit + 1):
        ap = apply_A(p)
        pap = _dot(p, ap)
        if pap <= 0.0:
            break
        alpha = rs / pap
        x = x + alpha * p
        r = r - alpha * ap
        rs_new = _dot(r, r)
        res = rs_new ** 0.5
        if res < best_res:
            best, best_res = (x.clone() if D.is_tensor(x) else x.copy()), res
        if res <= tol * b_norm:
            return x, True, it, res / b_norm
        p = r + (rs_new / rs) * p
        rs = rs_new
    return best, False, it, best_res / b_norm


def mm_direction(obj: Objective, x_slab, slab_z0: int, block: SliceBlock,
                 cg_tol: float = 1e-8, cg_maxit: int = 200):
    """Full block model minimiser A_S d = -g by CG."""
    if cg_tol <= 0:
        raise ValueError("cg_tol must be strictly positive")
    g = grad_block(obj, x_slab, block, slab_z0)
    finite = bool(torch.isfinite(g).all()) if D.is_tensor(g) else bool(np.isfinite(g).all())
    if not finite:
        raise ValueError("non-finite gradient")
    if not (bool(g.any()) if D.is_tensor(g) else g.any()):
        return g * 0
    maj = MajorantOperator(obj, x_slab, block, slab_z0)
    d, conv, iters, relres = cg_solve(maj.apply, -g, cg_tol, cg_maxit)
    if not conv:
        warnings.warn(f"inner solve stopped after {iters} iterations at relative residual "
                      f"{relres:.3e} (target {cg_tol:.1e})", MmSolveWarning)
    return d
