"""The restoration criterion, its gradient, block restrictions and the block
majorant, evaluated by the fused sm_100a kernels.

Drop-in for ``bd3mg.objective`` (reference pkg/src/bd3mg/objective.py):

    f(x) = 1/2 ||Hx - y||^2 + eta * dist^2(x, [x_min, x_max])
         + lam * sum sqrt((Dx x)^2 + (Dy x)^2 + delta^2) + kappa * ||Dz x||^2

Arrays may be numpy (host float64; results come back as numpy) or CUDA
tensors (float64 or float32; results stay on the device).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import blur
from . import device as D
from .volume import Dims3, SliceBlock, dims_of, philox


@dataclass(frozen=True)
class RegParams:
    """Criterion weights (reference objective.py:46-62)."""

    lam: float = 0.1
    eta: float = 1.0
    kappa: float = 0.05
    delta: float = 0.05
    x_min: float = 0.0
    x_max: float = 1.0

    def __post_init__(self):
        if min(self.lam, self.eta, self.kappa, self.delta) <= 0:
            raise ValueError("lam, eta, kappa, delta must be strictly positive")
        if not self.x_min < self.x_max:
            raise ValueError("x_min must be < x_max")


@dataclass
class Objective:
    """PSF stack, observation and weights (reference objective.py:65-82).
    The observation is uploaded once per (dtype, device)."""

    psf: blur.PsfStack
    y: np.ndarray
    params: RegParams
    _dev: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        if D.is_tensor(self.y):
            t = self.y.detach()
            if t.is_cuda and t.dtype in (torch.float64, torch.float32):
                # already resident (e.g. volume.read_volume(..., device=)): reuse it
                self._dev[(t.dtype, t.device.index)] = t.contiguous()
            self.y = t.to("cpu", torch.float64).numpy()
        self.y = np.ascontiguousarray(self.y, dtype=np.float64)
        if dims_of(self.y) != self.psf.dims:
            raise ValueError("observation dims do not match PSF dims")
        if not np.isfinite(self.y).all():
            raise ValueError("observation contains non-finite entries")

    @property
    def dims(self) -> Dims3:
        return self.psf.dims

    def device_y(self, dtype: torch.dtype = torch.float64, device=None) -> torch.Tensor:
        dev = torch.device(device) if device is not None else D.default_device()
        key = (dtype, dev.index if dev.index is not None else torch.cuda.current_device())
        t = self._dev.get(key)
        if t is None:
            t = torch.from_numpy(self.y).to(dev).to(dtype).contiguous()
            self._dev[key] = t
        return t

    def geom(self, dtype: torch.dtype) -> N.Geom:
        return D.geom(self.dims, self.psf.kdims, dtype)


def _dtype_of(a) -> torch.dtype:
    return torch.float32 if D.is_tensor(a) and a.dtype == torch.float32 else torch.float64


# ---------------------------------------------------------------------------
def eval_terms(obj: Objective, x, snap=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device vector [data, box, tv, axial, f, |x-snap|^2, |snap|^2]
    (objective.py:140-156 and the stop-rule norms of scheduler.py:218-219)."""
    dt = _dtype_of(x)
    xt = D.to_device(x, dt)
    if dims_of(xt) != obj.dims:
        raise ValueError("volume dims do not match objective dims")
    st = D.to_device(snap, dt) if snap is not None else None
    g = obj.geom(dt)
    nbytes = N.ws_bytes(N.lib.bd3mg_eval_f_ws_bytes(D.byref(g)))
    ws = D.workspace(nbytes)
    if out is None:
        out = torch.empty(N.EVAL_DOUBLES, dtype=torch.float64, device=xt.device)
    k = obj.psf.device_kernels(dt, xt.device)
    N.check(N.lib.bd3mg_eval_f(D.byref(g), D.byref(D.reg(obj.params)), k.data_ptr(),
                               obj.device_y(dt, xt.device).data_ptr(), xt.data_ptr(), D.ptr(st),
                               out.data_ptr(), ws.data_ptr(), nbytes, D.stream_handle()))
    return out


def eval_f(obj: Objective, x) -> float:
    """Full objective value; raises if not finite (objective.py:140-156)."""
    value = float(eval_terms(obj, x)[4].item())
    if not math.isfinite(value):
        raise ValueError("objective evaluated to a non-finite value")
    return value


def grad_rows_device(obj: Objective, frag, frag_z0: int, lo: int, hi: int):
    """(g, omega) rows [lo, hi] as device tensors (objective.py:159-187)."""
    dt = _dtype_of(frag)
    ft = D.to_device(frag, dt)
    g = obj.geom(dt)
    nbytes = N.ws_bytes(N.lib.bd3mg_grad_rows_ws_bytes(D.byref(g), lo, hi))
    ws = D.workspace(nbytes)
    ny, nx = obj.dims.ny, obj.dims.nx
    gout = torch.empty((hi - lo + 1, ny, nx), dtype=dt, device=ft.device)
    wout = torch.empty_like(gout)
    k = obj.psf.device_kernels(dt, ft.device)
    N.check(N.lib.bd3mg_grad_rows(D.byref(g), D.byref(D.reg(obj.params)), k.data_ptr(),
                                  obj.device_y(dt, ft.device).data_ptr(), ft.data_ptr(), frag_z0,
                                  ft.shape[0], lo, hi, gout.data_ptr(), wout.data_ptr(), ws.data_ptr(),
                                  nbytes, D.stream_handle()))
    return gout, wout


def grad_f(obj: Objective, x):
    """Gradient of the full objective (objective.py:190-195)."""
    if dims_of(x) != obj.dims:
        raise ValueError("volume dims do not match objective dims")
    g, _ = grad_rows_device(obj, x, 0, 0, obj.dims.nz - 1)
    return g if D.is_tensor(x) else D.to_host(g)


def _check_slab(obj: Objective, frag, frag_z0: int, block: SliceBlock) -> None:
    slab = blur.slab_support(obj.psf, block)
    top = frag_z0 + frag.shape[0] - 1
    if frag_z0 > slab.z_lo or top < slab.z_hi:
        raise ValueError(
            f"slab [{frag_z0}, {top}] does not cover the required support "
            f"[{slab.z_lo}, {slab.z_hi}] of block {block}")


def grad_block(obj: Objective, x, block: SliceBlock, x_z0: int = 0):
    """Block restriction of the gradient, flattened (objective.py:206-214)."""
    _check_slab(obj, x, x_z0, block)
    g, _ = grad_rows_device(obj, x, x_z0, block.z_lo, block.z_hi)
    g = g.reshape(-1)
    return g if D.is_tensor(x) else D.to_host(g)


class MajorantOperator:
    """Matrix-free principal submatrix A_S(x~) of the curvature operator for
    one block, half-quadratic weights cached at construction
    (objective.py:217-287)."""

    def __init__(self, obj: Objective, anchor, block: SliceBlock, anchor_z0: int = 0):
        self.obj = obj
        self.block = block.check_within(obj.dims)
        self._host = not D.is_tensor(anchor)
        self.dtype = _dtype_of(anchor)
        self.anchor = np.ascontiguousarray(anchor, dtype=np.float64) if self._host else anchor
        self.anchor_z0 = anchor_z0
        _check_slab(obj, self.anchor, anchor_z0, block)
        at = D.to_device(self.anchor, self.dtype)
        self._dev_anchor = at
        g = obj.geom(self.dtype)
        d = obj.dims
        self.omega = torch.empty((block.height, d.ny, d.nx), dtype=self.dtype, device=at.device)
        N.check(N.lib.bd3mg_omega_rows(D.byref(g), D.byref(D.reg(obj.params)), at.data_ptr(), anchor_z0,
                                       at.shape[0], block.z_lo, block.z_hi, self.omega.data_ptr(),
                                       D.stream_handle()))
        rows = self.anchor[block.z_lo - anchor_z0:block.z_hi - anchor_z0 + 1]
        self._anchor_rows = rows.copy() if self._host else rows.clone()
        self.n = block.count(obj.dims)
        self._f_anchor = None
        self._g_anchor = None

    def apply_device(self, v: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        vt = D.to_device(v, self.dtype)
        if vt.numel() != self.n or (vt.ndim == 1 and vt.shape[0] != self.n):
            raise ValueError(f"expected flat vector of length {self.n}, got {tuple(vt.shape)}")
        g = self.obj.geom(self.dtype)
        blk = self.block
        nbytes = N.ws_bytes(N.lib.bd3mg_majorant_apply_ws_bytes(D.byref(g), blk.z_lo, blk.z_hi))
        ws = D.workspace(nbytes)
        if out is None:
            out = torch.empty(self.n, dtype=self.dtype, device=vt.device)
        k = self.obj.psf.device_kernels(self.dtype, vt.device)
        N.check(N.lib.bd3mg_majorant_apply(D.byref(g), D.byref(D.reg(self.obj.params)), k.data_ptr(),
                                           self.omega.data_ptr(), vt.data_ptr(), blk.z_lo, blk.z_hi,
                                           out.data_ptr(), ws.data_ptr(), nbytes, D.stream_handle()))
        return out

    def apply(self, v):
        """A_S(x~) v for a flat block vector (objective.py:245-275)."""
        if not D.is_tensor(v):
            v = np.asarray(v, dtype=np.float64)
            if v.shape != (self.n,):
                raise ValueError(f"expected flat vector of length {self.n}, got {v.shape}")
            return D.to_host(self.apply_device(v))
        if tuple(v.shape) != (self.n,):
            raise ValueError(f"expected flat vector of length {self.n}, got {tuple(v.shape)}")
        return self.apply_device(v)

    def solve_cg(self, b, tol: float, maxit: int):
        """Conjugate gradients for A_S(x~) w = b on the device
        (bd3mg_cg_solve; reference directions.py:117-149): no host round trip
        per iteration.  Returns (w, converged, iterations, relative_residual)
        with w a device tensor for tensor input, numpy otherwise."""
        bt = D.to_device(b, self.dtype).reshape(-1)
        if bt.numel() != self.n:
            raise ValueError(f"expected flat vector of length {self.n}, got {tuple(bt.shape)}")
        g = self.obj.geom(self.dtype)
        blk = self.block
        nbytes = N.ws_bytes(N.lib.bd3mg_cg_solve_ws_bytes(D.byref(g), blk.z_lo, blk.z_hi))
        ws = D.workspace(nbytes)
        out = torch.empty(self.n, dtype=self.dtype, device=bt.device)
        state = torch.zeros(16, dtype=torch.float64, device=bt.device)
        k = self.obj.psf.device_kernels(self.dtype, bt.device)
        N.check(N.lib.bd3mg_cg_solve(D.byref(g), D.byref(D.reg(self.obj.params)), k.data_ptr(), self.omega.data_ptr(),
                                     bt.contiguous().data_ptr(), blk.z_lo, blk.z_hi, float(tol), int(maxit),
                                     out.data_ptr(), state.data_ptr(), ws.data_ptr(), nbytes, D.stream_handle()))
        st = state.cpu().numpy()
        status, iters = int(st[5]), int(st[6])
        relres = float(st[7]) if status != 0 else float(st[2] / st[0])
        w = out if D.is_tensor(b) else D.to_host(out)
        return w, status == 1, iters, relres

    def _anchor_data(self):
        if self._g_anchor is None:
            if self.anchor_z0 != 0 or self.anchor.shape[0] != self.obj.dims.nz:
                raise ValueError("quadratic model value requires a full-volume anchor")
            cur = self.anchor[self.block.z_lo:self.block.z_hi + 1]
            same = (np.array_equal(cur, self._anchor_rows) if self._host
                    else bool(torch.equal(cur, self._anchor_rows)))
            if not same:
                raise RuntimeError("anchor mutated after the weight cache was built")
            self._f_anchor = eval_f(self.obj, self.anchor)
            self._g_anchor = grad_block(self.obj, self.anchor, self.block)
        return self._f_anchor, self._g_anchor


def majorant_apply(maj: MajorantOperator, v):
    return maj.apply(v)


def majorant_Q(maj: MajorantOperator, v) -> float:
    """Q_S(v, x~) = f(x~) + <g, v - x~_S> + 1/2 <v - x~_S, A_S (v - x~_S)>
    (objective.py:294-298); evaluated in float64 on the host."""
    f0, g = maj._anchor_data()
    g = np.asarray(D.to_host(g) if D.is_tensor(g) else g, dtype=np.float64)
    rows = maj._anchor_rows
    rows = D.to_host(rows) if D.is_tensor(rows) else rows
    vv = D.to_host(v) if D.is_tensor(v) else np.asarray(v, dtype=np.float64)
    d = vv - rows.ravel()
    ad = maj.apply(d)
    return f0 + float(g @ d) + 0.5 * float(d @ ad)


# -- Lipschitz bound (reference objective.py:301-375; ablation support) ------
_DIFF_NORM_SQ = 4.0


def lipschitz_bound(rho_hth: float, params: RegParams | None = None, *, lam: float = None,
                    eta: float = None, kappa: float = None, delta: float = None) -> float:
    if params is not None:
        lam, eta, kappa, delta = params.lam, params.eta, params.kappa, params.delta
    return rho_hth + 2.0 * eta + (lam / delta) * 2.0 * _DIFF_NORM_SQ + 2.0 * kappa * _DIFF_NORM_SQ


def operator_norm_bound(psf: blur.PsfStack) -> float:
    """||H||_1 ||H||_inf >= rho(H^T H) (reference objective.py:322-342)."""
    nz, kz = psf.dims.nz, psf.kdims.kz
    rz = (kz - 1) // 2
    a = np.abs(psf.kernels)
    hinf = float(a.reshape(nz, -1).sum(axis=1).max())
    page = a.sum(axis=(2, 3))
    h1 = 0.0
    for zi in range(nz):
        tot = 0.0
        for k in range(kz):
            zo = zi + rz - k
            if 0 <= zo < nz:
                tot += page[zo, k]
        h1 = max(h1, tot)
    return h1 * hinf


def rho_hth_estimate(psf: blur.PsfStack, iters: int = 50, seed: int = 0) -> float:
    """Power iteration on H^T H, inflated 5%, capped by the norm bound
    (reference objective.py:345-370).  The iteration runs on the device
    (bd3mg_power_hth: every |H^T H v| is kept in a device array, one host
    read at the end); should H annihilate an iterate, the remaining steps
    replay the reference's RNG restarts on the host path."""
    rng = philox(seed)
    dev = D.default_device()
    v = torch.from_numpy(rng.uniform(0.1, 1.0, psf.dims.shape)).to(dev)
    v /= torch.linalg.vector_norm(v)
    dt = torch.float64
    g = D.geom(psf.dims, psf.kdims, dt)
    nbytes = N.ws_bytes(N.lib.bd3mg_power_hth_ws_bytes(D.byref(g)))
    ws = D.workspace(nbytes)
    norms = torch.zeros(max(iters, 1), dtype=torch.float64, device=dev)
    state = torch.zeros(2, dtype=torch.float64, device=dev)
    k = psf.device_kernels(dt, dev)
    N.check(N.lib.bd3mg_power_hth(D.byref(g), k.data_ptr(), v.data_ptr(), int(iters), norms.data_ptr(),
                                  state.data_ptr(), ws.data_ptr(), nbytes, D.stream_handle()))
    nrm = norms.cpu().numpy()[:iters]
    bound = operator_norm_bound(psf)
    if state[0].item() != 0.0:
        return _rho_hth_host(psf, iters, seed)
    est = float(nrm[-1]) if iters >= 1 else 0.0
    prev = float(nrm[-2]) if iters >= 2 else 0.0
    if not (est > 0 and abs(est - prev) <= 1e-3 * est):
        return bound
    return min(1.05 * est, bound)


def _rho_hth_host(psf: blur.PsfStack, iters: int, seed: int) -> float:
    """Host-orchestrated power iteration (device operators, one sync per
    step) reproducing the reference's RNG restarts when H annihilates an
    iterate (objective.py:361-364)."""
    rng = philox(seed)
    v = torch.from_numpy(rng.uniform(0.1, 1.0, psf.dims.shape)).to(D.default_device())
    v /= torch.linalg.vector_norm(v)
    est = prev = 0.0
    for _ in range(iters):
        w = blur.apply_Ht(psf, blur.apply_H(psf, v))
        nrm = float(torch.linalg.vector_norm(w).item())
        if nrm == 0.0:
            v = torch.from_numpy(rng.uniform(0.1, 1.0, psf.dims.shape)).to(v.device)
            v /= torch.linalg.vector_norm(v)
            continue
        prev, est = est, nrm
        v = w / nrm
    bound = operator_norm_bound(psf)
    if not (est > 0 and abs(est - prev) <= 1e-3 * est):
        return bound
    return min(1.05 * est, bound)


def lipschitz_estimate(obj: Objective, iters: int = 50, seed: int = 0) -> float:
    return lipschitz_bound(rho_hth_estimate(obj.psf, iters, seed), obj.params)
