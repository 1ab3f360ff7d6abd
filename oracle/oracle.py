"""TEST INFRASTRUCTURE ONLY -- CPU oracle of the BD3MG hot path.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module; the product package never does (it has no CPU path).

A numpy restatement of the reference algorithm (arXiv 2002.02328 CPU
reference, /root/reference/pkg/src/bd3mg), each routine citing the lines it
follows.  The operator loops H / H^T come from one of two native cores:

* ``"c"``   -- oracle/bd3mg_oracle.c, a plain-C restatement of _core.pyx
               (built by ``make -C oracle``), OpenMP over output rows;
* ``"ref"`` -- the reference's own Cython core, compiled from
               /root/reference by ``make -C oracle ref`` into oracle/_ref/.

Pinning: tests/test_oracle_golden.py checks this module against vectors
produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import heapq
import importlib.util
import math
import os
import sysconfig
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
C_LIB = HERE / "liboracle_bd3mg.so"
REF_CORE = HERE / "_ref" / ("_core" + sysconfig.get_config_var("EXT_SUFFIX"))

PRUNE_TOL = 1e-14  # directions.py:19
PINV_TOL = 1e-12   # directions.py:22


# ---------------------------------------------------------------------------
# native cores
class _CCore:
    name = "c"

    def __init__(self, threads: int):
        if not C_LIB.exists():
            raise ImportError(f"{C_LIB} missing: run `make -C oracle`")
        self.lib = ctypes.CDLL(str(C_LIB))
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        args = [vp, i64, i64, i64, vp, i64, i64, i64, i64, i64, i64, i64, vp, ctypes.c_int]
        self.lib.oracle_correlate.argtypes = args
        self.lib.oracle_correlate_adjoint.argtypes = args
        self.threads = threads

    def _run(self, fn, frag, ker, z0, lo, hi):
        frag = np.ascontiguousarray(frag, dtype=np.float64)
        ker = np.ascontiguousarray(ker, dtype=np.float64)
        nzf, ny, nx = frag.shape
        nzk, kz, ky, kx = ker.shape
        out = np.zeros((hi - lo + 1, ny, nx))
        rc = fn(frag.ctypes.data, nzf, ny, nx, ker.ctypes.data, nzk, kz, ky, kx, z0, lo, hi,
                out.ctypes.data, self.threads)
        if rc:
            raise ValueError("invalid row range")
        return out

    def correlate(self, frag, ker, z0, lo, hi):
        return self._run(self.lib.oracle_correlate, frag, ker, z0, lo, hi)

    def correlate_adjoint(self, frag, ker, z0, lo, hi):
        return self._run(self.lib.oracle_correlate_adjoint, frag, ker, z0, lo, hi)


class _RefCore:
    """The reference's compiled _core (src/_core.pyx), single-threaded per
    call with the GIL released, exactly as the reference runs it."""

    name = "ref"

    def __init__(self):
        if not REF_CORE.exists():
            raise ImportError(f"{REF_CORE} missing: run `make -C oracle ref` where /root/reference exists")
        spec = importlib.util.spec_from_file_location("_core", REF_CORE)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        self.mod = mod

    def correlate(self, frag, ker, z0, lo, hi):
        return self.mod.depthvar_correlate(np.ascontiguousarray(frag, dtype=np.float64), ker, z0, lo, hi)

    def correlate_adjoint(self, frag, ker, z0, lo, hi):
        return self.mod.depthvar_correlate_adjoint(np.ascontiguousarray(frag, dtype=np.float64), ker, z0, lo, hi)


class _ScipyCore:
    """Restatement of the reference's fallback backend (src/_kernels_np.py:15-46):
    per output row and tap page, one 2-D ``scipy.ndimage.correlate`` with
    zero padding, accumulated in tap order; the adjoint correlates the page
    flipped in y and x (:43).  Same contract as the compiled core; rounding
    differs from it by <= 1e-13 (reference tests/test_blur.py:151-159).  Used
    by bench.py's reference arm, which reports the faster of the two
    reference backends."""

    name = "scipy"

    def __init__(self):
        from scipy import ndimage
        self.nd = ndimage

    def correlate(self, frag, ker, z0, lo, hi):
        frag = np.ascontiguousarray(frag, dtype=np.float64)
        nzf, ny, nx = frag.shape
        kz = ker.shape[1]
        rz = (kz - 1) // 2
        out = np.zeros((hi - lo + 1, ny, nx))
        for zo in range(lo, hi + 1):
            for a in range(kz):
                zi = zo + a - rz - z0
                if 0 <= zi < nzf:
                    out[zo - lo] += self.nd.correlate(frag[zi], ker[zo, a], mode="constant", cval=0.0)
        return out

    def correlate_adjoint(self, frag, ker, z0, lo, hi):
        frag = np.ascontiguousarray(frag, dtype=np.float64)
        nzf, ny, nx = frag.shape
        nzk, kz = ker.shape[0], ker.shape[1]
        rz = (kz - 1) // 2
        out = np.zeros((hi - lo + 1, ny, nx))
        for zi in range(lo, hi + 1):
            for a in range(kz):
                zo = zi + rz - a
                if 0 <= zo < nzk and 0 <= zo - z0 < nzf:
                    out[zi - lo] += self.nd.correlate(frag[zo - z0], ker[zo, a, ::-1, ::-1], mode="constant",
                                                      cval=0.0)
        return out


_core = None


def core(kind: str | None = None, threads: int | None = None):
    """Select/return the active H/H^T core ("c" default, "ref" or "scipy")."""
    global _core
    if kind is not None or _core is None:
        kind = kind or os.environ.get("BD3MG_ORACLE_CORE", "c")
        if kind == "ref":
            _core = _RefCore()
        elif kind == "scipy":
            _core = _ScipyCore()
        else:
            _core = _CCore(threads or int(os.environ.get("BD3MG_ORACLE_THREADS", "1")))
    return _core


def ref_core_available() -> bool:
    return REF_CORE.exists()


# ---------------------------------------------------------------------------
# operator layer (reference blur.py:163-198)
def H_rows(ker, frag, z0, lo, hi):
    return core().correlate(frag, ker, z0, lo, hi)


def Ht_rows(ker, frag, z0, lo, hi):
    return core().correlate_adjoint(frag, ker, z0, lo, hi)


def H(ker, x):
    return H_rows(ker, x, 0, 0, x.shape[0] - 1)


def Ht(ker, v):
    return Ht_rows(ker, v, 0, 0, v.shape[0] - 1)


def support(nz: int, kz: int, lo: int, hi: int) -> tuple[int, int]:
    """slab_support: block dilated by kz planes, clamped (blur.py:190-198)."""
    return max(0, lo - kz), min(nz - 1, hi + kz)


def gaussian_psf(kx, ky, kz, s1, s2, s3, phi, theta):
    """Rotated anisotropic Gaussian, unit sum (blur.py:100-124)."""
    rzm = np.array([[math.cos(phi), -math.sin(phi), 0.0], [math.sin(phi), math.cos(phi), 0.0], [0.0, 0.0, 1.0]])
    rym = np.array([[math.cos(theta), 0.0, math.sin(theta)], [0.0, 1.0, 0.0],
                    [-math.sin(theta), 0.0, math.cos(theta)]])
    r = rym @ rzm
    q = r.T @ np.diag([s1**-2, s2**-2, s3**-2]) @ r
    ax = [np.arange(n, dtype=np.float64) - (n - 1) / 2 for n in (kx, ky, kz)]
    gz, gy, gx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    e = (q[0, 0] * gx**2 + q[1, 1] * gy**2 + q[2, 2] * gz**2
         + 2.0 * (q[0, 1] * gx * gy + q[0, 2] * gx * gz + q[1, 2] * gy * gz))
    k = np.exp(-0.5 * e)
    return k / k.sum()


# ---------------------------------------------------------------------------
# criterion (reference objective.py:87-298)
def _fd(a, axis):
    out = np.zeros_like(a)
    if a.shape[axis] > 1:
        hi = [slice(None)] * 3
        lo = [slice(None)] * 3
        hi[axis], lo[axis] = slice(1, None), slice(None, -1)
        out[tuple(lo)] = a[tuple(hi)] - a[tuple(lo)]
    return out


def _fd_adj(w, axis):
    """Exact adjoint of _fd along `axis` (objective.py:101-120)."""
    out = np.zeros_like(w)
    n = w.shape[axis]
    if n == 1:
        return out

    def sl(s):
        idx = [slice(None)] * 3
        idx[axis] = s
        return tuple(idx)

    out[sl(0)] = -w[sl(0)]
    out[sl(slice(1, -1))] = w[sl(slice(None, -2))] - w[sl(slice(1, -1))]
    out[sl(-1)] = w[sl(-2)]
    return out


@dataclass
class Criterion:
    """f(x) = 1/2||Hx-y||^2 + eta dist^2(x,[x_min,x_max]) + lam TV_delta(x)
    + kappa ||Dz x||^2 (objective.py:1-33)."""

    kernels: np.ndarray
    y: np.ndarray
    lam: float = 0.1
    eta: float = 1.0
    kappa: float = 0.05
    delta: float = 0.05
    x_min: float = 0.0
    x_max: float = 1.0

    @property
    def nz(self):
        return self.y.shape[0]

    @property
    def rz(self):
        return (self.kernels.shape[1] - 1) // 2

    @property
    def kz(self):
        return self.kernels.shape[1]

    def weights(self, rows):
        """1/sqrt(dx^2+dy^2+delta^2) (objective.py:130-132)."""
        return 1.0 / np.sqrt(_fd(rows, 2) ** 2 + _fd(rows, 1) ** 2 + self.delta**2)

    def terms(self, x):
        """(data, box, tv, axial) of eval_f (objective.py:140-156)."""
        r = H(self.kernels, x) - self.y
        data = 0.5 * float(np.vdot(r, r))
        e = x - np.clip(x, self.x_min, self.x_max)
        box = self.eta * float(np.vdot(e, e))
        tv = self.lam * float(np.sqrt(_fd(x, 2) ** 2 + _fd(x, 1) ** 2 + self.delta**2).sum())
        dz = _fd(x, 0)
        axial = self.kappa * float(np.vdot(dz, dz))
        return data, box, tv, axial

    def value(self, x):
        v = sum(self.terms(x))
        if not math.isfinite(v):
            raise ValueError("objective evaluated to a non-finite value")
        return v

    def grad_rows(self, frag, z0, lo, hi):
        """Gradient rows [lo, hi] from a fragment (objective.py:159-187)."""
        nz, rz = self.nz, self.rz
        olo, ohi = max(0, lo - rz), min(nz - 1, hi + rz)
        r = H_rows(self.kernels, frag, z0, olo, ohi) - self.y[olo:ohi + 1]
        g = Ht_rows(self.kernels, r, olo, lo, hi)
        rows = frag[lo - z0:hi - z0 + 1]
        g += 2.0 * self.eta * (rows - np.clip(rows, self.x_min, self.x_max))
        w = self.weights(rows)
        g += self.lam * (_fd_adj(w * _fd(rows, 2), 2) + _fd_adj(w * _fd(rows, 1), 1))
        dz = np.zeros((hi - lo + 2,) + frag.shape[1:])
        for t, z in enumerate(range(lo - 1, hi + 1)):
            if 0 <= z < nz - 1:
                dz[t] = frag[z + 1 - z0] - frag[z - z0]
        g += 2.0 * self.kappa * (dz[:-1] - dz[1:])
        return g

    def grad(self, x):
        return self.grad_rows(x, 0, 0, self.nz - 1)

    def check_slab(self, frag_z0, nzf, lo, hi):
        s_lo, s_hi = support(self.nz, self.kz, lo, hi)
        if frag_z0 > s_lo or frag_z0 + nzf - 1 < s_hi:
            raise ValueError(f"slab [{frag_z0}, {frag_z0 + nzf - 1}] does not cover the required support "
                             f"[{s_lo}, {s_hi}]")

    def grad_block(self, frag, lo, hi, z0=0):
        self.check_slab(z0, frag.shape[0], lo, hi)
        return self.grad_rows(frag, z0, lo, hi).ravel()

    def majorant(self, anchor, lo, hi, z0=0):
        """v -> A_S(x~) v for block [lo, hi] (objective.py:227-275)."""
        self.check_slab(z0, anchor.shape[0], lo, hi)
        w = self.weights(anchor[lo - z0:hi - z0 + 1])
        nz, rz, h = self.nz, self.rz, hi - lo + 1
        shape = (h,) + anchor.shape[1:]

        def apply(v):
            v = np.asarray(v, dtype=np.float64)
            if v.shape != (h * shape[1] * shape[2],):
                raise ValueError(f"expected flat vector of length {h * shape[1] * shape[2]}, got {v.shape}")
            vb = np.ascontiguousarray(v.reshape(shape))
            olo, ohi = max(0, lo - rz), min(nz - 1, hi + rz)
            out = Ht_rows(self.kernels, H_rows(self.kernels, vb, lo, olo, ohi), olo, lo, hi)
            out += 2.0 * self.eta * vb
            out += self.lam * (_fd_adj(w * _fd(vb, 2), 2) + _fd_adj(w * _fd(vb, 1), 1))
            dz = np.zeros((h + 1,) + shape[1:])
            if lo - 1 >= 0:
                dz[0] = vb[0]
            dz[1:h] = vb[1:] - vb[:-1]
            if hi < nz - 1:
                dz[h] = -vb[h - 1]
            out += 2.0 * self.kappa * (dz[:-1] - dz[1:])
            return out.ravel()

        apply.omega = w
        return apply


# ---------------------------------------------------------------------------
# step (reference directions.py:43-94)
def pinv_sym(m, tol=PINV_TOL):
    m = np.asarray(m, dtype=np.float64)
    if m.size == 0:
        return m.copy()
    lam, vec = np.linalg.eigh(m)
    top = float(np.abs(lam).max())
    if top == 0.0:
        return np.zeros_like(m)
    inv = np.where(np.abs(lam) > tol * top, np.divide(1.0, lam, where=lam != 0), 0.0)
    return (vec * inv) @ vec.T


@dataclass
class Step:
    increment: np.ndarray
    gram: np.ndarray
    rhs: np.ndarray
    coeffs: np.ndarray
    ncols: int


def subspace_step(g, d_mem, metric) -> Step:
    g = np.asarray(g, dtype=np.float64)
    if not np.isfinite(g).all():
        raise ValueError("non-finite gradient")
    empty = Step(np.zeros_like(g), np.zeros((0, 0)), np.zeros(0), np.zeros(0), 0)
    if not g.any():
        return empty
    gn = float(np.linalg.norm(g))
    basis = []
    if gn > PRUNE_TOL * (1.0 + gn):
        basis.append(-g)
    if d_mem is not None:
        d_mem = np.asarray(d_mem, dtype=np.float64)
        if float(np.linalg.norm(d_mem)) > PRUNE_TOL * (1.0 + gn):
            basis.append(d_mem)
    if not basis:
        return empty
    B = np.stack(basis, axis=1)
    AB = np.stack([metric(B[:, j]) for j in range(B.shape[1])], axis=1)
    G = B.T @ AB
    G = 0.5 * (G + G.T)
    rhs = B.T @ g
    u = -pinv_sym(G) @ rhs
    return Step(B @ u, G, rhs, u, B.shape[1])


def mg_step(crit: Criterion, slab, z0, lo, hi, d_mem) -> Step:
    g = crit.grad_block(slab, lo, hi, z0)
    return subspace_step(g, d_mem, crit.majorant(slab, lo, hi, z0))


def mg_direction(crit: Criterion, slab, z0, lo, hi, d_mem):
    return mg_step(crit, slab, z0, lo, hi, d_mem).increment


# ---------------------------------------------------------------------------
# master + engines (reference scheduler.py:92-219, runtime.py:108-292)
@dataclass
class Ledger:
    x: np.ndarray
    blocks: list
    k: int = 0
    cursor: int = 0
    busy: dict = field(default_factory=dict)      # worker -> (block index, issue k)
    prev: np.ndarray = None
    snap: np.ndarray = None
    visited: set = field(default_factory=set)
    tau_hat: int = 0
    staleness: list = field(default_factory=list)
    grants: list = field(default_factory=list)


def blocks_of(nz, h):
    return [(lo, min(lo + h - 1, nz - 1)) for lo in range(0, nz, h)]


def start(x0, workers, h):
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    L = Ledger(x=x0.copy(), blocks=blocks_of(x0.shape[0], h), prev=np.zeros_like(x0), snap=x0.copy())
    if workers * h > x0.shape[0]:
        raise ValueError("too many workers")
    L.cursor = workers % len(L.blocks)
    for c in range(1, workers + 1):
        L.busy[c] = (c - 1, 0)
        L.grants.append(c - 1)
    return L


def task(L, crit, worker):
    """Snapshot of the slab + memory direction (scheduler.py:186-194)."""
    bi, issue = L.busy[worker]
    lo, hi = L.blocks[bi]
    s_lo, s_hi = support(L.x.shape[0], crit.kz, lo, hi)
    return (worker, bi, s_lo, L.x[s_lo:s_hi + 1].copy(), L.prev[lo:hi + 1].ravel().copy(), issue)


def apply_update(L, worker, inc):
    """receive_update (scheduler.py:133-164)."""
    bi, issue = L.busy.pop(worker)
    lo, hi = L.blocks[bi]
    inc = np.asarray(inc, dtype=np.float64).reshape((hi - lo + 1,) + L.x.shape[1:])
    L.x[lo:hi + 1] += inc
    L.prev[lo:hi + 1] = inc
    st = L.k - issue
    L.staleness.append(st)
    L.tau_hat = max(L.tau_hat, st)
    L.k += 1
    L.visited.add(bi)


def grant(L, worker):
    """Round-robin, skipping busy blocks (scheduler.py:167-183)."""
    held = {b for b, _ in L.busy.values()}
    n = len(L.blocks)
    for s in range(n):
        idx = (L.cursor + s) % n
        if idx not in held:
            L.cursor = (idx + 1) % n
            L.busy[worker] = (idx, L.k)
            L.grants.append(idx)
            return idx
    raise RuntimeError("no free block")


def _sweep_record(L, crit, log, tol, max_updates, now):
    """_Recorder.after_update (runtime.py:126-141) + should_stop/roll_sweep."""
    if len(L.visited) == len(L.blocks):
        log.append((L.k, now, crit.value(L.x), L.tau_hat))
        if max_updates is not None and L.k >= max_updates:
            stop = True
        elif math.isinf(tol):
            stop = True
        else:
            stop = float(np.linalg.norm(L.x - L.snap)) <= tol * float(np.linalg.norm(L.snap))
        L.snap = L.x.copy()
        L.visited.clear()
        return stop
    if max_updates is not None and L.k >= max_updates:
        log.append((L.k, now, crit.value(L.x), L.tau_hat))
        return True
    return False


def _service(seed, base=1.0, jitter=0.3):
    rng = np.random.Generator(np.random.Philox(seed))
    return lambda: max(1e-9, base + jitter * (2.0 * rng.random() - 1.0))


def run_bd3mg(crit, x0, workers, h, tol=1e-30, max_updates=None, seed=0):
    """Simulated asynchronous engine (runtime.py:158-180); workers = 1 is
    the deterministic cyclic schedule.  Returns (x, log)."""
    L = start(x0, workers, h)
    draw = _service(seed)
    heap, seq = [], 0
    for c in range(1, workers + 1):
        heapq.heappush(heap, (draw(), seq, task(L, crit, c)))
        seq += 1
    log = []
    while heap:
        now, _, t = heapq.heappop(heap)
        worker, bi, s_lo, slab, dm, _ = t
        lo, hi = L.blocks[bi]
        apply_update(L, worker, mg_direction(crit, slab, s_lo, lo, hi, dm))
        if _sweep_record(L, crit, log, tol, max_updates, now):
            break
        grant(L, worker)
        heapq.heappush(heap, (now + draw(), seq, task(L, crit, worker)))
        seq += 1
    return L.x.copy(), log, L


def run_bp3mg(crit, x0, workers, h, tol=1e-30, max_updates=None, seed=0):
    """Barrier engine (runtime.py:244-292): all workers anchored at the same
    iterate, increments applied jointly."""
    L = start(x0, workers, h)
    draw = _service(seed)
    tasks = [task(L, crit, c) for c in range(1, workers + 1)]
    log, now, stop = [], 0.0, False
    while not stop:
        incs = []
        for worker, bi, s_lo, slab, dm, _ in tasks:
            lo, hi = L.blocks[bi]
            incs.append(mg_direction(crit, slab, s_lo, lo, hi, dm))
        now += max(draw() for _ in tasks)
        for t, inc in zip(tasks, incs):
            apply_update(L, t[0], inc)
            if _sweep_record(L, crit, log, tol, max_updates, now):
                stop = True
        if stop:
            break
        for c in range(1, workers + 1):
            grant(L, c)
        tasks = [task(L, crit, c) for c in range(1, workers + 1)]
    return L.x.copy(), log, L


# ---------------------------------------------------------------------------
# ablation directions + Lipschitz estimate (reference directions.py:97-168,
# objective.py:301-375)
def gd_direction(crit: Criterion, slab, z0, lo, hi, L):
    """-g / L (directions.py:95-104)."""
    if L <= 0:
        raise ValueError("L must be strictly positive")
    g = crit.grad_block(slab, lo, hi, z0)
    if not np.isfinite(g).all():
        raise ValueError("non-finite gradient")
    return -g / L


def cg_direction(crit: Criterion, slab, z0, lo, hi, d_mem, L):
    """Memory-gradient step with the scalar metric L*Id (directions.py:107-114)."""
    if L <= 0:
        raise ValueError("L must be strictly positive")
    g = crit.grad_block(slab, lo, hi, z0)
    return subspace_step(g, d_mem, lambda v: L * v).increment


def cg_solve(apply_A, b, tol, maxit):
    """Conjugate gradients, best iterate on breakdown / budget (directions.py:117-149)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    b_norm = float(np.linalg.norm(b))
    if b_norm == 0.0:
        return x, True, 0, 0.0
    r = b.copy()
    p = r.copy()
    rs = float(r @ r)
    best, best_res = x.copy(), b_norm
    it = 0
    for it in range(1, maxit + 1):
        ap = apply_A(p)
        p_ap = float(p @ ap)
        if p_ap <= 0.0:
            break
        alpha = rs / p_ap
        x += alpha * p
        r -= alpha * ap
        rs_new = float(r @ r)
        res = rs_new ** 0.5
        if res < best_res:
            best, best_res = x.copy(), res
        if res <= tol * b_norm:
            return x, True, it, res / b_norm
        p = r + (rs_new / rs) * p
        rs = rs_new
    return best, False, it, best_res / b_norm


def mm_direction(crit: Criterion, slab, z0, lo, hi, cg_tol=1e-8, cg_maxit=200):
    """A_S(x) d = -g by CG (directions.py:152-168); the warning is the caller's."""
    if cg_tol <= 0:
        raise ValueError("cg_tol must be strictly positive")
    g = crit.grad_block(slab, lo, hi, z0)
    if not np.isfinite(g).all():
        raise ValueError("non-finite gradient")
    if not g.any():
        return np.zeros_like(g)
    d, _, _, _ = cg_solve(crit.majorant(slab, lo, hi, z0), -g, cg_tol, cg_maxit)
    return d


def operator_norm_bound(ker):
    """||H||_1 ||H||_inf (objective.py:322-342)."""
    nz, kz = ker.shape[0], ker.shape[1]
    rz = (kz - 1) // 2
    a = np.abs(ker)
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


def rho_hth_estimate(ker, shape, iters=50, seed=0):
    """Power iteration on H^T H, +5%, capped by the norm bound (objective.py:345-370)."""
    rng = np.random.Generator(np.random.Philox(seed))
    v = rng.uniform(0.1, 1.0, shape)
    v /= np.linalg.norm(v)
    est = prev = 0.0
    for _ in range(iters):
        w = Ht(ker, H(ker, v))
        nrm = float(np.linalg.norm(w))
        if nrm == 0.0:
            v = rng.uniform(0.1, 1.0, shape)
            v /= np.linalg.norm(v)
            continue
        prev, est = est, nrm
        v = w / nrm
    bound = operator_norm_bound(ker)
    if not (est > 0 and abs(est - prev) <= 1e-3 * est):
        return bound
    return min(1.05 * est, bound)


def lipschitz_bound(rho, lam, eta, kappa, delta):
    """rho + 2 eta + (lam/delta) 2*4 + 2 kappa 4 (objective.py:307-319)."""
    return rho + 2.0 * eta + (lam / delta) * 2.0 * 4.0 + 2.0 * kappa * 4.0
