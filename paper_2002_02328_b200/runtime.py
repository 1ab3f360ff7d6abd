"""Execution engines binding the scheduler to the fused block-step kernels
(drop-in for ``bd3mg.runtime``, reference pkg/src/bd3mg/runtime.py).

* ``simulated`` asynchronous engine: seeded discrete-event order of worker
  completions (service = base +- jitter from Philox), bitwise the reference
  interleaving; workers = 1 is the deterministic cyclic schedule.
* barrier mode (``method="bp3mg"``): all workers anchored at one iterate,
  increments applied jointly.  With workers = #blocks every cycle is one
  block-Jacobi sweep, launched as ONE batched ``bd3mg_mg_steps`` call that
  updates the iterate and the memory store in place.
* ``live`` engine: the simulated ordering replaced by real concurrency --
  each worker owns a CUDA stream, the master applies increments as workers
  finish (see ``_run_live``).

The iterate, memory directions and sweep snapshot stay on the GPU for the
whole run; per sweep one fused pass returns f(x) and the stop-rule norms.
"""

from __future__ import annotations

import csv
import ctypes as C
import heapq
import math
import queue
import threading
import time
from dataclasses import dataclass, field
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _native as N
from . import device as D
from . import directions, scheduler
from .objective import Objective, eval_terms, grad_f, lipschitz_estimate
from .volume import rel_dist as _rel_dist
from .volume import snr_db as _snr_db

METHODS = ("bd3mg", "bp3mg", "async_gd", "async_cg", "async_mm")
ENGINES = ("live", "simulated")


@dataclass(frozen=True)
class RunConfig:
    """Reference runtime.py:43-66, plus the device arithmetic type."""

    method: str = "bd3mg"
    workers: int = 1
    block_height: int = 1
    tol: float = 1e-6
    max_updates: Optional[int] = None
    seed: int = 0
    cg_tol: float = 1e-8
    cg_maxit: int = 200
    engine: str = "simulated"
    service_base: float = 1.0
    service_jitter: float = 0.3
    record_cycle_f: bool = False
    dtype: str = "f64"

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if self.engine not in ENGINES:
            raise ValueError(f"unknown engine {self.engine!r}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.tol <= 0:
            raise ValueError("tol must be strictly positive")
        if self.dtype not in ("f64", "f32"):
            raise ValueError("dtype must be 'f64' or 'f32'")

    @property
    def torch_dtype(self) -> torch.dtype:
        return torch.float64 if self.dtype == "f64" else torch.float32


class IterationLogEntry(NamedTuple):
    k: int
    wall_seconds: float
    f_value: float
    snr_db: Optional[float]
    rel_dist: Optional[float]
    max_staleness: int


@dataclass
class RunResult:
    x_final: np.ndarray
    log: list[IterationLogEntry]
    stop_reason: str
    tau_hat: int
    trace: list[scheduler.TraceEvent]
    grant_log: list[int]
    wall_seconds: float
    method: str
    workers: int
    cycle_f: list[float] = field(default_factory=list)


def compute_increment(obj: Objective, task: scheduler.TaskMessage, method: str, L: Optional[float],
                      cg_tol: float, cg_maxit: int):
    """One worker step on a task snapshot (runtime.py:92-105)."""
    z0 = task.slab.z_lo
    if method in ("bd3mg", "bp3mg"):
        return directions.mg_direction(obj, task.x_slab, z0, task.block, task.d_mem)
    if method == "async_gd":
        return directions.gd_direction(obj, task.x_slab, z0, task.block, L)
    if method == "async_cg":
        return directions.cg_direction(obj, task.x_slab, z0, task.block, task.d_mem, L)
    if method == "async_mm":
        return directions.mm_direction(obj, task.x_slab, z0, task.block, cg_tol, cg_maxit)
    raise ValueError(f"unknown method {method!r}")


# ---------------------------------------------------------------------------
class _StepLog:
    """Device record of every fused step's StepInfo.  A failed step (status
    1 = non-finite gradient, 2 = non-finite increment; nothing applied) is
    raised as the reference's ValueError / ProtocolError: before its ledger
    entry where the engine checks each step (one worker, barrier cycles),
    else at the next host sync."""

    def __init__(self, device):
        self.buf = torch.empty((256, N.INFO_DOUBLES), dtype=torch.float64, device=device)
        self.n = 0
        self.checked = 0

    def slot(self, count: int) -> torch.Tensor:
        if self.n + count > self.buf.shape[0]:
            self.check()
            if self.n + count > self.buf.shape[0]:
                self.n = self.checked = 0
            if count > self.buf.shape[0]:
                # a batch wider than the ring (e.g. a barrier cycle of > 256
                # workers): the native step writes count rows, so grow first
                self.buf = torch.empty((max(count, 2 * self.buf.shape[0]), N.INFO_DOUBLES),
                                       dtype=torch.float64, device=self.buf.device)
        out = self.buf[self.n:self.n + count]
        self.n += count
        return out

    def check(self) -> None:
        if self.n > self.checked:
            status = self.buf[self.checked:self.n, 8]
            self.checked = self.n
            scheduler.raise_step_status(status)


class _Recorder:
    """Per-sweep logging + stop decision (runtime.py:108-141): one fused
    device pass gives f(x) and ||x - snap||, ||snap||."""

    def __init__(self, obj, cfg, truth, x_star, steps: _StepLog | None = None):
        self.obj, self.cfg = obj, cfg
        self.truth = None if truth is None else np.asarray(truth, dtype=np.float64)
        self.x_star = None if x_star is None else np.asarray(x_star, dtype=np.float64)
        self.log: list[IterationLogEntry] = []
        self.stop_reason = "budget"
        self.steps = steps

    def _append(self, state, wall, snap=None):
        terms = eval_terms(self.obj, state.x, snap).cpu().numpy()
        if self.steps is not None:
            self.steps.check()
        f_val = float(terms[4])
        if not math.isfinite(f_val):
            raise ValueError("objective evaluated to a non-finite value")
        snr = rd = None
        if self.truth is not None or self.x_star is not None:
            xh = D.to_host(state.x)
            snr = _snr_db(self.truth, xh) if self.truth is not None else None
            rd = _rel_dist(xh, self.x_star) if self.x_star is not None else None
        self.log.append(IterationLogEntry(state.k, wall, f_val, snr, rd, state.tau_hat))
        return math.sqrt(max(terms[5], 0.0)), math.sqrt(max(terms[6], 0.0))

    def after_update(self, state, wall) -> bool:
        cfg = self.cfg
        if scheduler.sweep_complete(state):
            norms = self._append(state, wall, state.sweep_snapshot)
            stop = scheduler.should_stop(state, cfg.tol, cfg.max_updates, norms=norms)
            if stop:
                self.stop_reason = ("budget" if cfg.max_updates is not None and state.k >= cfg.max_updates
                                    else "tolerance")
            scheduler.roll_sweep(state)
            return stop
        if cfg.max_updates is not None and state.k >= cfg.max_updates:
            self._append(state, wall)
            self.stop_reason = "budget"
            return True
        return False


def _needs_L(method: str) -> bool:
    return method in ("async_gd", "async_cg")


def _service_sampler(cfg: RunConfig):
    rng = np.random.Generator(np.random.Philox(cfg.seed))

    def draw() -> float:
        return max(1e-9, cfg.service_base + cfg.service_jitter * (2.0 * rng.random() - 1.0))

    return draw


def _fused(method: str) -> bool:
    return method in ("bd3mg", "bp3mg")


def _rows(t: torch.Tensor, lo: int, hi: int) -> torch.Tensor:
    return t[lo:hi + 1]


def _fused_task(state, task: scheduler.TaskMessage, inc_out=None, in_place=True) -> N.Task:
    blk = task.block
    return N.Task(task.x_slab.data_ptr(), task.slab.z_lo, task.x_slab.shape[0], blk.z_lo, blk.z_hi,
                  task.d_mem.data_ptr(), D.ptr(inc_out),
                  _rows(state.x, blk.z_lo, blk.z_hi).data_ptr() if in_place else None,
                  _rows(state.prev_increment, blk.z_lo, blk.z_hi).data_ptr() if in_place else None)


def _start(obj: Objective, x0, cfg: RunConfig):
    x = D.to_device(x0, cfg.torch_dtype)
    state, tasks = scheduler.init_master(x, cfg.workers, cfg.block_height, obj.psf)
    return state, tasks


def _run_simulated(obj, x0, cfg, truth, x_star, L) -> RunResult:
    """Seeded DES (runtime.py:158-180); fused in-place block steps."""
    state, tasks = _start(obj, x0, cfg)
    steps = _StepLog(state.x.device)
    rec = _Recorder(obj, cfg, truth, x_star, steps)
    draw = _service_sampler(cfg)
    snap = cfg.workers > 1  # one worker: nothing can land between grant and compute
    if not snap:
        tasks = [scheduler.make_task(state, t.worker_id, t.block, snapshot=False) for t in tasks]
    heap, seq = [], 0
    for task in tasks:
        heapq.heappush(heap, (draw(), seq, task))
        seq += 1
    now = 0.0
    while heap:
        now, _, task = heapq.heappop(heap)
        msg = scheduler.UpdateMessage(task.worker_id, task.block, None, task.issue_k)
        if _fused(cfg.method):
            info = directions.mg_steps_device(obj, [_fused_task(state, task)], cfg.torch_dtype,
                                              info=steps.slot(1))
            # the reference raises in the worker (ValueError) or in
            # receive_update (ProtocolError) before its ledger moves
            scheduler.raise_step_status(info[:, 8])
            steps.checked = steps.n
            scheduler.receive_applied(state, msg)
        else:
            inc = compute_increment(obj, task, cfg.method, L, cfg.cg_tol, cfg.cg_maxit)
            scheduler.receive_update(state, scheduler.UpdateMessage(task.worker_id, task.block, inc,
                                                                    task.issue_k))
        if rec.after_update(state, now):
            break
        block = scheduler.next_block(state, task.worker_id)
        heapq.heappush(heap, (now + draw(), seq, scheduler.make_task(state, task.worker_id, block, snapshot=snap)))
        seq += 1
    steps.check()
    return RunResult(D.to_host(state.x), rec.log, rec.stop_reason, state.tau_hat, state.trace,
                     state.grant_log, now, cfg.method, cfg.workers)


def run_bp3mg_barrier(obj: Objective, x0, cfg: RunConfig, truth=None, x_star=None) -> RunResult:
    """Synchronous cycles (runtime.py:244-292): every task of a cycle is
    anchored at the same iterate, so the whole cycle is one batched launch
    (residual computed once over the union of the blocks' rows)."""
    L = lipschitz_estimate(obj) if _needs_L(cfg.method) else None
    state, tasks = _start(obj, x0, cfg)
    steps = _StepLog(state.x.device)
    rec = _Recorder(obj, cfg, truth, x_star, steps)
    draw = _service_sampler(cfg)
    live = cfg.engine == "live"
    nblocks = len(state.blocks)
    t0 = time.perf_counter()
    now = 0.0
    cycle_f: list[float] = []
    stop = False
    x_full = state.x
    while not stop:
        C = len(tasks)
        # the shared anchor is the full iterate (it covers every slab)
        anchored = [scheduler.TaskMessage(t.worker_id, t.block, scheduler.SliceBlock(0, state.dims.nz - 1),
                                          x_full, t.d_mem, t.issue_k) for t in tasks]
        # in place only when the whole cycle is one launch (<= 32 tasks): with
        # more, an in-place launch would move the anchor of the next one
        fused_in_place = (_fused(cfg.method) and C == nblocks and C <= N.MAX_TASKS_IN_PLACE
                          and (cfg.max_updates is None or state.k + C <= cfg.max_updates))
        if _fused(cfg.method):
            if fused_in_place:
                directions.mg_steps_device(obj, [_fused_task(state, t) for t in anchored], cfg.torch_dtype,
                                           info=steps.slot(C))
                incs = [None] * C
            else:
                incs = [torch.empty(t.block.count(state.dims), dtype=state.x.dtype, device=state.x.device)
                        for t in anchored]
                directions.mg_steps_device(obj, [_fused_task(state, t, inc, in_place=False)
                                                 for t, inc in zip(anchored, incs)], cfg.torch_dtype,
                                           info=steps.slot(C))
        else:
            incs = [compute_increment(obj, t, cfg.method, L, cfg.cg_tol, cfg.cg_maxit) for t in tasks]
        now += max(draw() for _ in tasks)
        if live:
            torch.cuda.current_stream().synchronize()
        if _fused(cfg.method):
            # one check per cycle, before any of its ledger entries
            # (the reference's pool.map raises before receive_update)
            steps.check()
        wall = (time.perf_counter() - t0) if live else now
        for t, inc in zip(tasks, incs):
            msg = scheduler.UpdateMessage(t.worker_id, t.block, inc, t.issue_k)
            if inc is None:
                scheduler.receive_applied(state, msg)
            elif _fused(cfg.method):
                blk = t.block
                N.check(N.lib.bd3mg_apply_increment(D.DTYPES[state.x.dtype],
                                                    _rows(state.x, blk.z_lo, blk.z_hi).data_ptr(),
                                                    _rows(state.prev_increment, blk.z_lo, blk.z_hi).data_ptr(),
                                                    inc.data_ptr(), inc.numel(), D.stream_handle()))
                scheduler.receive_applied(state, msg)
            else:
                scheduler.receive_update(state, msg)
            if rec.after_update(state, wall):
                stop = True
        if cfg.record_cycle_f:
            cycle_f.append(float(eval_terms(obj, state.x)[4].item()))
        if stop:
            break
        tasks = [scheduler.make_task(state, c, scheduler.next_block(state, c), snapshot=False)
                 for c in range(1, cfg.workers + 1)]
    steps.check()
    wall = (time.perf_counter() - t0) if live else now
    return RunResult(D.to_host(state.x), rec.log, rec.stop_reason, state.tau_hat, state.trace,
                     state.grant_log, wall, cfg.method, cfg.workers, cycle_f)


class _WorkerFailure(NamedTuple):
    worker_id: int
    error: BaseException


def _run_live(obj, x0, cfg, truth, x_star, L) -> RunResult:
    """Live asynchronous engine (runtime.py:188-241): C worker threads, each
    with its own CUDA stream, exchange immutable snapshots with the master
    through FIFO queues; the master applies increments in arrival order."""
    state, tasks = _start(obj, x0, cfg)
    rec = _Recorder(obj, cfg, truth, x_star)
    dev = state.x.device
    master_stream = torch.cuda.current_stream(dev)
    inboxes = {c: queue.Queue() for c in range(1, cfg.workers + 1)}
    outbox: queue.Queue = queue.Queue()

    def worker(c):
        stream = torch.cuda.Stream(dev)
        while True:
            item = inboxes[c].get()
            if item is None:
                return
            task, ready = item
            try:
                with torch.cuda.stream(stream):
                    stream.wait_event(ready)
                    if _fused(cfg.method):
                        inc = torch.empty(task.block.count(state.dims), dtype=state.x.dtype, device=dev)
                        info = directions.mg_steps_device(
                            obj, [N.Task(task.x_slab.data_ptr(), task.slab.z_lo, task.x_slab.shape[0],
                                         task.block.z_lo, task.block.z_hi, task.d_mem.data_ptr(),
                                         inc.data_ptr(), None, None)], cfg.torch_dtype, stream=stream)
                        scheduler.raise_step_status(info[:, 8])
                    else:
                        inc = compute_increment(obj, task, cfg.method, L, cfg.cg_tol, cfg.cg_maxit)
                    done = torch.cuda.Event()
                    done.record(stream)
                outbox.put((scheduler.UpdateMessage(task.worker_id, task.block, inc, task.issue_k), done))
            except BaseException as exc:  # surfaced by the master as an abort
                outbox.put(_WorkerFailure(c, exc))
                return

    def send(task):
        ev = torch.cuda.Event()
        ev.record(master_stream)
        inboxes[task.worker_id].put((task, ev))

    threads = [threading.Thread(target=worker, args=(c,), name=f"bd3mg-worker-{c}")
               for c in range(1, cfg.workers + 1)]
    for t in threads:
        t.start()
    t0 = time.perf_counter()
    failure = None
    try:
        for task in tasks:
            send(task)
        while True:
            item = outbox.get()
            if isinstance(item, _WorkerFailure):
                failure = item
                break
            msg, done = item
            master_stream.wait_event(done)
            blk = msg.block
            if _fused(cfg.method):
                N.check(N.lib.bd3mg_apply_increment(D.DTYPES[state.x.dtype],
                                                    _rows(state.x, blk.z_lo, blk.z_hi).data_ptr(),
                                                    _rows(state.prev_increment, blk.z_lo, blk.z_hi).data_ptr(),
                                                    msg.increment.data_ptr(), msg.increment.numel(),
                                                    D.stream_handle(master_stream)))
                scheduler.receive_applied(state, msg)
            else:
                scheduler.receive_update(state, msg)
            if rec.after_update(state, time.perf_counter() - t0):
                break
            block = scheduler.next_block(state, msg.worker_id)
            send(scheduler.make_task(state, msg.worker_id, block))
    finally:
        for q in inboxes.values():
            q.put(None)
        for t in threads:
            t.join()
    if failure is not None:
        raise RuntimeError(f"worker {failure.worker_id} aborted at master iteration {state.k}") from failure.error
    wall = time.perf_counter() - t0
    return RunResult(D.to_host(state.x), rec.log, rec.stop_reason, state.tau_hat, state.trace,
                     state.grant_log, wall, cfg.method, cfg.workers)


def run(obj: Objective, x0, cfg: RunConfig, truth=None, x_star=None) -> RunResult:
    """Execute the configured method to its stopping rule (runtime.py:295-301)."""
    if cfg.method == "bp3mg":
        return run_bp3mg_barrier(obj, x0, cfg, truth, x_star)
    L = lipschitz_estimate(obj) if _needs_L(cfg.method) else None
    engine = _run_live if cfg.engine == "live" else _run_simulated
    return engine(obj, x0, cfg, truth, x_star, L)


def stationarity(obj: Objective, x, ref_grad_norm: Optional[float] = None) -> float:
    g = grad_f(obj, x)
    norm = float(torch.linalg.vector_norm(g).item()) if D.is_tensor(g) else float(np.linalg.norm(g))
    return norm if ref_grad_norm is None else norm / (1.0 + ref_grad_norm)


def write_log_csv(log: list[IterationLogEntry], sink) -> None:
    def fmt(v):
        return "" if v is None else repr(v)

    close = False
    if not hasattr(sink, "write"):
        sink, close = open(sink, "w", newline=""), True
    try:
        w = csv.writer(sink)
        w.writerow(["k", "wall_seconds", "f", "snr_db", "rel_dist", "max_staleness"])
        for e in log:
            w.writerow([e.k, repr(e.wall_seconds), repr(e.f_value), fmt(e.snr_db), fmt(e.rel_dist),
                        e.max_staleness])
    finally:
        if close:
            sink.close()


# ---------------------------------------------------------------------------
class JacobiSweeper:
    """Device-resident block-Jacobi driver: ``run_bp3mg_barrier`` with
    workers = #blocks, every cycle one sweep (runtime.py:244-292).

    One sweep = ONE ``bd3mg_jacobi_sweep`` call: the recorder pass of the
    anchor x_k (f(x_k) and the stop-rule norms against the previous
    snapshot, runtime.py:120 / scheduler.py:208-219 -- its data term is the
    residual the block steps compute anyway), the snapshot roll, and the
    fused steps of all blocks at the anchor with the in-place update.  The
    recorder of sweep k's result therefore runs at the start of sweep k+1;
    ``finish()`` records the last one.  All buffers are preallocated and all
    launches go to the current stream, so a sweep can be a CUDA graph.

    ``hd_cache=True`` selects the "hd-cache" variant: H E_S d_mem is kept
    from each block's previous visit (linearity of H) so the Gram needs one
    forward correlation instead of two.  ``incremental=True`` (implies
    hd_cache) selects "hd-incremental": the residual r = H x - y is kept on
    the device as well, r += sum_b H E_b inc_b, so the sweep runs no residual
    correlation; it is recomputed exactly on the first sweep and every
    ``refresh_every`` sweeps (0: never again).
    """

    def __init__(self, obj: Objective, x0, block_height: int, dtype: torch.dtype = torch.float64,
                 blocks: list | None = None, hd_cache: bool = False, incremental: bool = False,
                 refresh_every: int = 0):
        hd_cache = hd_cache or incremental
        self.obj = obj
        self.dtype = dtype
        self.x = D.to_device(x0, dtype).clone()
        self.prev = torch.zeros_like(self.x)
        self.snap = self.x.clone()
        dims = obj.dims
        self.blocks = blocks or scheduler.partition_blocks(dims.nz, block_height)
        self._barr = (C.c_int64 * (2 * len(self.blocks)))(*[v for b in self.blocks for v in (b.z_lo, b.z_hi)])
        self.geom = obj.geom(dtype)
        self.reg = D.reg(obj.params)
        self.sw = N.Sweep(self.x.data_ptr(), self.prev.data_ptr(), 0, dims.nz, self._barr, len(self.blocks),
                          0, dims.nz - 1, self.snap.data_ptr(), None)
        dev = self.x.device
        self.hd = None
        if hd_cache:
            n = N.lib.bd3mg_jacobi_cache_elems(D.byref(self.geom), D.byref(self.sw))
            self.hd = torch.zeros(n, dtype=dtype, device=dev)
            self.sw.hd_cache = self.hd.data_ptr()
        self.ws_bytes = N.ws_bytes(N.lib.bd3mg_jacobi_sweep_ws_bytes(D.byref(self.geom), D.byref(self.sw)))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.eval_bytes = N.ws_bytes(N.lib.bd3mg_eval_f_ws_bytes(D.byref(self.geom)))
        self.ews = torch.empty(self.eval_bytes, dtype=torch.uint8, device=dev)
        self.info = torch.empty((len(self.blocks), N.INFO_DOUBLES), dtype=torch.float64, device=dev)
        self.terms = torch.empty(N.EVAL_DOUBLES, dtype=torch.float64, device=dev)
        self.K = obj.psf.device_kernels(dtype, dev)
        self.Y = obj.device_y(dtype, dev)
        self.k = 0
        self.sweeps = 0
        self.graph = None
        self.graphs = {}
        self.refresh_every = refresh_every
        self.resid = torch.zeros_like(self.x) if incremental else None

    @property
    def nblocks(self) -> int:
        return len(self.blocks)

    def _refresh_due(self) -> bool:
        return self.sweeps == 0 or (self.refresh_every > 0 and self.sweeps % self.refresh_every == 0)

    def _launch(self, refresh: bool = False) -> None:
        if self.resid is not None:
            N.check(N.lib.bd3mg_jacobi_sweep_incremental(
                D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(), self.Y.data_ptr(), D.byref(self.sw),
                self.resid.data_ptr(), int(refresh), self.terms.data_ptr(), self.info.data_ptr(),
                self.ws.data_ptr(), self.ws_bytes, D.stream_handle()))
            return
        N.check(N.lib.bd3mg_jacobi_sweep(D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(),
                                         self.Y.data_ptr(), D.byref(self.sw), self.terms.data_ptr(),
                                         self.info.data_ptr(), self.ws.data_ptr(), self.ws_bytes,
                                         D.stream_handle()))

    def capture(self) -> None:
        """Record the sweep as a CUDA graph (after one eager warm-up sweep);
        the incremental variant records its refresh sweep too."""
        for refresh in ((False, True) if self.resid is not None else (False,)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch(refresh)
            self.graphs[refresh] = g
        self.graph = self.graphs[False]

    def sweep(self) -> None:
        refresh = self.resid is not None and self._refresh_due()
        if self.graphs:
            self.graphs[refresh].replay()
        else:
            self._launch(refresh)
        self.sweeps += 1
        self.k += len(self.blocks)

    def finish(self) -> float:
        """Recorder pass of the current iterate (the last sweep's log entry)."""
        N.check(N.lib.bd3mg_eval_f(D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(), self.Y.data_ptr(),
                                   self.x.data_ptr(), self.snap.data_ptr(), self.terms.data_ptr(),
                                   self.ews.data_ptr(), self.eval_bytes, D.stream_handle()))
        return self.f()

    def check(self) -> None:
        scheduler.raise_step_status(self.info[:, 8])

    def f(self) -> float:
        """f of the anchor recorded by the last sweep (or by finish())."""
        return float(self.terms[4].item())


class CyclicSweeper:
    """Device-resident deterministic cyclic schedule (reference bd3mg with one
    worker: blocks 0..B-1 in order, each step seeing every earlier update,
    runtime.py:158-180) followed by the per-sweep recorder.  One fused
    ``bd3mg_mg_steps`` launch set per block (in place); capturable as a
    CUDA graph like JacobiSweeper.

    ``incremental=True`` selects the "hd-incremental" variant of the same
    schedule: each block keeps H E_S d_mem from its previous visit and the
    residual r = H x - y is kept on the device by linearity
    (bd3mg_mg_steps_incremental), so no step runs a residual correlation and
    the recorder takes its data term from r (bd3mg_eval_f_resid); r is
    recomputed exactly on the first sweep and every ``refresh_every``
    sweeps (0: never again)."""

    def __init__(self, obj: Objective, x0, block_height: int, dtype: torch.dtype = torch.float64,
                 incremental: bool = False, refresh_every: int = 0):
        self.obj, self.dtype = obj, dtype
        self.x = D.to_device(x0, dtype).clone()
        self.prev = torch.zeros_like(self.x)
        self.snap = self.x.clone()
        dims = obj.dims
        self.blocks = scheduler.partition_blocks(dims.nz, block_height)
        self.geom = obj.geom(dtype)
        self.reg = D.reg(obj.params)
        self.tasks = [(N.Task * 1)(N.Task(self.x.data_ptr(), 0, dims.nz, b.z_lo, b.z_hi,
                                          _rows(self.prev, b.z_lo, b.z_hi).data_ptr(), None,
                                          _rows(self.x, b.z_lo, b.z_hi).data_ptr(),
                                          _rows(self.prev, b.z_lo, b.z_hi).data_ptr())) for b in self.blocks]
        self.ws_bytes = max(N.ws_bytes(N.lib.bd3mg_mg_steps_ws_bytes(D.byref(self.geom), t, 1)) for t in self.tasks)
        dev = self.x.device
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.eval_bytes = N.ws_bytes(N.lib.bd3mg_eval_f_ws_bytes(D.byref(self.geom)))
        self.ews = torch.empty(self.eval_bytes, dtype=torch.uint8, device=dev)
        self.info = torch.empty((len(self.blocks), N.INFO_DOUBLES), dtype=torch.float64, device=dev)
        self.terms = torch.empty(N.EVAL_DOUBLES, dtype=torch.float64, device=dev)
        self.K = obj.psf.device_kernels(dtype, dev)
        self.Y = obj.device_y(dtype, dev)
        self.k = 0
        self.sweeps = 0
        self.graph = None
        self.graphs = {}
        self.refresh_every = refresh_every
        self.resid = None
        if incremental:
            rz = (obj.psf.kdims.kz - 1) // 2
            plane = dims.ny * dims.nx
            rows = [min(dims.nz - 1, b.z_hi + rz) - max(0, b.z_lo - rz) + 1 for b in self.blocks]
            self.hd = torch.zeros(sum(rows) * plane, dtype=dtype, device=dev)
            offs = np.cumsum([0] + rows[:-1]) * plane
            esz = self.hd.element_size()
            self._hd = [(C.c_void_p * 1)(self.hd.data_ptr() + int(o) * esz) for o in offs]
            self.resid = torch.zeros_like(self.x)
            self.ws_bytes = max(N.ws_bytes(N.lib.bd3mg_mg_steps_incremental_ws_bytes(D.byref(self.geom), t, 1))
                                for t in self.tasks)
            self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)

    @property
    def nblocks(self) -> int:
        return len(self.blocks)

    def _refresh_due(self) -> bool:
        return self.sweeps == 0 or (self.refresh_every > 0 and self.sweeps % self.refresh_every == 0)

    def _launch(self, refresh: bool = False) -> None:
        s = D.stream_handle()
        if self.resid is not None and refresh:  # r = H x - y exactly (the device H, then minus y)
            from .blur import correlate_rows
            correlate_rows(self.obj.psf, self.x, 0, 0, self.obj.dims.nz - 1, False, out=self.resid)
            self.resid.sub_(self.Y)
        for i, t in enumerate(self.tasks):
            if self.resid is not None:
                N.check(N.lib.bd3mg_mg_steps_incremental(
                    D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(), self.Y.data_ptr(), t, 1, self._hd[i],
                    self.resid.data_ptr(), self.info[i].data_ptr(), self.ws.data_ptr(), self.ws_bytes, s))
            else:
                N.check(N.lib.bd3mg_mg_steps(D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(),
                                             self.Y.data_ptr(), t, 1, self.info[i].data_ptr(), self.ws.data_ptr(),
                                             self.ws_bytes, s))
        if self.resid is not None:
            N.check(N.lib.bd3mg_eval_f_resid(D.byref(self.geom), D.byref(self.reg), self.resid.data_ptr(),
                                             self.x.data_ptr(), self.snap.data_ptr(), self.terms.data_ptr(),
                                             self.ews.data_ptr(), self.eval_bytes, s))
        else:
            N.check(N.lib.bd3mg_eval_f(D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(), self.Y.data_ptr(),
                                       self.x.data_ptr(), self.snap.data_ptr(), self.terms.data_ptr(),
                                       self.ews.data_ptr(), self.eval_bytes, s))
        self.snap.copy_(self.x)

    def capture(self) -> None:
        for refresh in ((False, True) if self.resid is not None else (False,)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch(refresh)
            self.graphs[refresh] = g
        self.graph = self.graphs[False]

    def sweep(self) -> None:
        refresh = self.resid is not None and self._refresh_due()
        if self.graphs:
            self.graphs[refresh].replay()
        else:
            self._launch(refresh)
        self.sweeps += 1
        self.k += len(self.blocks)

    def check(self) -> None:
        scheduler.raise_step_status(self.info[:, 8])

    def f(self) -> float:
        """f after the last sweep (the reference's per-sweep log value)."""
        return float(self.terms[4].item())
