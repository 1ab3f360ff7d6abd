"""Multi-GPU block-Jacobi over z-slabs (one process per GPU).

Layout: the B blocks are split into P contiguous
ranges, rank p owns the planes of its blocks.  Each rank keeps a local slab
= its owned planes plus kz halo planes per side (the reference's
slab_support reach, blur.py:190-198), clamped to the volume.  Blocks never
span ranks, so a sweep is:

  1. halo exchange -- every rank receives the halo planes it does not own
     from their owners (torch.distributed P2P, NCCL over NVLink on GPUs,
     grouped in one batch_isend_irecv); halos can span several ranks when a
     rank owns fewer than kz planes;
  2. ONE bd3mg_jacobi_sweep over the owned blocks: recorder pass of the
     anchor on owned rows (f terms + stop-rule norms), then the fused block
     steps at the common anchor (in place);
  3. ONE all-reduce of the 7 recorder terms.

Per-block arithmetic is identical to the single-GPU sweep (same rows, same
fixed reduction trees), so the iterate is bitwise independent of P.  As on
one GPU, the recorder pass of sweep k's result runs at the start of sweep
k+1 (after the halo exchange makes x_k current on every rank); ``finish()``
evaluates the last one.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .volume import SliceBlock


@dataclass(frozen=True)
class SlabLayout:
    """Block ownership and halo plan for `world` ranks."""

    nz: int
    kz: int
    blocks: tuple
    world: int

    @staticmethod
    def build(nz: int, kz: int, block_height: int, world: int) -> "SlabLayout":
        blocks = tuple(SliceBlock(lo, min(lo + block_height - 1, nz - 1)) for lo in range(0, nz, block_height))
        if world > len(blocks):
            raise ValueError(f"{world} ranks for {len(blocks)} blocks: every rank needs a block")
        return SlabLayout(nz, kz, blocks, world)

    def owned_blocks(self, rank: int) -> list[SliceBlock]:
        B, P = len(self.blocks), self.world
        lo = (rank * B) // P
        hi = ((rank + 1) * B) // P
        return list(self.blocks[lo:hi])

    def owned(self, rank: int) -> tuple[int, int]:
        ob = self.owned_blocks(rank)
        return ob[0].z_lo, ob[-1].z_hi

    def local(self, rank: int) -> tuple[int, int]:
        o_lo, o_hi = self.owned(rank)
        return max(0, o_lo - self.kz), min(self.nz - 1, o_hi + self.kz)

    def transfers(self, rank: int):
        """(peer, lo, hi, 'recv'|'send') plane ranges for this rank."""
        out = []
        me_lo, me_hi = self.owned(rank)
        l_lo, l_hi = self.local(rank)
        for q in range(self.world):
            if q == rank:
                continue
            q_lo, q_hi = self.owned(q)
            ql_lo, ql_hi = self.local(q)
            # what I need from q: my local range minus my owned range, within q's owned
            for a, b in ((l_lo, me_lo - 1), (me_hi + 1, l_hi)):
                lo, hi = max(a, q_lo), min(b, q_hi)
                if lo <= hi:
                    out.append((q, lo, hi, "recv"))
            for a, b in ((ql_lo, q_lo - 1), (q_hi + 1, ql_hi)):
                lo, hi = max(a, me_lo), min(b, me_hi)
                if lo <= hi:
                    out.append((q, lo, hi, "send"))
        return out


def exchange_halos(buf: torch.Tensor, z0: int, plan, group=None) -> None:
    """Fill the halo planes of the local slab `buf` (plane 0 = depth z0)."""
    ops = []
    for peer, lo, hi, kind in plan:
        view = buf[lo - z0:hi - z0 + 1]
        if kind == "send":
            ops.append(dist.P2POp(dist.isend, view, peer, group))
        else:
            ops.append(dist.P2POp(dist.irecv, view, peer, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


class _RawDevice:
    """A raw device allocation seen by torch (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, n: int, dtype: torch.dtype):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8" if dtype == torch.float64 else "<f4",
                                         "data": (ptr, False), "strides": None, "version": 3}


class PeerHalo:
    """Halo exchange by NVLink peer stores, fused into the sweep's update.

    Every rank owns a halo INBOX: its received halo planes (the "recv" plan
    of SlabLayout.transfers, in plan order), twice -- one copy per sweep
    parity.  Sweep t of a rank (1) copies inbox[t % 2] into the halo planes
    of its local slab (a device-local copy), (2) runs the fused sweep
    (``bd3mg_jacobi_sweep_mirrored``) whose in-place update stores the
    updated rows each neighbour keeps as halo straight into that neighbour's
    inbox[(t + 1) % 2] -- mapped into this process with cudaIpc, so the
    stores go over NVLink while the update streams through HBM, and no
    ncclSend/Recv is left on the sweep's critical path.  (3) The recorder
    all-reduce that ends every sweep is the only synchronisation: a rank
    enters sweep t + 1 (reading inbox[(t + 1) % 2]) only after every rank's
    sweep t work -- its peer stores included -- completed, and no rank can
    write inbox[t % 2] again (sweep t + 1) before every rank finished
    reading it (sweep t).  The iterate is bitwise that of the NCCL-halo
    path.  Peer pointers come from ``connect_ipc`` (one process per GPU) or
    ``connect`` (virtual ranks of one process)."""

    def __init__(self, shard: "ShardedJacobi"):
        import ctypes as C

        from . import _native as N
        self.N, self.C = N, C
        self.shard = shard
        lay, me = shard.layout, shard.rank
        self.recv = [(q, lo, hi) for q, lo, hi, k in lay.transfers(me) if k == "recv"]
        self.send = [(q, lo, hi) for q, lo, hi, k in lay.transfers(me) if k == "send"]
        self.nplanes = sum(hi - lo + 1 for _, lo, hi in self.recv)
        self.plane = shard.plane
        self.esz = shard.x.element_size()
        n = max(1, 2 * self.nplanes * self.plane)
        ptr, self.handle = C.c_void_p(), (C.c_ubyte * N.IPC_HANDLE_BYTES)()
        from . import device as D
        D.bind(shard.x.device.index)
        # a failed allocation is reported by connect_ipc on EVERY rank (after
        # the handle exchange), so no rank is left waiting in a collective
        self.alloc_error = None
        if N.lib.bd3mg_peer_alloc(n * self.esz, C.byref(ptr), self.handle) != N.BD3MG_OK:
            self.alloc_error = (N.lib.bd3mg_last_error() or b"").decode() or "peer allocation failed"
            if not dist.is_initialized():
                raise RuntimeError(self.alloc_error)
            n = max(1, 2 * self.nplanes * self.plane)
            self.fallback = torch.empty(n, dtype=shard.x.dtype, device=shard.x.device)  # keeps the layout valid
            ptr = C.c_void_p(self.fallback.data_ptr())
        self.ptr = ptr.value
        self.opened: list[int] = []
        dims = shard.x.shape[1:]
        self.inbox = torch.as_tensor(_RawDevice(self.ptr, n, shard.x.dtype), device=shard.x.device)
        self.inbox = self.inbox[:2 * self.nplanes * self.plane].view(2, self.nplanes, *dims)
        self.slots = []  # (inbox plane offset, x plane offset, count) per received range
        off = 0
        for _, lo, hi in self.recv:
            self.slots.append((off, lo - shard.l_lo, hi - lo + 1))
            off += hi - lo + 1
        for o, xo, c in self.slots:  # parity 0 = the initial iterate's halos
            self.inbox[0, o:o + c].copy_(shard.x[xo:xo + c])
        self.mirrors = None

    @staticmethod
    def inbox_offset(layout: SlabLayout, rank: int, src: int, lo: int, hi: int) -> tuple[int, int]:
        """(plane offset of src's range [lo, hi] in rank's inbox, planes per parity)."""
        off, total, at = 0, 0, None
        for q, a, b, k in layout.transfers(rank):
            if k != "recv":
                continue
            if (q, a, b) == (src, lo, hi):
                at = total
            total += b - a + 1
        if at is None:
            raise ValueError(f"rank {rank} receives no planes [{lo}, {hi}] from rank {src}")
        return at, total

    def connect(self, bases: dict) -> None:
        """bases[q] = device address of rank q's inbox (mapped here) for every
        rank this one sends to; builds the mirror lists of both parities."""
        N, C = self.N, self.C
        lay, me = self.shard.layout, self.shard.rank
        self.mirrors = []
        for parity in (0, 1):
            arr = (N.Mirror * max(1, len(self.send)))()
            for i, (q, lo, hi) in enumerate(self.send):
                off, total = self.inbox_offset(lay, q, me, lo, hi)
                arr[i] = N.Mirror(lo, hi, bases[q] + (parity * total + off) * self.plane * self.esz)
            self.mirrors.append(arr)

    def connect_ipc(self, group=None) -> None:
        """One process per GPU: exchange the inbox cudaIpc handles, map the
        inboxes of the ranks this one sends to (NVLink peer access)."""
        N, C = self.N, self.C
        world = dist.get_world_size(group)
        handles = [None] * world
        dist.all_gather_object(handles, None if self.alloc_error else bytes(self.handle), group=group)
        if any(h is None for h in handles):
            raise RuntimeError(f"p2p halos: peer allocation failed on rank(s) "
                               f"{[q for q, h in enumerate(handles) if h is None]}")
        bases = {}
        for q in sorted({q for q, _, _ in self.send}):
            ptr = C.c_void_p()
            buf = (C.c_ubyte * N.IPC_HANDLE_BYTES).from_buffer_copy(handles[q])
            N.check(N.lib.bd3mg_peer_open(buf, C.byref(ptr)))
            bases[q] = ptr.value
            self.opened.append(ptr.value)
        self.connect(bases)

    def unpack(self, parity: int) -> None:
        """Halo planes of the local slab <- inbox[parity] (device-local copies)."""
        for o, xo, c in self.slots:
            self.shard.x[xo:xo + c].copy_(self.inbox[parity, o:o + c])

    def close(self) -> None:
        for p in self.opened:
            self.N.lib.bd3mg_peer_close(p)
        self.opened = []
        if self.ptr:
            self.inbox = None
            if self.alloc_error is None:
                self.N.lib.bd3mg_peer_free(self.ptr)
            self.ptr = 0


class ShardedJacobi:
    """GPU block-Jacobi shard of this rank: halos + one fused
    ``bd3mg_jacobi_sweep`` over the owned blocks (recorder on owned rows,
    whose 7 terms are all-reduced).

    halo="nccl": one grouped ncclSend/Recv of the halo planes per sweep.
    halo="p2p": the update kernel stores the neighbour-facing rows straight
    into the neighbours' halo inboxes over NVLink (PeerHalo); with
    ``rank``/``world`` given (virtual ranks of one process) the caller
    connects the inboxes itself."""

    def __init__(self, obj, x0, block_height: int, dtype: torch.dtype = torch.float64, group=None,
                 rank: int | None = None, world: int | None = None, hd_cache: bool = False,
                 halo: str = "nccl"):
        if halo not in ("nccl", "p2p"):
            raise ValueError(f"unknown halo transport {halo!r}")
        import ctypes as C

        from . import _native as N
        from . import device as D

        self.N, self.D = N, D
        self.obj, self.dtype, self.group = obj, dtype, group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        dims = obj.dims
        self.layout = SlabLayout.build(dims.nz, obj.psf.kdims.kz, block_height, self.world)
        self.blocks = self.layout.owned_blocks(self.rank)
        self.o_lo, self.o_hi = self.layout.owned(self.rank)
        self.l_lo, self.l_hi = self.layout.local(self.rank)
        self.plan = self.layout.transfers(self.rank)
        dev = torch.device("cuda", torch.cuda.current_device())
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        self.x = torch.from_numpy(x0[self.l_lo:self.l_hi + 1]).to(dev).to(dtype).contiguous()
        self.y = torch.from_numpy(obj.y[self.l_lo:self.l_hi + 1]).to(dev).to(dtype).contiguous()
        self.prev = torch.zeros_like(self.x)
        self.plane = dims.ny * dims.nx
        self.snap = self.x[self.o_lo - self.l_lo:self.o_hi - self.l_lo + 1].clone()
        esz = self.x.element_size()
        self.y_shift = self.y.data_ptr() - self.l_lo * self.plane * esz  # y + z*plane = row z (C ABI contract)
        self._barr = (C.c_int64 * (2 * len(self.blocks)))(*[v for b in self.blocks for v in (b.z_lo, b.z_hi)])
        self.geom = obj.geom(dtype)
        self.reg = D.reg(obj.params)
        self.sw = N.Sweep(self.x.data_ptr(), self.prev.data_ptr(), self.l_lo, self.x.shape[0], self._barr,
                          len(self.blocks), self.o_lo, self.o_hi, self.snap.data_ptr(), None)
        self.hd = None
        if hd_cache:
            n = N.lib.bd3mg_jacobi_cache_elems(D.byref(self.geom), D.byref(self.sw))
            self.hd = torch.zeros(n, dtype=dtype, device=dev)
            self.sw.hd_cache = self.hd.data_ptr()
        self.ws_bytes = N.ws_bytes(N.lib.bd3mg_jacobi_sweep_ws_bytes(D.byref(self.geom), D.byref(self.sw)))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.ev_bytes = N.ws_bytes(N.lib.bd3mg_eval_rows_ws_bytes(D.byref(self.geom), self.o_lo, self.o_hi))
        self.ews = torch.empty(self.ev_bytes, dtype=torch.uint8, device=dev)
        self.info = torch.empty((len(self.blocks), N.INFO_DOUBLES), dtype=torch.float64, device=dev)
        self.terms = torch.zeros(N.EVAL_DOUBLES, dtype=torch.float64, device=dev)
        self.K = obj.psf.device_kernels(dtype, dev)
        self.k = 0
        self.sweeps = 0
        self.halo = halo
        self.graphs = None
        self.peer = PeerHalo(self) if halo == "p2p" else None
        if self.peer is not None and rank is None:
            self.peer.connect_ipc(group)

    @property
    def nblocks(self) -> int:
        return len(self.layout.blocks)

    def _sync_terms(self) -> None:
        """Sum the recorder terms over the ranks.  On the p2p path this is
        also the sweep's synchronisation point (stream-ordered on NCCL; a
        host barrier after a device synchronise on gloo)."""
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self.terms, group=self.group)
        else:
            torch.cuda.synchronize()
            t = self.terms.cpu()
            dist.all_reduce(t, group=self.group)
            self.terms.copy_(t)

    # -- phases (sweep() runs them; a single-process emulation of several
    #    ranks drives them itself) -----------------------------------------
    def exchange(self) -> None:
        exchange_halos(self.x, self.l_lo, self.plan, self.group)

    def _launch(self, parity: int) -> None:
        N, D = self.N, self.D
        if self.peer is None:
            N.check(N.lib.bd3mg_jacobi_sweep(D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(), self.y_shift,
                                             D.byref(self.sw), self.terms.data_ptr(), self.info.data_ptr(),
                                             self.ws.data_ptr(), self.ws_bytes, D.stream_handle()))
            return
        if self.peer.mirrors is None:
            raise RuntimeError("p2p halos: inboxes not connected")
        self.peer.unpack(parity)
        mir = self.peer.mirrors[(parity + 1) % 2]
        N.check(N.lib.bd3mg_jacobi_sweep_mirrored(
            D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(), self.y_shift, D.byref(self.sw), mir,
            len(self.peer.send), self.terms.data_ptr(), self.info.data_ptr(), self.ws.data_ptr(), self.ws_bytes,
            D.stream_handle()))

    def local_sweep(self) -> None:
        """Recorder terms of the anchor on owned rows (local sums) + the fused
        steps of the owned blocks (p2p: after unpacking this sweep's inbox,
        with the neighbour-facing rows mirrored into the peers' next one)."""
        parity = self.sweeps % 2
        if self.graphs is not None:
            self.graphs[parity].replay()
        else:
            self._launch(parity)
        self.sweeps += 1
        self.k += self.nblocks

    def sweep(self) -> None:
        if self.peer is None:
            self.exchange()
        self.local_sweep()
        self._sync_terms()

    def record_local(self) -> None:
        """Recorder terms of the current iterate on owned rows (halos must be current)."""
        N, D = self.N, self.D
        off = (self.o_lo - self.l_lo) * self.plane * self.x.element_size()
        N.check(N.lib.bd3mg_eval_rows(D.byref(self.geom), D.byref(self.reg), self.K.data_ptr(),
                                      self.y.data_ptr() + off, self.x.data_ptr(), self.l_lo, self.x.shape[0],
                                      self.o_lo, self.o_hi, self.snap.data_ptr(), self.terms.data_ptr(),
                                      self.ews.data_ptr(), self.ev_bytes, D.stream_handle()))

    def finish(self) -> float:
        """Recorder pass of the last sweep's result; returns f(x)."""
        if self.peer is None:
            self.exchange()
        else:
            self.peer.unpack(self.sweeps % 2)
        self.record_local()
        self._sync_terms()
        return float(self.terms[4].item())

    def capture(self) -> None:
        """p2p halos: the inbox unpack + fused sweep of each parity become a
        CUDA graph (the recorder all-reduce stays outside).  NCCL halos stay
        eager."""
        if self.peer is None:
            return
        graphs = []
        for parity in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._launch(parity)
            graphs.append(g)
        self.graphs = graphs

    def close(self) -> None:
        self.graphs = None
        if self.peer is not None:
            self.peer.close()

    def check(self) -> None:
        from . import scheduler
        scheduler.raise_step_status(self.info[:, 8])

    def f(self) -> float:
        return float(self.terms[4].item())

    def gather(self) -> np.ndarray | None:
        """Full iterate on rank 0 (owned planes from every rank)."""
        own = self.x[self.o_lo - self.l_lo:self.o_hi - self.l_lo + 1].contiguous()
        if dist.get_backend(self.group) != "nccl":
            own = own.cpu()  # gloo moves host tensors
        if self.rank == 0:
            parts = [own]
            for q in range(1, self.world):
                lo, hi = self.layout.owned(q)
                t = torch.empty((hi - lo + 1,) + tuple(own.shape[1:]), dtype=own.dtype, device=own.device)
                dist.recv(t, q, group=self.group)
                parts.append(t)
            return torch.cat(parts).double().cpu().numpy()
        dist.send(own, 0, group=self.group)
        return None


# ---------------------------------------------------------------------------
# Asynchronous mode: stale peer halos with a bounded delay.
#
# Each rank walks its own blocks cyclically without global barriers.  After
# every block update it ships the planes each neighbour keeps as halo (the
# fixed per-pair range of SlabLayout.transfers) with version = its update
# count.  Before updating a block whose slab reaches a
# neighbour's planes, it takes the newest halo that has arrived and waits
# only if that version lags its own update count by more than `max_delay`
# (the stale-synchronous rule; BASELINE C4: max delay <= 2 block updates).
# The staleness used at every update is logged like the reference's
# TraceEvent ledger (scheduler.py:60-67, :156-160).

class TorchP2P:
    """Halo transport over torch.distributed messages: gloo (on CPU tensors,
    or through host memory when the run's group is NCCL, see __init__)."""

    def __init__(self, buf: torch.Tensor, z0: int, plan, group=None):
        self.buf, self.z0, self.group = buf, z0, group
        # NCCL runs every point-to-point op of a rank pair on one stream, so a
        # receive posted ahead of its send (this protocol keeps one posted per
        # neighbour) would block the peer's send queued behind the peer's own
        # posted receive: a deadlock.  On an NCCL group the messages therefore
        # travel over a gloo group through host memory, whose receives
        # complete on gloo's own threads.  Collective: every rank of `group`
        # builds its transport at the same point (AsyncEngine.__init__).
        self.dev = buf.device
        self.host = dist.get_backend(group) == "nccl"
        if self.host:
            ranks = dist.get_process_group_ranks(group) if group is not None else None
            self.group = dist.new_group(ranks=ranks, backend="gloo")
        self.mdev = torch.device("cpu") if self.host else self.dev
        self.recvs = {}   # peer -> (lo, hi, staging, header, [reqs])
        self.sends = {}   # peer -> (lo, hi)
        for peer, lo, hi, kind in plan:
            if kind == "recv":
                self.recvs.setdefault(peer, []).append((lo, hi))
            else:
                self.sends.setdefault(peer, []).append((lo, hi))
        self.pending = {}
        self.inflight = []
        for peer in self.recvs:
            self._post(peer)

    def _planes(self, ranges):
        return torch.cat([self.buf[lo - self.z0:hi - self.z0 + 1] for lo, hi in ranges])

    def _post(self, peer):
        shape = self._planes(self.recvs[peer]).shape
        stage = torch.empty(shape, dtype=self.buf.dtype, device=self.mdev)
        hdr = torch.zeros(1, dtype=torch.int64, device=self.mdev)
        reqs = [dist.irecv(hdr, peer, group=self.group), dist.irecv(stage, peer, group=self.group)]
        self.pending[peer] = (stage, hdr, reqs)

    def neighbours_sent_to(self):
        return list(self.sends)

    def send(self, peer, version: int):
        data = self._planes(self.sends[peer]).contiguous().to(self.mdev)
        hdr = torch.tensor([version], dtype=torch.int64, device=self.mdev)
        self.inflight.append((data, hdr, [dist.isend(hdr, peer, group=self.group),
                                          dist.isend(data, peer, group=self.group)]))
        self.inflight = [m for m in self.inflight if not all(r.is_completed() for r in m[2])]

    def _apply(self, peer, stage):
        off = 0
        for lo, hi in self.recvs[peer]:
            n = hi - lo + 1
            self.buf[lo - self.z0:hi - self.z0 + 1].copy_(stage[off:off + n])
            off += n

    DONE = -1  # version of the terminating message

    def poll(self, peer, need: int | None = None, until_done: bool = False) -> int | None:
        """Apply every halo message from `peer` that has arrived; block while
        the newest version is below `need` (or, with until_done, until the
        peer's terminating message).  Returns the newest version seen."""
        newest = None
        while peer in self.pending:
            stage, hdr, reqs = self.pending[peer]
            if not all(r.is_completed() for r in reqs):
                satisfied = need is None or (newest is not None and newest >= need)
                if satisfied and not until_done:
                    break
                for r in reqs:
                    r.wait()
            v = int(hdr.item())
            self._apply(peer, stage)
            if v == self.DONE:        # the peer has stopped: no more receives from it
                del self.pending[peer]
                break
            newest = v
            self._post(peer)
        return newest

    def finish(self):
        """End-of-run protocol: send a terminating copy of the halo planes to
        every neighbour, drain every neighbour up to its terminator (so every
        posted receive is matched), then complete the sends."""
        for peer in self.sends:
            self.send(peer, self.DONE)
        for peer in list(self.pending):
            self.poll(peer, until_done=True)
        for data, hdr, reqs in self.inflight:
            for r in reqs:
                r.wait()
        self.inflight = []


class AsyncShard:
    """One rank of the asynchronous block schedule.  `step_fn(shard, block)`
    updates x / prev of the block in place from the local slab (fused CUDA
    step on GPUs; the oracle in CPU tests)."""

    def __init__(self, layout: SlabLayout, rank: int, x_local: torch.Tensor, prev_local: torch.Tensor, transport,
                 step_fn, max_delay: int = 2):
        self.layout, self.rank = layout, rank
        self.x, self.prev = x_local, prev_local
        self.blocks = layout.owned_blocks(rank)
        self.o_lo, self.o_hi = layout.owned(rank)
        self.l_lo, self.l_hi = layout.local(rank)
        self.net = transport
        self.step_fn = step_fn
        self.max_delay = max_delay
        self.t = 0                      # local block updates
        self.version = {q: 0 for q in {p for p, _, _, k in layout.transfers(rank) if k == "recv"}}
        self.recv_ranges = {}
        for p, lo, hi, k in layout.transfers(rank):
            if k == "recv":
                self.recv_ranges.setdefault(p, []).append((lo, hi))
        self.send_ranges = {}
        for p, lo, hi, k in layout.transfers(rank):
            if k == "send":
                self.send_ranges.setdefault(p, []).append((lo, hi))
        self.staleness: list[int] = []  # per update: max over used halos of (t - version)
        self.waits = 0
        self.infos: list = []

    def _needs(self, block):
        s_lo = max(0, block.z_lo - self.layout.kz)
        s_hi = min(self.layout.nz - 1, block.z_hi + self.layout.kz)
        return [q for q, rs in self.recv_ranges.items() if any(lo <= s_hi and hi >= s_lo for lo, hi in rs)]

    def update(self) -> None:
        bi = self.t % len(self.blocks)
        block = self.blocks[bi]
        stale = 0
        lazy = getattr(self.net, "lazy", False)  # peer rings: read only the peers this block needs
        if not lazy:
            for q in self.recv_ranges:
                v = self.net.poll(q)
                if v is not None:
                    self.version[q] = v
        for q in self._needs(block):
            need = self.t - self.max_delay
            if lazy:
                self.version[q] = self.net.poll(q)
            if self.version[q] < need:
                self.waits += 1
                v = self.net.poll(q, need)
                if v is not None:
                    self.version[q] = v
            stale = max(stale, max(0, self.t - self.version[q]))
        self.staleness.append(stale)
        if lazy:
            # the update kernel stores the neighbour-facing rows into the
            # peers' rings; the publish that follows it on the stream makes
            # them (and the update count t+1) visible
            self.step_fn(self, block, self.net.mirrors_for(bi, self.t))
            self.t += 1
            self.net.publish(bi, self.t)
            return
        self.step_fn(self, block)
        self.t += 1
        # every update publishes the neighbour-facing planes with version t,
        # so a version always equals the sender's update count
        for q in self.send_ranges:
            self.net.send(q, self.t)

    def run(self, sweeps: int) -> None:
        for _ in range(sweeps * len(self.blocks)):
            self.update()
        self.net.finish()


class LocalP2P:
    """In-process transport between the AsyncShards of one process (several
    virtual ranks on one device): the same message discipline as TorchP2P,
    without blocking -- the driver's schedule must respect the delay bound."""

    def __init__(self, mailbox: dict, me: int, buf: torch.Tensor, z0: int, plan):
        self.box, self.me, self.buf, self.z0 = mailbox, me, buf, z0
        self.recvs, self.sends = {}, {}
        for peer, lo, hi, kind in plan:
            (self.recvs if kind == "recv" else self.sends).setdefault(peer, []).append((lo, hi))

    def send(self, peer, version: int):
        data = torch.cat([self.buf[lo - self.z0:hi - self.z0 + 1] for lo, hi in self.sends[peer]]).clone()
        self.box.setdefault((self.me, peer), []).append((version, data))

    def poll(self, peer, need: int | None = None) -> int | None:
        q = self.box.get((peer, self.me), [])
        newest = None
        while q:
            v, data = q.pop(0)
            off = 0
            for lo, hi in self.recvs[peer]:
                n = hi - lo + 1
                self.buf[lo - self.z0:hi - self.z0 + 1].copy_(data[off:off + n])
                off += n
            newest = v
        if need is not None and (newest is None or newest < need):
            raise RuntimeError("virtual schedule violated the delay bound (would block)")
        return newest

    def finish(self):
        pass


class RingPlan:
    """Units of the asynchronous peer halo rings.

    A unit is the rows one writer block contributes to one reader's halo:
    (writer, reader, writer-block index, z_lo, z_hi).  A block update
    changes exactly its own rows, so each unit carries its own data version
    (the writer's update count when the rows were last written) and its own
    ring of `slots` copies in the READER's memory; slot v % slots holds data
    version v (slot 0 = the initial iterate).  Flag words (int64, host
    memory every rank maps): dv[u] per unit, then count[p] per writer (p's
    completed updates -- the version the bounded-delay rule reads)."""

    def __init__(self, layout: SlabLayout, slots: int):
        self.layout, self.slots = layout, slots
        self.units = []
        for p in range(layout.world):
            blocks = layout.owned_blocks(p)
            for q, lo, hi, kind in layout.transfers(p):
                if kind != "send":
                    continue
                for bi, b in enumerate(blocks):
                    a, c = max(lo, b.z_lo), min(hi, b.z_hi)
                    if a <= c:
                        self.units.append((p, q, bi, a, c))
        self.offset = []                       # unit -> plane offset in the reader's ring
        self.ring_planes = [0] * layout.world  # ring size (planes) per reader
        for p, q, bi, a, c in self.units:
            self.offset.append(self.ring_planes[q])
            self.ring_planes[q] += slots * (c - a + 1)
        self.nflags = len(self.units) + layout.world

    def count_index(self, p: int) -> int:
        return len(self.units) + p

    def writes(self, p: int, bi: int) -> list[int]:
        return [u for u, (w, _, b, _, _) in enumerate(self.units) if w == p and b == bi]

    def reads(self, q: int, p: int) -> list[int]:
        return [u for u, (w, r, _, _, _) in enumerate(self.units) if r == q and w == p]

    def slot_plane(self, u: int, version: int) -> int:
        """Plane offset of data version `version` of unit u in its reader's ring."""
        p, q, bi, a, c = self.units[u]
        return self.offset[u] + (version % self.slots) * (c - a + 1)


def _map_flags(path: str | None, nbytes: int):
    """Host flag page(s): a shared file mapping (one per job, every rank maps
    it) or an anonymous one (virtual ranks of one process), registered for
    device access.  Returns (mmap, int64 view, device address)."""
    import ctypes as C
    import mmap

    from . import _native as N
    nbytes = max(mmap.PAGESIZE, -(-nbytes // mmap.PAGESIZE) * mmap.PAGESIZE)
    if path is None:
        mm = mmap.mmap(-1, nbytes)
    else:
        import os
        fd = os.open(path, os.O_RDWR)
        try:
            mm = mmap.mmap(fd, nbytes)
        finally:
            os.close(fd)
    from . import device as D
    D.bind(torch.cuda.current_device())
    words = np.frombuffer(mm, dtype=np.int64)
    host = C.addressof(C.c_char.from_buffer(mm))
    dev = C.c_void_p()
    N.check(N.lib.bd3mg_host_register(host, nbytes, C.byref(dev)))
    return mm, words, host, dev.value


class PeerRing:
    """Asynchronous-mode halo transport over peer memory (SURVEY.md 8(e):
    "P2P stores into peer halo rings with version counters").

    Writer side: the block's update kernel stores the rows of every unit it
    feeds into slot (t+1) % slots of the reader's ring (NVLink stores into
    cudaIpc-mapped memory; ``mirrors_for``), then a one-thread publish kernel
    on the same stream stores dv[u] = t+1 and count[me] = t+1, each after a
    system-scope fence (``publish``).  Reader side (``poll``): reads count
    and dv from the host-mapped flags, spins while count < need (the
    bounded-delay rule), and copies the newest slot of each unit into its
    slab with a stream-ordered device copy.  Only the peers the current
    block needs are read (``lazy``), so a reader copies only after the
    writer satisfied the delay bound; with that, a writer can move at most
    2*max_delay + 2 updates ahead of a copy still queued on the reader's
    stream, which `slots` covers (the writer blocks on the reader in turn).
    No kernel waits on another rank: all waiting is host-side."""

    lazy = True

    def __init__(self, plan: RingPlan, rank: int, x: torch.Tensor, z0: int, ring_ptr: int, ring_bases: dict,
                 flags: np.ndarray, flags_dev: int, timeout_s: float = 120.0):
        from . import _native as N
        self.N = N
        self.plan, self.me, self.x, self.z0 = plan, rank, x, z0
        self.plane = int(np.prod(x.shape[1:]))
        self.esz = x.element_size()
        self.bases = ring_bases
        self.flags, self.flags_dev = flags, flags_dev
        self.timeout_s = timeout_s
        nring = max(1, plan.ring_planes[rank] * self.plane)
        self.ring = torch.as_tensor(_RawDevice(ring_ptr, nring, x.dtype), device=x.device)
        self.applied = {}
        for u, (p, q, bi, a, c) in enumerate(plan.units):
            if q == rank:  # slot 0 of my rings = the initial iterate's rows
                off = plan.slot_plane(u, 0) * self.plane
                self.ring[off:off + (c - a + 1) * self.plane].copy_(x[a - z0:c - z0 + 1].reshape(-1))
                self.applied[u] = 0
        self.reads = {p: plan.reads(rank, p) for p in range(plan.layout.world)}
        self.writes = [plan.writes(rank, bi) for bi in range(len(plan.layout.owned_blocks(rank)))]

    def mirrors_for(self, bi: int, t: int):
        N, plan = self.N, self.plan
        out = []
        for u in self.writes[bi]:
            p, q, _, a, c = plan.units[u]
            out.append(N.Mirror(a, c, self.bases[q] + plan.slot_plane(u, t + 1) * self.plane * self.esz))
        return out

    def publish(self, bi: int, t: int) -> None:
        from . import device as D
        N, plan = self.N, self.plan
        words = [u for u in self.writes[bi]] + [plan.count_index(self.me)]
        arr = (N.Flag * len(words))(*[N.Flag(self.flags_dev + 8 * w, t) for w in words])
        N.check(N.lib.bd3mg_publish(arr, len(words), D.stream_handle()))

    def count(self, p: int) -> int:
        return int(self.flags[self.plan.count_index(p)])

    def poll(self, p: int, need: int | None = None) -> int:
        """Newest update count of writer p (waiting while it is below
        `need`); its newest unit data is copied into the slab."""
        import time
        v = self.count(p)
        if need is not None and v < need:
            t_end = time.monotonic() + self.timeout_s
            while v < need:
                if time.monotonic() > t_end:
                    raise TimeoutError(f"rank {self.me}: writer {p} stuck at update {v} < {need}")
                time.sleep(0)
                v = self.count(p)
        for u in self.reads[p]:
            d = int(self.flags[u])
            if d > self.applied[u]:
                _, _, _, a, c = self.plan.units[u]
                off = self.plan.slot_plane(u, d) * self.plane
                self.x[a - self.z0:c - self.z0 + 1].copy_(
                    self.ring[off:off + (c - a + 1) * self.plane].view((c - a + 1,) + tuple(self.x.shape[1:])))
                self.applied[u] = d
        return v

    def finish(self) -> None:
        """Nothing is in flight between ranks once the stream drained."""
        torch.cuda.synchronize()


def ring_slots(max_delay: int) -> int:
    """Ring depth covering a writer's lead over a queued reader copy."""
    return 2 * max_delay + 6


class RingHub:
    """Rings + flags of every rank of one asynchronous job.

    ``RingHub.local(...)``: virtual ranks of one process (rings allocated
    here, flags in an anonymous mapping).  ``RingHub.ipc(...)``: one rank per
    process: a shared flag file under /dev/shm (rank 0 creates it), each
    rank's ring exported as a cudaIpc handle and mapped by its writers."""

    def __init__(self):
        self.mm = None
        self.path = None
        self.host = 0
        self.own = []
        self.opened = []

    @classmethod
    def local(cls, plan: RingPlan, xs: list, z0s: list) -> tuple["RingHub", list]:
        import ctypes as C

        from . import _native as N
        hub = cls()
        hub.mm, flags, hub.host, fdev = _map_flags(None, plan.nflags * 8)
        ptrs = []
        for q, x in enumerate(xs):
            ptr, h = C.c_void_p(), (C.c_ubyte * N.IPC_HANDLE_BYTES)()
            N.check(N.lib.bd3mg_peer_alloc(max(1, plan.ring_planes[q] * int(np.prod(x.shape[1:])))
                                           * x.element_size(), C.byref(ptr), h))
            ptrs.append(ptr.value)
            hub.own.append(ptr.value)
        bases = dict(enumerate(ptrs))
        rings = [PeerRing(plan, q, x, z0, ptrs[q], bases, flags, fdev) for q, (x, z0) in enumerate(zip(xs, z0s))]
        return hub, rings

    @classmethod
    def ipc(cls, plan: RingPlan, rank: int, x: torch.Tensor, z0: int, group=None) -> tuple["RingHub", PeerRing]:
        import ctypes as C
        import os
        import uuid

        from . import _native as N
        hub = cls()
        world = plan.layout.world
        nbytes = plan.nflags * 8
        # every failure is agreed on by all ranks before it is raised, so no
        # rank is left waiting in a collective
        msg = [None]
        if rank == 0:
            path = f"/dev/shm/bd3mg_async_{uuid.uuid4().hex}"
            try:
                fd = os.open(path, os.O_RDWR | os.O_CREAT | os.O_EXCL, 0o600)
                os.ftruncate(fd, max(4096, -(-nbytes // 4096) * 4096))
                os.close(fd)
                msg = [("ok", path)]
            except OSError as e:
                msg = [("error", f"flag page: {e}")]
        dist.broadcast_object_list(msg, src=0, group=group)
        if msg[0][0] != "ok":
            raise RuntimeError(f"async peer rings: {msg[0][1]}")
        hub.path = msg[0][1]
        ptr, h = C.c_void_p(), (C.c_ubyte * N.IPC_HANDLE_BYTES)()
        mine = None
        try:
            hub.mm, flags, hub.host, fdev = _map_flags(hub.path, nbytes)
            N.check(N.lib.bd3mg_peer_alloc(
                max(1, plan.ring_planes[rank] * int(np.prod(x.shape[1:]))) * x.element_size(), C.byref(ptr), h))
            hub.own.append(ptr.value)
            mine = bytes(h)
        except (RuntimeError, ValueError, OSError):
            mine = None
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        if any(q is None for q in handles):
            hub.close(group=None)
            raise RuntimeError(f"async peer rings: setup failed on rank(s) {[q for q, v in enumerate(handles) if v is None]}")
        bases = {rank: ptr.value}
        err = ""
        for q in sorted({q for p, q, _, _, _ in plan.units if p == rank}):
            dp = C.c_void_p()
            if N.lib.bd3mg_peer_open((C.c_ubyte * N.IPC_HANDLE_BYTES).from_buffer_copy(handles[q]),
                                     C.byref(dp)) != N.BD3MG_OK:
                err = (N.lib.bd3mg_last_error() or b"").decode() or f"cannot map rank {q}'s ring"
                break
            bases[q] = dp.value
            hub.opened.append(dp.value)
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        if any(errs):
            hub.close(group=None)
            raise RuntimeError(f"async peer rings: {next(e for e in errs if e)}")
        ring = PeerRing(plan, rank, x, z0, ptr.value, bases, flags, fdev)
        torch.cuda.synchronize()  # slot 0 of every ring written before anyone reads it
        dist.barrier(group=group)
        return hub, ring

    def close(self, group=None) -> None:
        from . import _native as N
        torch.cuda.synchronize()
        if self.path is not None and dist.is_initialized():
            dist.barrier(group=group)  # no rank still writes into a ring or a flag
        for p in self.opened:
            N.lib.bd3mg_peer_close(p)
        for p in self.own:
            N.lib.bd3mg_peer_free(p)
        self.opened, self.own = [], []
        if self.host:
            N.lib.bd3mg_host_unregister(self.host)
            self.host = 0
        if self.path is not None:
            try:
                import os
                os.unlink(self.path)
            except FileNotFoundError:
                pass
            self.path = None


def cuda_block_step(obj, dtype: torch.dtype = torch.float64):
    """Fused in-place block step on the shard's local slab (bd3mg_mg_steps;
    the observation is the device copy of the full y)."""
    from . import _native as N
    from .directions import mg_steps_device

    def step(shard: AsyncShard, block: SliceBlock, mirrors=None) -> None:
        z0 = shard.l_lo
        rows = slice(block.z_lo - z0, block.z_hi - z0 + 1)
        task = N.Task(shard.x.data_ptr(), z0, shard.x.shape[0], block.z_lo, block.z_hi,
                      shard.prev[rows].data_ptr(), None, shard.x[rows].data_ptr(), shard.prev[rows].data_ptr())
        info = mg_steps_device(obj, [task], dtype, mirrors=mirrors)
        shard.infos.append(info)

    return step


class _NoPeers:
    """Transport of a single rank (nothing to exchange)."""

    def send(self, peer, version):
        pass

    def poll(self, peer, need=None, until_done=False):
        return None

    def finish(self):
        pass


class AsyncEngine:
    """bench/runtime driver of the asynchronous mode on this rank: one
    ``sweep()`` = one pass over the rank's own blocks, no global barrier.
    halo="p2p": peer halo rings (PeerRing); "nccl": TorchP2P messages."""

    def __init__(self, obj, x0, block_height: int, dtype: torch.dtype = torch.float64, max_delay: int = 2,
                 group=None, halo: str = "p2p"):
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.layout = SlabLayout.build(obj.dims.nz, obj.psf.kdims.kz, block_height, world)
        lo, hi = self.layout.local(rank)
        dev = torch.device("cuda", torch.cuda.current_device())
        x = torch.from_numpy(np.ascontiguousarray(x0[lo:hi + 1], dtype=np.float64)).to(dev).to(dtype).contiguous()
        prev = torch.zeros_like(x)
        self.hub = None
        if world == 1:
            net = _NoPeers()
        elif halo == "p2p":
            self.hub, net = RingHub.ipc(RingPlan(self.layout, ring_slots(max_delay)), rank, x, lo, group)
        else:
            net = TorchP2P(x, lo, self.layout.transfers(rank), group)
        self.group = group
        self.shard = AsyncShard(self.layout, rank, x, prev, net, cuda_block_step(obj, dtype), max_delay)
        self.x = x
        self.nblocks_local = len(self.shard.blocks)

    @property
    def nblocks(self) -> int:
        return len(self.layout.blocks)

    def sweep(self) -> None:
        for _ in range(self.nblocks_local):
            self.shard.update()
        if len(self.shard.infos) > 4 * self.nblocks_local:
            self.shard.infos = self.shard.infos[-self.nblocks_local:]

    def capture(self) -> None:
        """Host-driven schedule (polls between launches): stays eager."""

    def check(self) -> None:
        for info in self.shard.infos:
            from . import scheduler
            scheduler.raise_step_status(info[:, 8])

    def f(self) -> float:
        return float("nan")

    def finish(self) -> None:
        self.shard.net.finish()
        if self.hub is not None:
            self.hub.close(self.group)
            self.hub = None
