"""Test infrastructure: the sharded block-Jacobi layout, halo exchange and
recorder schedule of distributed.ShardedJacobi with the CPU oracle as the
per-block step (the host-logic check of the multi-rank path over gloo).
Lives under tests/ because it executes the oracle."""

import numpy as np
import torch
import torch.distributed as dist

from paper_2002_02328_b200.distributed import SlabLayout, exchange_halos


class OracleShardedJacobi:
    """Same layout, exchange and recorder schedule with the CPU oracle as the
    per-block step -- the host-logic check of the sharded path (gloo tests).
    Test infrastructure only: the oracle module is passed in by the caller."""

    def __init__(self, oracle, crit, x0, block_height: int, group=None):
        self.O, self.crit, self.group = oracle, crit, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        nz = x0.shape[0]
        self.layout = SlabLayout.build(nz, crit.kz, block_height, self.world)
        self.blocks = self.layout.owned_blocks(self.rank)
        self.o_lo, self.o_hi = self.layout.owned(self.rank)
        self.l_lo, self.l_hi = self.layout.local(self.rank)
        self.plan = self.layout.transfers(self.rank)
        self.x = torch.from_numpy(np.ascontiguousarray(x0[self.l_lo:self.l_hi + 1], dtype=np.float64)).clone()
        self.prev = torch.zeros_like(self.x)
        self.sweeps = 0

    def sweep(self) -> None:
        exchange_halos(self.x, self.l_lo, self.plan, self.group)
        xl = self.x.numpy()
        incs = []
        for b in self.blocks:
            s_lo, s_hi = self.O.support(self.layout.nz, self.crit.kz, b.z_lo, b.z_hi)
            slab = xl[s_lo - self.l_lo:s_hi - self.l_lo + 1].copy()
            d = self.prev.numpy()[b.z_lo - self.l_lo:b.z_hi - self.l_lo + 1].ravel().copy()
            incs.append(self.O.mg_direction(self.crit, slab, s_lo, b.z_lo, b.z_hi, d))
        for b, inc in zip(self.blocks, incs):
            sl = slice(b.z_lo - self.l_lo, b.z_hi - self.l_lo + 1)
            inc = torch.from_numpy(inc.reshape((b.height,) + tuple(self.x.shape[1:])))
            self.x[sl] += inc
            self.prev[sl] = inc
        self.sweeps += 1

    def gather(self) -> np.ndarray | None:
        own = self.x[self.o_lo - self.l_lo:self.o_hi - self.l_lo + 1].contiguous()
        if self.rank == 0:
            parts = [own]
            for q in range(1, self.world):
                lo, hi = self.layout.owned(q)
                t = torch.empty((hi - lo + 1,) + tuple(own.shape[1:]), dtype=own.dtype)
                dist.recv(t, q, group=self.group)
                parts.append(t)
            return torch.cat(parts).numpy()
        dist.send(own, 0, group=self.group)
        return None
