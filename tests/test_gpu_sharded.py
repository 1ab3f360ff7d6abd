"""GPU side of the multi-GPU path on ONE device: P virtual ranks (local
slabs with kz halos, shifted observation rows, owned-row recorder pass)
driven in one process, halos copied between the shards' device buffers.
The iterate must equal the single-GPU block-Jacobi sweep bit for bit and the
summed recorder terms must equal the full-volume f."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _exchange(shards):
    for s in shards:
        for peer, lo, hi, kind in s.plan:
            if kind == "recv":
                src = shards[peer]
                s.x[lo - s.l_lo:hi - s.l_lo + 1].copy_(src.x[lo - src.l_lo:hi - src.l_lo + 1])


@pytest.mark.parametrize("world,cfgname", [(2, "C1"), (3, "C1"), (8, "C2")])
def test_virtual_ranks_bitwise(world, cfgname):
    from paper_2002_02328_b200 import configs, objective, runtime
    from paper_2002_02328_b200.distributed import ShardedJacobi
    cfg = configs.CONFIGS[cfgname]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    single = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64)
    shards = [ShardedJacobi(obj, x0, cfg.block_height, torch.float64, rank=r, world=world) for r in range(world)]
    sweeps = 3
    for it in range(sweeps):
        single.sweep()
        _exchange(shards)
        if it > 0:
            for s in shards:
                s.record_local()
            total = sum(s.terms for s in shards)
            assert abs(float(total[4]) - f_prev) <= 1e-12 * abs(f_prev)
            for s in shards:
                s.snap.copy_(s.x)
        for s in shards:
            s.step()
        f_prev = single.f()
    full = torch.cat([s.x[s.o_lo - s.l_lo:s.o_hi - s.l_lo + 1] for s in shards])
    assert torch.equal(full, single.x)
