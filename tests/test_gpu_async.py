"""Asynchronous multi-rank mode on ONE GPU: virtual ranks exchanging halo
messages in process (the TorchP2P discipline without NCCL), fused CUDA block
steps on each rank's local slab.

With a lockstep round-robin schedule and max delay 1 every rank sees its
lower neighbour's newest planes and its upper neighbour's previous ones,
i.e. the global update order (rank 0 block t, rank 1 block t, ...) run
Gauss-Seidel -- reproduced here by the oracle to 1e-10.  A seeded random
schedule bounded by max delay 2 must respect the bound and descend."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _shards(obj, x0, h, world, max_delay):
    from paper_2002_02328_b200.distributed import AsyncShard, LocalP2P, SlabLayout, cuda_block_step
    lay = SlabLayout.build(obj.dims.nz, obj.psf.kdims.kz, h, world)
    box = {}
    step = cuda_block_step(obj, torch.float64)
    shards = []
    for r in range(world):
        lo, hi = lay.local(r)
        x = torch.from_numpy(np.ascontiguousarray(x0[lo:hi + 1])).cuda()
        prev = torch.zeros_like(x)
        shards.append(AsyncShard(lay, r, x, prev, LocalP2P(box, r, x, lo, lay.transfers(r)), step, max_delay))
    return lay, shards


def _gather(shards):
    return torch.cat([s.x[s.o_lo - s.l_lo:s.o_hi - s.l_lo + 1] for s in shards]).cpu().numpy()


@pytest.fixture(scope="module")
def c1(request):
    from paper_2002_02328_b200 import configs, objective
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    return objective.Objective(psf, y, params), x0, cfg


def test_lockstep_matches_oracle_order(c1, oracle_mod):
    obj, x0, cfg = c1
    h, world, rounds = 4, 3, 4          # 6 blocks of 4 planes, 2 per rank
    lay, shards = _shards(obj, x0, h, world, max_delay=1)
    for _ in range(rounds):
        for s in shards:
            s.update()
    got = _gather(shards)
    crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, cfg.lam, cfg.eta, cfg.kappa, cfg.delta)
    x = x0.copy()
    prev = np.zeros_like(x)
    for t in range(rounds):
        for r in range(world):
            ob = lay.owned_blocks(r)
            b = ob[t % len(ob)]
            s_lo, s_hi = oracle_mod.support(crit.nz, crit.kz, b.z_lo, b.z_hi)
            inc = oracle_mod.mg_direction(crit, x[s_lo:s_hi + 1].copy(), s_lo, b.z_lo, b.z_hi,
                                          prev[b.z_lo:b.z_hi + 1].ravel().copy())
            inc = inc.reshape((b.height,) + x.shape[1:])
            x[b.z_lo:b.z_hi + 1] += inc
            prev[b.z_lo:b.z_hi + 1] = inc
    assert np.linalg.norm(got - x) <= 1e-10 * np.linalg.norm(x)
    assert all(st <= 1 for s in shards for st in s.staleness)


def test_random_schedule_bounded_delay_descends(c1):
    from paper_2002_02328_b200 import objective
    obj, x0, cfg = c1
    h, world, updates = 4, 3, 24
    lay, shards = _shards(obj, x0, h, world, max_delay=2)
    rng = np.random.default_rng(5)
    f0 = objective.eval_f(obj, x0)
    for _ in range(updates * world):
        lo = min(s.t for s in shards)
        ready = [s for s in shards if s.t - lo < 2]   # keeps every wait satisfiable
        rng.choice(ready).update()
    for s in shards:       # final halo refresh
        for q in s.recv_ranges:
            s.net.poll(q)
    x = _gather(shards)
    assert max(st for s in shards for st in s.staleness) <= 2
    assert max(s.staleness for s in shards) and objective.eval_f(obj, x) < f0
    for s in shards:
        assert not any(bool((i[:, 8] != 0).any()) for i in s.infos)


def _ring_shards(obj, x0, h, world, max_delay):
    from paper_2002_02328_b200.distributed import (AsyncShard, RingHub, RingPlan, SlabLayout, cuda_block_step,
                                                   ring_slots)
    lay = SlabLayout.build(obj.dims.nz, obj.psf.kdims.kz, h, world)
    xs, z0s = [], []
    for r in range(world):
        lo, hi = lay.local(r)
        xs.append(torch.from_numpy(np.ascontiguousarray(x0[lo:hi + 1])).cuda())
        z0s.append(lo)
    hub, rings = RingHub.local(RingPlan(lay, ring_slots(max_delay)), xs, z0s)
    step = cuda_block_step(obj, torch.float64)
    shards = [AsyncShard(lay, r, xs[r], torch.zeros_like(xs[r]), rings[r], step, max_delay) for r in range(world)]
    return lay, hub, shards


def test_peer_rings_lockstep_matches_oracle_order(c1, oracle_mod):
    """Peer halo rings (update-kernel stores into the readers' rings, flags
    published by a fenced kernel, host-side reads): the lockstep schedule
    reproduces the same Gauss-Seidel order as the message transport."""
    obj, x0, cfg = c1
    h, world, rounds = 4, 3, 4
    lay, hub, shards = _ring_shards(obj, x0, h, world, max_delay=1)
    for _ in range(rounds):
        for s in shards:
            s.update()
            torch.cuda.synchronize()  # one host thread drives every virtual rank: publish before the next reads
    got = _gather(shards)
    crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, cfg.lam, cfg.eta, cfg.kappa, cfg.delta)
    x = x0.copy()
    prev = np.zeros_like(x)
    for t in range(rounds):
        for r in range(world):
            ob = lay.owned_blocks(r)
            b = ob[t % len(ob)]
            s_lo, s_hi = oracle_mod.support(crit.nz, crit.kz, b.z_lo, b.z_hi)
            inc = oracle_mod.mg_direction(crit, x[s_lo:s_hi + 1].copy(), s_lo, b.z_lo, b.z_hi,
                                          prev[b.z_lo:b.z_hi + 1].ravel().copy())
            inc = inc.reshape((b.height,) + x.shape[1:])
            x[b.z_lo:b.z_hi + 1] += inc
            prev[b.z_lo:b.z_hi + 1] = inc
    assert np.linalg.norm(got - x) <= 1e-10 * np.linalg.norm(x)
    assert all(st <= 1 for s in shards for st in s.staleness)
    # the flags record every writer's count and the rings its newest rows
    for s in shards:
        assert s.net.count(s.rank) == rounds
    hub.close()


def test_peer_rings_random_schedule_bounded(c1):
    from paper_2002_02328_b200 import objective
    obj, x0, cfg = c1
    h, world, updates = 4, 3, 24
    lay, hub, shards = _ring_shards(obj, x0, h, world, max_delay=2)
    rng = np.random.default_rng(5)
    f0 = objective.eval_f(obj, x0)
    for _ in range(updates * world):
        lo = min(s.t for s in shards)
        ready = [s for s in shards if s.t - lo < 2]
        rng.choice(ready).update()
    torch.cuda.synchronize()
    for s in shards:  # final halo refresh
        for q in s.recv_ranges:
            s.net.poll(q)
    x = _gather(shards)
    assert max(st for s in shards for st in s.staleness) <= 2
    assert objective.eval_f(obj, x) < f0
    hub.close()


def _async_ipc_worker(rank, world, port, sweeps, out_dir):
    """Real asynchronous ranks as processes on the one GPU: rings mapped with
    cudaIpc, flags in a shared /dev/shm page; all waiting is host-side."""
    import os

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2002_02328_b200 import configs, objective
        from paper_2002_02328_b200.distributed import AsyncEngine
        cfg = configs.CONFIGS["C1"]
        psf, truth, y, x0, params = configs.make_problem(cfg)
        obj = objective.Objective(psf, y, params)
        eng = AsyncEngine(obj, x0, 4, torch.float64, max_delay=2, halo="p2p")
        for _ in range(sweeps):
            eng.sweep()
        torch.cuda.synchronize()
        st = max(eng.shard.staleness)
        sh = eng.shard
        own = sh.x[sh.o_lo - sh.l_lo:sh.o_hi - sh.l_lo + 1].cpu()
        eng.finish()
        parts = [None] * world
        dist.all_gather_object(parts, (own.numpy(), st))
        if rank == 0:
            np.save(f"{out_dir}/x.npy", np.concatenate([p[0] for p in parts]))
            np.save(f"{out_dir}/stale.npy", np.array([p[1] for p in parts]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_rings_ipc_processes(world, tmp_path, c1):
    import socket

    import torch.multiprocessing as mp

    from paper_2002_02328_b200 import objective
    obj, x0, cfg = c1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_async_ipc_worker, args=(world, port, 3, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x = np.load(tmp_path / "x.npy")
    assert x.shape == x0.shape
    assert int(np.load(tmp_path / "stale.npy").max()) <= 2
    assert objective.eval_f(obj, x) < objective.eval_f(obj, x0)


def test_peer_rings_fp32_lockstep_tracks_fp64(c1):
    """fp32 ranks on peer halo rings under the lockstep schedule track the
    fp64 ranks to fp32 rounding."""
    from paper_2002_02328_b200.distributed import AsyncShard, RingHub, RingPlan, SlabLayout, cuda_block_step, ring_slots
    obj, x0, cfg = c1
    out = {}
    for dtype in (torch.float64, torch.float32):
        lay = SlabLayout.build(obj.dims.nz, obj.psf.kdims.kz, 4, 3)
        xs, z0s = [], []
        for r in range(3):
            lo, hi = lay.local(r)
            xs.append(torch.from_numpy(np.ascontiguousarray(x0[lo:hi + 1])).cuda().to(dtype))
            z0s.append(lo)
        hub, rings = RingHub.local(RingPlan(lay, ring_slots(1)), xs, z0s)
        step = cuda_block_step(obj, dtype)
        shards = [AsyncShard(lay, r, xs[r], torch.zeros_like(xs[r]), rings[r], step, 1) for r in range(3)]
        for _ in range(4):
            for s in shards:
                s.update()
                torch.cuda.synchronize()
        out[dtype] = _gather(shards).astype(np.float64)
        hub.close()
    a, b = out[torch.float64], out[torch.float32]
    assert np.linalg.norm(a - b) <= 2e-5 * np.linalg.norm(a)
