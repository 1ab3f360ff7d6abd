"""Multi-rank path on CPU: the slab layout / halo plan, and a sharded
block-Jacobi over `gloo` (world sizes 2 and 4, halos spanning several ranks)
that must reproduce the single-process block-Jacobi bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2002_02328_b200.distributed import SlabLayout


def test_layout_plan_is_consistent():
    for nz, kz, h, world in [(64, 11, 8, 8), (64, 11, 8, 2), (24, 5, 2, 4), (30, 7, 4, 3), (16, 3, 16, 1)]:
        lay = SlabLayout.build(nz, kz, h, world)
        owned = [lay.owned(r) for r in range(world)]
        assert owned[0][0] == 0 and owned[-1][1] == nz - 1
        assert all(owned[r][1] + 1 == owned[r + 1][0] for r in range(world - 1))
        sends = {(r, p, lo, hi) for r in range(world) for p, lo, hi, k in lay.transfers(r) if k == "send"}
        recvs = {(p, r, lo, hi) for r in range(world) for p, lo, hi, k in lay.transfers(r) if k == "recv"}
        assert sends == recvs  # every receive has its matching send
        for r in range(world):  # halos exactly cover local minus owned
            got = sorted(z for p, lo, hi, k in lay.transfers(r) if k == "recv" for z in range(lo, hi + 1))
            l_lo, l_hi = lay.local(r)
            want = [z for z in range(l_lo, l_hi + 1) if not owned[r][0] <= z <= owned[r][1]]
            assert got == want
    with pytest.raises(ValueError):
        SlabLayout.build(16, 3, 8, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, sweeps, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from _oracle_shards import OracleShardedJacobi
        O.core("c", threads=1)
        crit, x0, h = _problem(O)
        eng = OracleShardedJacobi(O, crit, x0, h)
        for _ in range(sweeps):
            eng.sweep()
        full = eng.gather()
        if rank == 0:
            np.save(out_path, full)
    finally:
        dist.destroy_process_group()


def _problem(O):
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    dims = Dims3(20, 18, 16)
    psf = blur.depth_variant_stack(dims, (3, 3, 5), (0.8, 1.6), (1.0, 2.0))
    rng = np.random.Generator(np.random.Philox(3))
    y = rng.uniform(0, 1, dims.shape)
    x0 = rng.uniform(0, 1, dims.shape)
    crit = O.Criterion(psf.kernels, y, lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2)
    return crit, x0, 2


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_jacobi_matches_single_process(world, tmp_path, oracle_mod):
    sweeps = 3
    out = tmp_path / "x.npy"
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, sweeps, str(out)), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    crit, x0, h = _problem(oracle_mod)
    B = -(-x0.shape[0] // h)
    want, _, _ = oracle_mod.run_bp3mg(crit, x0, B, h, max_updates=sweeps * B)
    assert np.array_equal(got, want)


def _async_worker(rank, world, port, sweeps, max_delay, out_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2002_02328_b200.distributed import AsyncShard, SlabLayout, TorchP2P
        O.core("c", threads=1)
        crit, x0, h = _problem(O)
        lay = SlabLayout.build(x0.shape[0], crit.kz, h, world)
        lo, hi = lay.local(rank)
        x = torch.from_numpy(np.ascontiguousarray(x0[lo:hi + 1])).clone()
        prev = torch.zeros_like(x)

        def step(shard, b):  # oracle block step on the local slab
            z0 = shard.l_lo
            s_lo, s_hi = O.support(lay.nz, crit.kz, b.z_lo, b.z_hi)
            xl = shard.x.numpy()
            inc = O.mg_direction(crit, xl[s_lo - z0:s_hi - z0 + 1].copy(), s_lo, b.z_lo, b.z_hi,
                                 shard.prev.numpy()[b.z_lo - z0:b.z_hi - z0 + 1].ravel().copy())
            inc = torch.from_numpy(inc.reshape((b.height,) + tuple(shard.x.shape[1:])))
            shard.x[b.z_lo - z0:b.z_hi - z0 + 1] += inc
            shard.prev[b.z_lo - z0:b.z_hi - z0 + 1] = inc

        shard = AsyncShard(lay, rank, x, prev, TorchP2P(x, lo, lay.transfers(rank)), step, max_delay)
        shard.run(sweeps)
        dist.barrier()
        own = x[shard.o_lo - lo:shard.o_hi - lo + 1].contiguous()
        stale = torch.tensor([max(shard.staleness)], dtype=torch.int64)
        dist.all_reduce(stale, op=dist.ReduceOp.MAX)
        if rank == 0:
            parts = [own]
            for q in range(1, world):
                qlo, qhi = lay.owned(q)
                t = torch.empty((qhi - qlo + 1,) + tuple(own.shape[1:]), dtype=own.dtype)
                dist.recv(t, q)
                parts.append(t)
            np.save(out_path, torch.cat(parts).numpy())
            np.save(str(out_path) + ".stale.npy", stale.numpy())
        else:
            dist.send(own, 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_async_bounded_delay_gloo(world, tmp_path, oracle_mod):
    """Real asynchronous ranks (gloo P2P, no barriers between updates):
    staleness stays within the bound and the objective descends."""
    sweeps, max_delay = 3, 2
    out = tmp_path / "xa.npy"
    mp.start_processes(_async_worker, args=(world, _free_port(), sweeps, max_delay, str(out)), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    stale = int(np.load(str(out) + ".stale.npy")[0])
    crit, x0, h = _problem(oracle_mod)
    assert stale <= max_delay
    assert crit.value(got) < crit.value(x0)
    B = -(-x0.shape[0] // h)
    sync, _, _ = oracle_mod.run_bp3mg(crit, x0, B, h, max_updates=sweeps * B)
    assert abs(crit.value(got) - crit.value(sync)) <= 0.05 * crit.value(sync)


def test_p2p_inbox_plan():
    """Every send of the halo plan lands at a distinct, in-range slot of the
    receiver's inbox, and the inbox slots tile the receiver's halo planes."""
    from paper_2002_02328_b200.distributed import PeerHalo
    for nz, kz, h, world in [(64, 11, 8, 8), (64, 11, 8, 2), (24, 5, 2, 4), (30, 7, 4, 3), (512, 21, 64, 8)]:
        lay = SlabLayout.build(nz, kz, h, world)
        slots = {q: [] for q in range(world)}
        for r in range(world):
            for q, lo, hi, k in lay.transfers(r):
                if k != "send":
                    continue
                off, total = PeerHalo.inbox_offset(lay, q, r, lo, hi)
                assert 0 <= off and off + (hi - lo + 1) <= total
                slots[q].append((off, off + hi - lo + 1))
        for q in range(world):
            l_lo, l_hi = lay.local(q)
            o_lo, o_hi = lay.owned(q)
            halo = (l_hi - l_lo + 1) - (o_hi - o_lo + 1)
            covered = sorted(slots[q])
            assert sum(b - a for a, b in covered) == halo
            assert all(covered[i][1] == covered[i + 1][0] for i in range(len(covered) - 1))
        with pytest.raises(ValueError):
            PeerHalo.inbox_offset(lay, 0, 0, 0, 0)


def test_ring_plan_units_tile_the_halos():
    """Async peer rings: the units of every reader tile its halo planes, each
    writer block publishes within the flag limit, ring slots do not overlap."""
    from paper_2002_02328_b200._native import MAX_FLAGS
    from paper_2002_02328_b200.distributed import RingPlan, ring_slots
    for nz, kz, h, world in [(64, 11, 8, 8), (64, 11, 8, 2), (24, 5, 2, 4), (30, 7, 4, 3), (256, 15, 8, 8)]:
        lay = SlabLayout.build(nz, kz, h, world)
        plan = RingPlan(lay, ring_slots(2))
        for q in range(world):
            l_lo, l_hi = lay.local(q)
            o_lo, o_hi = lay.owned(q)
            got = sorted(z for p, r, bi, a, c in plan.units if r == q for z in range(a, c + 1))
            assert got == [z for z in range(l_lo, l_hi + 1) if not o_lo <= z <= o_hi]
            spans = sorted((plan.slot_plane(u, v), plan.slot_plane(u, v) + plan.units[u][4] - plan.units[u][3] + 1)
                           for u in range(len(plan.units)) if plan.units[u][1] == q for v in range(plan.slots))
            assert all(spans[i][1] <= spans[i + 1][0] for i in range(len(spans) - 1))
            assert not spans or spans[-1][1] <= plan.ring_planes[q]
        for p in range(world):
            for bi in range(len(lay.owned_blocks(p))):
                assert len(plan.writes(p, bi)) + 1 <= MAX_FLAGS
