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


@pytest.mark.parametrize("world,cfgname,hd", [(2, "C1", False), (3, "C1", True), (8, "C2", False)])
def test_virtual_ranks_bitwise(world, cfgname, hd):
    from paper_2002_02328_b200 import configs, objective, runtime
    from paper_2002_02328_b200.distributed import ShardedJacobi
    cfg = configs.CONFIGS[cfgname]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    single = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64, hd_cache=hd)
    shards = [ShardedJacobi(obj, x0, cfg.block_height, torch.float64, rank=r, world=world, hd_cache=hd)
              for r in range(world)]
    for it in range(4):
        single.sweep()
        _exchange(shards)
        for s in shards:
            s.local_sweep()
        total = sum(s.terms for s in shards)
        ref = single.terms
        # anchor terms of this sweep: f and the stop norms agree across layouts
        np.testing.assert_allclose(total[[0, 1, 2, 3, 4, 5, 6]].cpu().numpy(), ref.cpu().numpy(), rtol=1e-12)
    full = torch.cat([s.x[s.o_lo - s.l_lo:s.o_hi - s.l_lo + 1] for s in shards])
    assert torch.equal(full, single.x)
    _exchange(shards)
    for s in shards:
        s.record_local()
    assert abs(float(sum(s.terms for s in shards)[4]) - single.finish()) <= 1e-12 * abs(single.f())


def test_jacobi_sweeper_matches_barrier_runtime():
    """JacobiSweeper == runtime.run(method='bp3mg', workers=B) iterate and
    per-sweep f (the recorder lags one sweep by construction)."""
    from paper_2002_02328_b200 import configs, objective, runtime
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    eng = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64)
    fs = []
    for it in range(5):
        eng.sweep()
        if it > 0:
            fs.append(eng.f())
    fs.append(eng.finish())
    res = runtime.run(obj, x0, runtime.RunConfig(method="bp3mg", workers=3, block_height=8, tol=1e-30,
                                                 max_updates=15))
    np.testing.assert_allclose(fs, [e.f_value for e in res.log], rtol=1e-13)
    assert np.array_equal(eng.x.cpu().numpy(), res.x_final)


def test_hd_cache_variant_tracks_exact(oracle_mod):
    """hd-cache variant: same iterates as the exact recompute to rounding."""
    from paper_2002_02328_b200 import configs, objective, runtime
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    a = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64)
    b = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64, hd_cache=True)
    for _ in range(30):
        a.sweep()
        b.sweep()
    xa, xb = a.x.cpu().numpy(), b.x.cpu().numpy()
    assert np.linalg.norm(xa - xb) <= 1e-10 * np.linalg.norm(xa)
    assert abs(a.finish() - b.finish()) <= 1e-11 * abs(a.f())


def test_cyclic_sweeper_matches_runtime():
    """Device cyclic sweeps == runtime.run(bd3mg, workers=1) iterate and log."""
    from paper_2002_02328_b200 import configs, objective, runtime
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    eng = runtime.CyclicSweeper(obj, x0, cfg.block_height, torch.float64)
    eng.sweep()
    eng.capture()
    fs = [eng.f()]
    for _ in range(4):
        eng.sweep()
        fs.append(eng.f())
    res = runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=1, block_height=8, tol=1e-30,
                                                 max_updates=15))
    np.testing.assert_allclose(fs, [e.f_value for e in res.log], rtol=1e-13)
    assert np.array_equal(eng.x.cpu().numpy(), res.x_final)


@pytest.mark.parametrize("world,cfgname,dtype", [(2, "C1", torch.float64), (3, "C1", torch.float64),
                                                 (8, "C2", torch.float64), (3, "C1", torch.float32),
                                                 (8, "C2", torch.float32)])
def test_virtual_ranks_p2p_halos_bitwise(world, cfgname, dtype):
    """halo='p2p': the update kernel stores the neighbour-facing rows into the
    peers' double-buffered inboxes (here: virtual ranks of one process, the
    inbox addresses passed directly); the iterate must equal the
    single-GPU sweep bit for bit, eagerly and through the per-parity graphs."""
    from paper_2002_02328_b200 import configs, objective, runtime
    from paper_2002_02328_b200.distributed import ShardedJacobi
    cfg = configs.CONFIGS[cfgname]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    single = runtime.JacobiSweeper(obj, x0, cfg.block_height, dtype)
    shards = [ShardedJacobi(obj, x0, cfg.block_height, dtype, rank=r, world=world, halo="p2p")
              for r in range(world)]
    rtol = 1e-12 if dtype == torch.float64 else 1e-6  # fp32: the recorder sums group rows per rank
    bases = {r: s.peer.ptr for r, s in enumerate(shards)}
    for s in shards:
        s.peer.connect(bases)
    for it in range(5):
        if it == 2:
            for s in shards:
                s.capture()
        single.sweep()
        for s in shards:
            s.local_sweep()
        total = sum(s.terms for s in shards)
        np.testing.assert_allclose(total.cpu().numpy(), single.terms.cpu().numpy(), rtol=rtol)
    full = torch.cat([s.x[s.o_lo - s.l_lo:s.o_hi - s.l_lo + 1] for s in shards])
    assert torch.equal(full, single.x)
    # halos of every shard after the unpack equal the neighbours' owned rows
    for s in shards:
        s.peer.unpack(s.sweeps % 2)
        assert torch.equal(s.x, single.x[s.l_lo:s.l_hi + 1])
    for s in shards:
        s.record_local()
    assert abs(float(sum(s.terms for s in shards)[4]) - single.finish()) <= rtol * abs(single.f())
    for s in shards:
        s.close()


def test_mirror_rows_must_be_updated():
    """A mirror outside the sweep's blocks is rejected (EINVAL -> ValueError)."""
    from paper_2002_02328_b200 import _native as N, configs, device as D, objective
    from paper_2002_02328_b200.distributed import ShardedJacobi
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    s = ShardedJacobi(obj, x0, cfg.block_height, torch.float64, rank=0, world=2)
    buf = torch.zeros_like(s.x)
    bad = (N.Mirror * 1)(N.Mirror(s.o_hi + 1, s.o_hi + 2, buf.data_ptr()))
    with pytest.raises(ValueError, match="mirror"):
        N.check(N.lib.bd3mg_jacobi_sweep_mirrored(
            D.byref(s.geom), D.byref(s.reg), s.K.data_ptr(), s.y_shift, D.byref(s.sw), bad, 1,
            s.terms.data_ptr(), s.info.data_ptr(), s.ws.data_ptr(), s.ws_bytes, D.stream_handle()))


def _ipc_worker(rank, world, port, sweeps, out_dir):
    """One process per virtual rank, all on cuda:0: inboxes mapped with
    cudaIpc, host-side (gloo) synchronisation between sweeps -- kernels never
    wait on one another."""
    import os

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2002_02328_b200 import configs, objective
        from paper_2002_02328_b200.distributed import ShardedJacobi
        cfg = configs.CONFIGS["C1"]
        psf, truth, y, x0, params = configs.make_problem(cfg)
        obj = objective.Objective(psf, y, params)
        s = ShardedJacobi(obj, x0, cfg.block_height, torch.float64, halo="p2p")
        fs = []
        for _ in range(sweeps):
            s.sweep()
            fs.append(s.f())
        fs.append(s.finish())
        full = s.gather()
        if rank == 0:
            np.save(f"{out_dir}/x.npy", full)
            np.save(f"{out_dir}/f.npy", np.array(fs))
        dist.barrier()
        s.close()
    finally:
        dist.destroy_process_group()


def test_ipc_p2p_halos_two_processes(tmp_path):
    """halo='p2p' across processes: cudaIpc-mapped inboxes (both processes on
    the one GPU here; over NVLink on a multi-GPU node) reproduce the
    single-GPU sweep bit for bit."""
    import socket

    import torch.multiprocessing as mp

    from paper_2002_02328_b200 import configs, objective, runtime
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    sweeps = 4
    mp.start_processes(_ipc_worker, args=(2, port, sweeps, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    single = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64)
    fs = []
    for _ in range(sweeps):
        single.sweep()
        fs.append(single.f())
    fs.append(single.finish())
    assert np.array_equal(np.load(tmp_path / "x.npy"), single.x.cpu().numpy())
    np.testing.assert_allclose(np.load(tmp_path / "f.npy"), fs, rtol=1e-12)


@pytest.mark.parametrize("dtype,refresh", [(torch.float64, 0), (torch.float64, 4), (torch.float32, 0)])
def test_incremental_residual_variant_tracks_exact(dtype, refresh):
    """Variant "hd-incremental" (residual kept by linearity, no residual
    correlation per sweep): iterates and recorded f track the exact sweep to
    rounding, eagerly and through the captured graphs."""
    from paper_2002_02328_b200 import configs, objective, runtime
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    a = runtime.JacobiSweeper(obj, x0, cfg.block_height, dtype)
    b = runtime.JacobiSweeper(obj, x0, cfg.block_height, dtype, incremental=True, refresh_every=refresh)
    tol_x, tol_f = (1e-10, 1e-11) if dtype == torch.float64 else (2e-5, 1e-5)
    for it in range(30):
        if it == 3:
            a.capture()
            b.capture()
        a.sweep()
        b.sweep()
        if it > 0:
            assert abs(a.f() - b.f()) <= tol_f * abs(a.f()), (it, a.f(), b.f())
    xa, xb = a.x.double().cpu().numpy(), b.x.double().cpu().numpy()
    assert np.linalg.norm(xa - xb) <= tol_x * np.linalg.norm(xa)
    # the kept residual is H x - y of the current iterate
    from paper_2002_02328_b200 import blur
    r = blur.apply_H(psf, b.x) - obj.device_y(dtype)
    assert float(torch.linalg.vector_norm(r - b.resid)) <= (1e-11 if dtype == torch.float64 else 1e-4) * float(
        torch.linalg.vector_norm(r))


def test_incremental_residual_needs_whole_volume():
    from paper_2002_02328_b200 import configs, objective, runtime
    from paper_2002_02328_b200.volume import SliceBlock
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    with pytest.raises(ValueError):  # blocks that do not tile the volume
        eng = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64,
                                    blocks=[SliceBlock(0, 7), SliceBlock(8, 15)], incremental=True)
        eng.sweep()


def test_p2p_mirrors_keep_inboxes_current_on_nonfinite_gradient():
    """A block whose gradient is non-finite applies no update; its mirror
    rows still land in the neighbour's inbox (unchanged x), so the next
    sweep's halos equal the owner's rows."""
    from paper_2002_02328_b200 import configs, objective
    from paper_2002_02328_b200.distributed import ShardedJacobi
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    x0 = x0.copy()
    x0[20, 5, 5] = np.nan  # rank 1 owns planes 8..23: both of its blocks see the NaN in their residual
    obj = objective.Objective(psf, y, params)
    shards = [ShardedJacobi(obj, x0, cfg.block_height, torch.float64, rank=r, world=2, halo="p2p") for r in range(2)]
    bases = {r: s.peer.ptr for r, s in enumerate(shards)}
    for s in shards:
        s.peer.connect(bases)
    before = shards[1].x.clone()
    for s in shards:
        s.local_sweep()
    torch.cuda.synchronize()
    assert bool((shards[1].info[:, 8] != 0).any())
    with pytest.raises(ValueError, match="non-finite"):
        shards[1].check()
    o1 = shards[1].o_lo - shards[1].l_lo
    assert torch.equal(torch.nan_to_num(shards[1].x[o1:]), torch.nan_to_num(before[o1:]))
    s0 = shards[0]
    s0.peer.unpack(s0.sweeps % 2)
    lo = s0.o_hi + 1
    got = s0.x[lo - s0.l_lo:s0.l_hi - s0.l_lo + 1]
    want = shards[1].x[lo - shards[1].l_lo:s0.l_hi - shards[1].l_lo + 1]
    assert torch.equal(got, want)
    for s in shards:
        s.close()


@pytest.mark.parametrize("dtype,refresh", [(torch.float64, 0), (torch.float64, 3), (torch.float32, 0)])
def test_cyclic_incremental_variant_tracks_exact(dtype, refresh):
    """The deterministic cyclic schedule in the "hd-incremental" variant
    (kept residual, cached H E_S d_mem, recorder from the kept residual)
    tracks the exact cyclic sweep to rounding, eagerly and as graphs."""
    from paper_2002_02328_b200 import blur, configs, objective, runtime
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    a = runtime.CyclicSweeper(obj, x0, cfg.block_height, dtype)
    b = runtime.CyclicSweeper(obj, x0, cfg.block_height, dtype, incremental=True, refresh_every=refresh)
    tol_x, tol_f = (1e-10, 1e-11) if dtype == torch.float64 else (2e-5, 1e-5)
    for it in range(20):
        if it == 2:
            a.capture()
            b.capture()
        a.sweep()
        b.sweep()
        assert abs(a.f() - b.f()) <= tol_f * abs(a.f()), (it, a.f(), b.f())
    xa, xb = a.x.double().cpu().numpy(), b.x.double().cpu().numpy()
    assert np.linalg.norm(xa - xb) <= tol_x * np.linalg.norm(xa)
    r = blur.apply_H(psf, b.x) - obj.device_y(dtype)
    assert float(torch.linalg.vector_norm(r - b.resid)) <= (1e-11 if dtype == torch.float64 else 1e-4) * float(
        torch.linalg.vector_norm(r))


def test_cyclic_incremental_ragged_blocks():
    """Cyclic hd-incremental with a ragged tail block tracks the exact cyclic sweep."""
    from paper_2002_02328_b200 import blur, objective, runtime
    from paper_2002_02328_b200.volume import Dims3
    dims = Dims3(40, 36, 22)
    psf = blur.depth_variant_stack(dims, (5, 5, 7), (0.8, 1.6), (1.0, 2.0))
    rng = np.random.Generator(np.random.Philox(9))
    y = rng.uniform(0, 1, dims.shape)
    x0 = rng.uniform(0, 1, dims.shape)
    obj = objective.Objective(psf, y, objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2))
    a = runtime.CyclicSweeper(obj, x0, 4, torch.float64)
    b = runtime.CyclicSweeper(obj, x0, 4, torch.float64, incremental=True)
    for _ in range(8):
        a.sweep()
        b.sweep()
        assert abs(a.f() - b.f()) <= 1e-11 * abs(a.f())
    xa, xb = a.x.cpu().numpy(), b.x.cpu().numpy()
    assert np.linalg.norm(xa - xb) <= 1e-10 * np.linalg.norm(xa)


def _sweeps_with_env(env, sweeps=3, dtype=torch.float64, cfg_name="C1", graph=False):
    """x, d_mem, StepInfo and recorder terms after `sweeps` block-Jacobi sweeps with `env` set."""
    import os
    from paper_2002_02328_b200 import configs, objective, runtime
    cfg = configs.CONFIGS[cfg_name]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        eng = runtime.JacobiSweeper(obj, x0, 4 if cfg_name == "C1" else cfg.block_height, dtype)
        terms = []
        eng.sweep()
        if graph:
            eng.capture()
        for _ in range(sweeps - 1):
            eng.sweep()
            terms.append(eng.terms.clone())
        torch.cuda.synchronize()
        return eng.x.clone(), eng.prev.clone(), eng.info.clone(), terms
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("graph", [False, True])
def test_chain_layouts_are_bitwise_equal(graph):
    """The GRAD -> Gram -> solve -> update chains of the batched step (1 to 4
    chains, per-chain regulariser-gradient launches enqueued before or after
    the residual correlation) only reorder independent launches: iterate,
    memory store, StepInfo and recorder terms must not change by a bit."""
    ref = _sweeps_with_env({"BD3MG_PARTS": "1", "BD3MG_GREG_AFTER": "0"}, graph=graph)
    for env in ({"BD3MG_PARTS": "2", "BD3MG_GREG_AFTER": "0"}, {"BD3MG_PARTS": "2", "BD3MG_GREG_AFTER": "1"},
                {"BD3MG_PARTS": "3", "BD3MG_GREG_AFTER": "1"}, {"BD3MG_PARTS": "4", "BD3MG_GREG_AFTER": "1"}, {}):
        got = _sweeps_with_env(env, graph=graph)
        assert torch.equal(got[0], ref[0]), env
        assert torch.equal(got[1], ref[1]), env
        assert torch.equal(got[2], ref[2]), env
        for u, v in zip(got[3], ref[3]):
            assert torch.equal(u, v), env


def test_fused_regulariser_gram_matches_the_stencil():
    """The regulariser Gram terms computed by the Gram correlation's tiles
    (rg_center, the default) against the separate reg_gram stencil
    (BD3MG_NO_RGF=1): same sums in another grouping -- Gram entries, rhs and
    coefficients to 1e-12, iterates to 1e-11 after three sweeps; the flags
    (column mask, status) exactly."""
    a = _sweeps_with_env({})
    b = _sweeps_with_env({"BD3MG_NO_RGF": "1"})
    ia, ib = a[2].cpu().numpy(), b[2].cpu().numpy()
    np.testing.assert_allclose(ia[:, :7], ib[:, :7], rtol=1e-11, atol=1e-300)
    assert np.array_equal(ia[:, [7, 8, 12]], ib[:, [7, 8, 12]])
    xa, xb = a[0].cpu().numpy(), b[0].cpu().numpy()
    assert np.linalg.norm(xa - xb) <= 1e-11 * np.linalg.norm(xb)
    assert not np.array_equal(ia[:, :3], ib[:, :3]) or np.array_equal(xa, xb)


def test_chain_layouts_fp32_bitwise_iterates():
    """fp32 sweeps run in chains too (up to 2^27 voxels per step): iterate,
    memory store and StepInfo must not depend on the layout by a bit; the
    recorder's data term regroups (the two-plane kernels pair other planes
    when the residual goes out per chain), so it is compared to fp32 rounding."""
    ref = _sweeps_with_env({"BD3MG_NO_CHAINS_F32": "1"}, dtype=torch.float32)
    for env in ({}, {"BD3MG_PARTS": "3"}, {"BD3MG_GREG_AFTER": "0"}):
        got = _sweeps_with_env(env, dtype=torch.float32)
        assert torch.equal(got[0], ref[0]), env
        assert torch.equal(got[1], ref[1]), env
        assert torch.equal(got[2], ref[2]), env
        for u, v in zip(got[3], ref[3]):
            torch.testing.assert_close(u, v, rtol=1e-6, atol=0)
