"""The persistent one-launch block-Jacobi sweep (csrc/sweep_pk.cuh) against
the multi-kernel sweep it replaces (BD3MG_NO_PK=1): iterate, memory store,
recorder terms and StepInfo must be BIT-identical after several sweeps --
(opt-in with BD3MG_PK=1 while it is slower than the multi-kernel sweep) --
both run the same tile functions with the same tile -> partial-row mapping
and the same final reduction trees.  Covers every tuned tap width, ragged
blocks and tiles, C1 / C2, fragments of a sharded layout with mirror
stores, and replay from a captured CUDA graph."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(obj, x0, h, sweeps, pk: bool, graph=False):
    from paper_2002_02328_b200 import runtime
    if pk:
        os.environ["BD3MG_PK"] = "1"
    else:
        os.environ.pop("BD3MG_PK", None)
    # the bitwise twin of the persistent sweep is the multi-kernel sweep with the separate regulariser-Gram
    # stencil (the default multi-kernel sweep folds those sums into the Gram correlation: other groupings)
    os.environ["BD3MG_NO_RGF"] = "1"
    from paper_2002_02328_b200 import _native as N
    n0 = N.lib.bd3mg_pk_launches()
    try:
        eng = runtime.JacobiSweeper(obj, x0, h, torch.float64)
        eng.sweep()
        assert (N.lib.bd3mg_pk_launches() > n0) == pk  # the persistent kernel ran exactly when asked
        if graph:
            eng.capture()
        terms = []
        for _ in range(sweeps - 1):
            eng.sweep()
            terms.append(eng.terms.clone())
        torch.cuda.synchronize()
        return eng, terms
    finally:
        os.environ.pop("BD3MG_PK", None)
        os.environ.pop("BD3MG_NO_RGF", None)


def _problem(k, nx, ny, nz, seed, kz=None):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3
    dims = Dims3(nx, ny, nz)
    psf = blur.depth_variant_stack(dims, (k, k, kz or min(2 * k + 1, 11)), (0.8, 1.6), (1.0, 2.0))
    rng = np.random.Generator(np.random.Philox(seed))
    y = rng.uniform(0, 1, dims.shape)
    x0 = rng.uniform(0, 1, dims.shape)
    obj = objective.Objective(psf, y, objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2))
    return obj, x0


def _same(a, b):
    """Iterate, memory store, snapshot and StepInfo bit for bit; recorder
    terms bit for bit except the data term (and f): the persistent sweep's
    residual tiles are 64 x 32 (4 CTAs per SM), so its sum of r^2 groups the
    pixels differently."""
    ea, ta = a
    eb, tb = b
    assert torch.equal(ea.x, eb.x)
    assert torch.equal(ea.prev, eb.prev)
    assert torch.equal(ea.snap, eb.snap)
    assert torch.equal(ea.info, eb.info)
    for u, v in zip(ta, tb):
        assert torch.equal(u[[1, 2, 3, 5, 6]], v[[1, 2, 3, 5, 6]])
        torch.testing.assert_close(u[[0, 4]], v[[0, 4]], rtol=1e-13, atol=0)


@pytest.mark.parametrize("k,nx,ny,nz,h", [(5, 64, 64, 24, 8), (3, 70, 45, 22, 4), (7, 64, 50, 40, 8),
                                          (9, 46, 66, 45, 16), (5, 130, 33, 19, 5)])
def test_persistent_sweep_bitwise_multi_kernel(k, nx, ny, nz, h):
    obj, x0 = _problem(k, nx, ny, nz, seed=nx + nz)
    _same(_run(obj, x0, h, 4, pk=True), _run(obj, x0, h, 4, pk=False))


def test_persistent_sweep_c2_and_graph():
    from paper_2002_02328_b200 import configs, objective
    cfg = configs.CONFIGS["C2"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    a = _run(obj, x0, cfg.block_height, 5, pk=True, graph=True)
    _same(a, _run(obj, x0, cfg.block_height, 5, pk=False))


def test_persistent_sweep_oracle_c1(oracle_mod):
    """The persistent path alone vs the oracle's bp3mg barrier cycles."""
    from paper_2002_02328_b200 import configs, objective
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    eng, _ = _run(obj, x0, cfg.block_height, 3, pk=True)
    crit = oracle_mod.Criterion(psf.kernels, y, cfg.lam, cfg.eta, cfg.kappa, cfg.delta)
    want, _, _ = oracle_mod.run_bp3mg(crit, x0, 3, cfg.block_height, max_updates=9)
    got = eng.x.cpu().numpy()
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("world", [2, 3])
def test_persistent_sweep_sharded_mirrors_bitwise(world):
    """Virtual ranks (local slabs with halos, mirror stores into the peers'
    inboxes): the persistent path equals the multi-kernel path per rank and
    the single-GPU sweep overall."""
    from paper_2002_02328_b200.distributed import ShardedJacobi
    obj, x0 = _problem(5, 48, 40, 30, seed=9)
    h = 5
    outs = []
    for pk in (True, False):
        if pk:
            os.environ["BD3MG_PK"] = "1"
        else:
            os.environ.pop("BD3MG_PK", None)
        os.environ["BD3MG_NO_RGF"] = "1"  # see _run
        try:
            from paper_2002_02328_b200 import _native as N
            n0 = N.lib.bd3mg_pk_launches()
            shards = [ShardedJacobi(obj, x0, h, torch.float64, rank=r, world=world, halo="p2p") for r in range(world)]
            bases = {r: s.peer.ptr for r, s in enumerate(shards)}
            for s in shards:
                s.peer.connect(bases)
            for _ in range(4):
                for s in shards:
                    s.local_sweep()
            torch.cuda.synchronize()
            assert (N.lib.bd3mg_pk_launches() > n0) == pk
            outs.append(torch.cat([s.x[s.o_lo - s.l_lo:s.o_hi - s.l_lo + 1] for s in shards]).clone())
            for s in shards:
                s.close()
        finally:
            os.environ.pop("BD3MG_PK", None)
            os.environ.pop("BD3MG_NO_RGF", None)
    assert torch.equal(outs[0], outs[1])
    single, _ = _run(obj, x0, h, 4, pk=True)
    assert torch.equal(outs[0], single.x)
