"""Every tuned kernel width (3/5/7/9 taps in x and y, plus a generic width),
TMA (even nx) and cp.async-fallback (odd nx) staging, in fp64 against the
oracle and in fp32 (packed FFMA2 two-plane kernels, dual-input Gram) against
the fp64 path: a fused block-Jacobi sweep end to end."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _problem(k, nx, ny=37, nz=20, seed=0):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3
    dims = Dims3(nx, ny, nz)
    kz = min(2 * k + 1, 11)
    psf = blur.depth_variant_stack(dims, (k, k, kz), (0.8, 1.6), (1.0, 2.0))
    rng = np.random.Generator(np.random.Philox(seed))
    y = rng.uniform(0, 1, dims.shape)
    x0 = rng.uniform(0, 1, dims.shape)
    obj = objective.Objective(psf, y, objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2))
    return obj, x0


@pytest.mark.parametrize("k", [3, 5, 7, 9, 11])
@pytest.mark.parametrize("nx", [64, 45])
def test_sweep_fp64_vs_oracle_and_fp32(k, nx, oracle_mod):
    from paper_2002_02328_b200 import runtime
    obj, x0 = _problem(k, nx)
    h = 4
    e64 = runtime.JacobiSweeper(obj, x0, h, torch.float64)
    e32 = runtime.JacobiSweeper(obj, x0, h, torch.float32)
    for _ in range(3):
        e64.sweep()
        e32.sweep()
    crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2)
    B = -(-x0.shape[0] // h)
    want, _, _ = oracle_mod.run_bp3mg(crit, x0, B, h, max_updates=3 * B)
    got64 = e64.x.cpu().numpy()
    assert np.linalg.norm(got64 - want) <= 1e-12 * np.linalg.norm(want)
    got32 = e32.x.double().cpu().numpy()
    assert np.linalg.norm(got32 - got64) <= 1e-5 * np.linalg.norm(got64)


@pytest.mark.parametrize("nz,h", [(40, 1), (21, 3)])
def test_barrier_engine_many_and_ragged_blocks(nz, h, oracle_mod):
    """runtime.run(bp3mg, workers = B): B = 40 > 32 (two launches per cycle,
    increments applied after both) and a ragged last block, vs the oracle."""
    from paper_2002_02328_b200 import blur, objective, runtime
    from paper_2002_02328_b200.volume import Dims3
    dims = Dims3(24, 20, nz)
    psf = blur.depth_variant_stack(dims, (3, 3, 5), (0.8, 1.6), (1.0, 2.0))
    rng = np.random.Generator(np.random.Philox(nz + h))
    y = rng.uniform(0, 1, dims.shape)
    x0 = rng.uniform(0, 1, dims.shape)
    params = objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2)
    obj = objective.Objective(psf, y, params)
    B = -(-nz // h)
    res = runtime.run(obj, x0, runtime.RunConfig(method="bp3mg", workers=B, block_height=h, tol=1e-30,
                                                 max_updates=2 * B, engine="simulated"))
    crit = oracle_mod.Criterion(psf.kernels, y, lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2)
    want, _, _ = oracle_mod.run_bp3mg(crit, x0, B, h, max_updates=2 * B)
    assert np.linalg.norm(res.x_final - want) <= 1e-12 * np.linalg.norm(want)
