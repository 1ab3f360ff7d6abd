"""the ablation directions (reference
directions.py:97-168) and the Lipschitz estimate (objective.py:301-375) on
the device operators, checked against their defining formulas on a problem
small enough for dense host matrices."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _problem(seed=4):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3
    d = Dims3(7, 6, 8)
    psf = blur.depth_variant_stack(d, (3, 3, 3), (0.6, 1.1), (0.7, 1.2))
    rng = np.random.Generator(np.random.Philox(seed))
    y = rng.uniform(0.0, 1.0, d.shape)
    x = rng.uniform(-0.2, 1.2, d.shape)
    obj = objective.Objective(psf, y, objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2))
    return obj, x, rng


def _slab(obj, x, blk):
    from paper_2002_02328_b200 import blur
    s = blur.slab_support(obj.psf, blk)
    return x[s.z_lo:s.z_hi + 1], s.z_lo


def test_gd_and_cg_directions_follow_their_formulas():
    from paper_2002_02328_b200 import directions, objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, rng = _problem()
    blk = SliceBlock(2, 4)
    slab, z0 = _slab(obj, x, blk)
    g = objective.grad_block(obj, x, blk)
    L = 7.5
    np.testing.assert_allclose(directions.gd_direction(obj, slab, z0, blk, L), -g / L, rtol=1e-14)
    # metric L*Id: with no memory the step is -g/L; with a memory column it is
    # the exact minimiser of <g,w> + L/2 |w|^2 over span{-g, d}
    np.testing.assert_allclose(directions.cg_direction(obj, slab, z0, blk, np.zeros_like(g), L), -g / L,
                               rtol=1e-12)
    d = rng.standard_normal(g.size)
    B = np.stack([-g, d], axis=1)
    c = -np.linalg.solve(L * (B.T @ B), B.T @ g)
    np.testing.assert_allclose(directions.cg_direction(obj, slab, z0, blk, d, L), B @ c, rtol=1e-9)
    with pytest.raises(ValueError):
        directions.gd_direction(obj, slab, z0, blk, 0.0)


def test_mm_direction_solves_the_block_model():
    """A_S w = -g by CG on the device majorant: matches a dense solve."""
    from paper_2002_02328_b200 import directions, objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, _ = _problem()
    blk = SliceBlock(3, 5)
    slab, z0 = _slab(obj, x, blk)
    g = objective.grad_block(obj, x, blk)
    maj = objective.MajorantOperator(obj, x, blk, 0)
    A = np.stack([maj.apply(e) for e in np.eye(g.size)], axis=1)
    want = np.linalg.solve(0.5 * (A + A.T), -g)
    got = directions.mm_direction(obj, slab, z0, blk, cg_tol=1e-12, cg_maxit=500)
    assert np.linalg.norm(got - want) <= 1e-8 * np.linalg.norm(want)


def test_lipschitz_estimate_bounds_the_spectrum(oracle_mod):
    """rho(H^T H) estimate: at least the true spectral radius (dense), at most
    the norm bound; the Lipschitz bound adds the regulariser constants."""
    from paper_2002_02328_b200 import objective
    obj, x, _ = _problem()
    n = x.size
    H = np.empty((n, n))
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        H[:, i] = oracle_mod.H(obj.psf.kernels, e.reshape(x.shape)).ravel()
    rho = float(np.linalg.eigvalsh(H.T @ H).max())
    est = objective.rho_hth_estimate(obj.psf, iters=200, seed=0)
    assert rho * (1 - 1e-6) <= est <= objective.operator_norm_bound(obj.psf) * (1 + 1e-12)
    assert est <= 1.05 * rho * (1 + 1e-3)
    p = obj.params
    L = objective.lipschitz_estimate(obj, iters=200, seed=0)
    assert abs(L - (est + 2 * p.eta + (p.lam / p.delta) * 8 + 2 * p.kappa * 4)) <= 1e-12 * L


@pytest.mark.parametrize("method", ["async_gd", "async_cg", "async_mm"])
def test_ablation_methods_descend_through_runtime(method):
    from paper_2002_02328_b200 import objective, runtime
    obj, x, _ = _problem()
    f0 = objective.eval_f(obj, x)
    res = runtime.run(obj, x, runtime.RunConfig(method=method, workers=1, block_height=2, tol=1e-30,
                                                max_updates=12))
    fs = [e.f_value for e in res.log]
    assert fs[-1] < f0 and all(b <= a * (1 + 1e-12) for a, b in zip(fs, fs[1:]))
