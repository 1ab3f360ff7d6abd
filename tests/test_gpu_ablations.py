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


@pytest.mark.parametrize("case", ["abl0", "abl1"])
def test_device_ablations_match_reference_goldens(case):
    """Device CG (bd3mg_cg_solve: converged and budget-stopped, same iteration
    counts), mm / gd / cg directions and the device power iteration
    (bd3mg_power_hth) vs the reference's own outputs
    (tests/golden/ablation.npz; reference directions.py:97-168,
    objective.py:301-375)."""
    from conftest import golden
    from paper_2002_02328_b200 import N_launches, blur, directions, objective
    from paper_2002_02328_b200.volume import Dims3, SliceBlock
    c = golden("ablation")[case]
    nz, ny, nx = c["x"].shape
    _, kz, ky, kx = c["kernels"].shape
    psf = blur.PsfStack(Dims3(nx, ny, nz), (kx, ky, kz), c["kernels"])
    lam, eta, kappa, delta, xmin, xmax = c["reg"]
    obj = objective.Objective(psf, c["y"], objective.RegParams(lam, eta, kappa, delta, xmin, xmax))
    rho = objective.rho_hth_estimate(psf)
    assert abs(rho - float(c["rho"])) <= 1e-12 * float(c["rho"])
    assert objective.rho_hth_estimate(psf, iters=3, seed=1) == float(c["rho3"])
    L = objective.lipschitz_estimate(obj)
    assert abs(L - float(c["L"])) <= 1e-12 * float(c["L"])
    x = c["x"]
    for j in range(2):
        lo, hi = (int(v) for v in c[f"b{j}_blk"])
        blk = SliceBlock(lo, hi)
        s = blur.slab_support(psf, blk)
        slab = x[s.z_lo:s.z_hi + 1]
        np.testing.assert_allclose(directions.gd_direction(obj, slab, s.z_lo, blk, float(c["L"])), c[f"b{j}_gd"],
                                   rtol=1e-12, atol=1e-15)
        got = directions.cg_direction(obj, slab, s.z_lo, blk, c[f"b{j}_dmem"], float(c["L"]))
        assert np.linalg.norm(got - c[f"b{j}_cg"]) <= 1e-10 * np.linalg.norm(c[f"b{j}_cg"])
        mm = directions.mm_direction(obj, slab, s.z_lo, blk, cg_tol=1e-8, cg_maxit=200)
        assert np.linalg.norm(mm - c[f"b{j}_mm"]) <= 1e-8 * np.linalg.norm(c[f"b{j}_mm"])
        g = objective.grad_block(obj, slab, blk, s.z_lo)
        maj = objective.MajorantOperator(obj, slab, blk, s.z_lo)
        for tag in ("conv", "budget"):
            conv, iters, relres, tol, maxit = c[f"b{j}_cg_{tag}_meta"]
            n0 = N_launches()
            xs, cv, it, rr = directions.cg_solve(maj.apply, -g, tol, int(maxit))
            assert N_launches() > n0  # the device solver ran (not the host loop)
            assert (cv, it) == (bool(conv), int(iters)), (case, j, tag, cv, it)
            # a converged solve's final residual (~1e-11) is rounding-dominated
            assert abs(rr - relres) <= (1e-2 if conv else 1e-6) * relres
            want = c[f"b{j}_cg_{tag}_x"]
            assert np.linalg.norm(xs - want) <= 1e-9 * np.linalg.norm(want)


def test_device_cg_edge_cases():
    """b = 0 (converged in 0 iterations, x = 0), maxit = 0 (the best iterate
    x = 0, relres 1) and fp32 tensors on the device, against the oracle's
    restatement of cg_solve (reference directions.py:117-149)."""
    from oracle import oracle as O
    from paper_2002_02328_b200 import directions, objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, rng = _problem()
    blk = SliceBlock(2, 5)
    maj = objective.MajorantOperator(obj, x, blk, 0)
    n = blk.count(obj.dims)
    xs, cv, it, rr = directions.cg_solve(maj.apply, np.zeros(n), 1e-8, 50)
    assert cv and it == 0 and rr == 0.0 and not xs.any()
    b = rng.standard_normal(n)
    xs, cv, it, rr = directions.cg_solve(maj.apply, b, 1e-8, 0)
    assert (cv, it, rr) == (False, 0, 1.0) and not xs.any()
    want = O.cg_solve(maj.apply, b, 1e-6, 100)
    got = directions.cg_solve(maj.apply, b, 1e-6, 100)
    assert (got[1], got[2]) == (want[1], want[2])
    assert np.linalg.norm(got[0] - want[0]) <= 1e-9 * np.linalg.norm(want[0])
    xt = torch.from_numpy(x).cuda().float()
    maj32 = objective.MajorantOperator(obj, xt, blk, 0)
    w32, cv32, it32, _ = directions.cg_solve(maj32.apply, torch.from_numpy(b).cuda().float(), 1e-4, 100)
    assert w32.is_cuda and w32.dtype == torch.float32 and cv32
    assert np.linalg.norm(w32.double().cpu().numpy() - want[0]) <= 1e-4 * np.linalg.norm(want[0])
