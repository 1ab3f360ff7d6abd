"""GPU parity of the fused objective kernels (eval_f, gradient, majorant,
memory-gradient block step) against the reference's outputs
(tests/golden/objective.npz) and properties from the reference suite
(reference tests/test_objective.py, tests/test_directions.py)."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))


@pytest.fixture(scope="module")
def cases():
    return golden("objective")


def build(c):
    from paper_2002_02328_b200 import blur, objective
    k = c["kernels"]
    nz, ny, nx = c["y"].shape
    psf = blur.PsfStack((nx, ny, nz), (k.shape[3], k.shape[2], k.shape[1]), k)
    lam, eta, kappa, delta, xmin, xmax = (float(v) for v in c["reg"])
    return objective.Objective(psf, c["y"], objective.RegParams(lam, eta, kappa, delta, xmin, xmax))


def test_eval_f_and_grad(cases):
    from paper_2002_02328_b200 import objective
    for name, c in cases.items():
        obj = build(c)
        assert objective.eval_f(obj, c["x"]) == pytest.approx(float(c["f"]), rel=1e-12), name
        assert rel(objective.grad_f(obj, c["x"]), c["grad"]) <= 1e-12, name


def test_grad_block_slab_and_majorant(cases):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import SliceBlock
    for name, c in cases.items():
        obj = build(c)
        x = c["x"]
        gfull = objective.grad_f(obj, x)
        for j, (lo, hi) in enumerate(c["blocks"]):
            blk = SliceBlock(int(lo), int(hi))
            s = blur.slab_support(obj.psf, blk)
            frag = x[s.z_lo:s.z_hi + 1]
            g = objective.grad_block(obj, frag, blk, s.z_lo)
            assert rel(g, c[f"b{j}_gblock"]) <= 1e-12, (name, j)
            # slab == full-volume restriction, bitwise (reference test_objective.py:90-97)
            assert np.array_equal(g, gfull[blk.z_lo:blk.z_hi + 1].ravel()), (name, j)
            maj = objective.MajorantOperator(obj, frag, blk, s.z_lo)
            np.testing.assert_allclose(maj.omega.cpu().numpy(), c[f"b{j}_omega"], rtol=1e-15, atol=0)
            assert rel(maj.apply(c[f"b{j}_v"]), c[f"b{j}_Av"]) <= 1e-12, (name, j)


def test_mg_step_matches_reference(cases):
    from paper_2002_02328_b200 import blur, directions
    from paper_2002_02328_b200.volume import SliceBlock
    for name, c in cases.items():
        obj = build(c)
        x = c["x"]
        for j, (lo, hi) in enumerate(c["blocks"]):
            blk = SliceBlock(int(lo), int(hi))
            s = blur.slab_support(obj.psf, blk)
            frag = x[s.z_lo:s.z_hi + 1]
            info = directions.mg_step(obj, frag, s.z_lo, blk, c[f"b{j}_dmem"])
            assert info.ncols == c[f"b{j}_gram"].shape[0]
            np.testing.assert_allclose(info.gram, c[f"b{j}_gram"], rtol=1e-11)
            np.testing.assert_allclose(info.rhs, c[f"b{j}_rhs"], rtol=1e-12)
            np.testing.assert_allclose(info.coeffs, c[f"b{j}_coeffs"], rtol=1e-10)
            assert rel(info.increment, c[f"b{j}_inc"]) <= 1e-10, (name, j)
            # first visit: zero memory -> Cauchy step, one column
            inc0 = directions.mg_direction(obj, frag, s.z_lo, blk, np.zeros_like(c[f"b{j}_dmem"]))
            assert rel(inc0, c[f"b{j}_inc0"]) <= 1e-12, (name, j)
            inc0n = directions.mg_direction(obj, frag, s.z_lo, blk, None)
            assert rel(inc0n, c[f"b{j}_inc0"]) <= 1e-12, (name, j)


def test_constant_volume_and_stationary_block():
    """reference test_objective.py:27-61, test_directions.py:96-102."""
    from paper_2002_02328_b200 import blur, directions, objective
    from paper_2002_02328_b200.volume import Dims3, SliceBlock
    psf = blur.generate_psf_stack(Dims3(6, 6, 4), blur.KernelDims(3, 3, 3), seed=3)
    x = np.full((4, 6, 6), 0.4)
    obj = objective.Objective(psf, blur.apply_H(psf, x), objective.RegParams())
    assert objective.eval_f(obj, x) == pytest.approx(obj.params.lam * x.size * obj.params.delta, rel=1e-13)
    assert not objective.grad_f(obj, x).any()
    d = directions.mg_direction(obj, x, 0, SliceBlock(1, 1), np.zeros(36))
    assert not d.any()


def test_nonfinite_gradient_rejected():
    from paper_2002_02328_b200 import blur, directions, objective
    from paper_2002_02328_b200.volume import Dims3, SliceBlock
    psf = blur.generate_psf_stack(Dims3(5, 5, 3), blur.KernelDims(3, 3, 3), seed=3)
    x = np.random.default_rng(0).uniform(0, 1, (3, 5, 5))
    obj = objective.Objective(psf, blur.apply_H(psf, x), objective.RegParams())
    x[0, 0, 0] = np.inf
    with np.errstate(invalid="ignore"), pytest.raises(ValueError):
        directions.mg_direction(obj, x, 0, SliceBlock(0, 0), np.zeros(25))


def test_insufficient_slab_rejected():
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3, SliceBlock
    psf = blur.generate_psf_stack(Dims3(6, 6, 10), blur.KernelDims(3, 3, 5), seed=3)
    obj = objective.Objective(psf, np.zeros((10, 6, 6)), objective.RegParams())
    with pytest.raises(ValueError, match="support"):
        objective.grad_block(obj, np.zeros((3, 6, 6)), SliceBlock(5, 5), 4)


def test_fp32_gradient_within_1e5(oracle_mod):
    from paper_2002_02328_b200 import configs, objective
    from paper_2002_02328_b200.blur import depth_variant_stack
    from paper_2002_02328_b200.volume import Dims3
    psf = depth_variant_stack(Dims3(128, 64, 24), (5, 5, 11), (0.8, 2.0), (1.5, 2.5))
    rng = np.random.default_rng(3)
    y = rng.uniform(0, 1, (24, 64, 128))
    x = rng.uniform(0, 1, (24, 64, 128))
    p = objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2)
    obj = objective.Objective(psf, y, p)
    crit = oracle_mod.Criterion(psf.kernels, y, p.lam, p.eta, p.kappa, p.delta)
    g32 = objective.grad_f(obj, torch.from_numpy(x).cuda().float()).double().cpu().numpy()
    assert rel(g32, crit.grad(x)) <= 1e-5
    g64 = objective.grad_f(obj, x)
    assert rel(g64, crit.grad(x)) <= 1e-12


def test_majorant_symmetric_pd(rng):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3, SliceBlock
    psf = blur.generate_psf_stack(Dims3(6, 6, 4), blur.KernelDims(3, 3, 3), seed=3)
    obj = objective.Objective(psf, rng.uniform(0, 1, (4, 6, 6)), objective.RegParams())
    anchor = rng.uniform(0, 1, (4, 6, 6))
    maj = objective.MajorantOperator(obj, anchor, SliceBlock(1, 2))
    for _ in range(5):
        u, v = rng.standard_normal(maj.n), rng.standard_normal(maj.n)
        assert abs(u @ maj.apply(v) - v @ maj.apply(u)) <= 1e-10 * (1 + abs(u @ maj.apply(v)))
        assert v @ maj.apply(v) >= 2 * obj.params.eta * (v @ v) - 1e-10
    with pytest.raises(ValueError, match="length"):
        maj.apply(np.zeros(maj.n + 1))
