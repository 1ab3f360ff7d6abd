"""The reference's own hot-path pins, restated against
the CUDA path: gradient vs central finite differences, lambda-linearity, the
majorant vs a dense principal submatrix built independently on the host
(dense H from the oracle core, difference matrices from numpy), the
majorization / tangency properties, the Cauchy step, a parallel memory
column, subspace optimality, and block descent for every tuned tap width.

Reference tests they follow: tests/test_objective.py:63-80, :119-131,
:177-251; tests/test_directions.py:57-76, :104-134, :267-286."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _problem(dims=(7, 6, 8), kdims=(3, 3, 3), seed=5, lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3
    d = Dims3(*dims)
    psf = blur.depth_variant_stack(d, kdims, (0.6, 1.1), (0.7, 1.2))
    rng = np.random.Generator(np.random.Philox(seed))
    y = rng.uniform(0.0, 1.0, d.shape)
    x = rng.uniform(-0.2, 1.2, d.shape)  # both sides of the box [0, 1]
    obj = objective.Objective(psf, y, objective.RegParams(lam=lam, eta=eta, kappa=kappa, delta=delta))
    return obj, x, rng


def test_gradient_matches_central_differences():
    from paper_2002_02328_b200 import objective
    obj, x, rng = _problem()
    g = objective.grad_f(obj, x)
    h = 1e-6
    for _ in range(12):
        i = tuple(int(rng.integers(0, n)) for n in x.shape)
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        fd = (objective.eval_f(obj, xp) - objective.eval_f(obj, xm)) / (2 * h)
        assert abs(fd - g[i]) <= 1e-5 * max(1.0, abs(g[i])), (i, fd, g[i])


def test_gradient_is_affine_in_lambda():
    from paper_2002_02328_b200 import objective
    grads = []
    lams = (1e-3, 1e-2, 3e-2)
    for lam in lams:
        obj, x, _ = _problem(lam=lam)
        grads.append(objective.grad_f(obj, x))
    d1, d2 = grads[1] - grads[0], grads[2] - grads[0]
    ratio = (lams[2] - lams[0]) / (lams[1] - lams[0])
    assert np.linalg.norm(d2 - ratio * d1) <= 1e-12 * np.linalg.norm(grads[2])


def _diff_matrix(shape, axis):
    """Forward difference along `axis` with a zero row at the far face."""
    n = int(np.prod(shape))
    idx = np.arange(n).reshape(shape)
    D = np.zeros((n, n))
    m = shape[axis]
    for k in range(m - 1):
        a = np.take(idx, k, axis=axis).ravel()
        b = np.take(idx, k + 1, axis=axis).ravel()
        D[a, a] = -1.0
        D[a, b] = 1.0
    return D


def test_majorant_equals_dense_principal_submatrix(oracle_mod):
    from paper_2002_02328_b200 import objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, _ = _problem()
    p = obj.params
    shape = x.shape
    n = x.size
    Hd = np.empty((n, n))
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        Hd[:, i] = oracle_mod.H(obj.psf.kernels, e.reshape(shape)).ravel()
    Dz, Dy, Dx = (_diff_matrix(shape, a) for a in (0, 1, 2))
    gx, gy = Dx @ x.ravel(), Dy @ x.ravel()
    w = 1.0 / np.sqrt(gx * gx + gy * gy + p.delta ** 2)
    A = Hd.T @ Hd + 2 * p.eta * np.eye(n) + p.lam * (Dx.T @ (w[:, None] * Dx) + Dy.T @ (w[:, None] * Dy)) \
        + 2 * p.kappa * Dz.T @ Dz
    for blk in (SliceBlock(0, 2), SliceBlock(3, 5), SliceBlock(6, 7)):
        plane = shape[1] * shape[2]
        S = np.arange(blk.z_lo * plane, (blk.z_hi + 1) * plane)
        A_S = A[np.ix_(S, S)]
        maj = objective.MajorantOperator(obj, x, blk, 0)
        got = np.stack([maj.apply(np.eye(len(S))[:, j]) for j in range(len(S))], axis=1)
        np.testing.assert_allclose(got, A_S, rtol=1e-10, atol=1e-12 * np.abs(A_S).max())
        assert np.allclose(got, got.T, rtol=1e-12, atol=1e-14 * np.abs(got).max())


def test_majorization_and_tangency():
    """Q(x~_S; x~) = f(x~), grad Q = grad_S f at the anchor, and Q >= f for
    block perturbations (half-quadratic majorant, reference Eq. (2))."""
    from paper_2002_02328_b200 import objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, rng = _problem()
    blk = SliceBlock(2, 4)
    maj = objective.MajorantOperator(obj, x, blk, 0)
    rows = x[blk.z_lo:blk.z_hi + 1].ravel()
    f0 = objective.eval_f(obj, x)
    assert abs(objective.majorant_Q(maj, rows) - f0) <= 1e-13 * abs(f0)
    g = objective.grad_block(obj, x, blk)
    h = 1e-6
    for _ in range(4):
        j = int(rng.integers(0, rows.size))
        e = np.zeros(rows.size)
        e[j] = h
        fd = (objective.majorant_Q(maj, rows + e) - objective.majorant_Q(maj, rows - e)) / (2 * h)
        assert abs(fd - g[j]) <= 1e-5 * max(1.0, abs(g[j]))
    for scale in (1e-3, 1e-1, 1.0):
        v = rows + scale * rng.standard_normal(rows.size)
        xv = x.copy()
        xv[blk.z_lo:blk.z_hi + 1] = v.reshape(xv[blk.z_lo:blk.z_hi + 1].shape)
        assert objective.majorant_Q(maj, v) >= objective.eval_f(obj, xv) - 1e-12 * abs(f0)


def _step(obj, x, blk, d_mem):
    from paper_2002_02328_b200 import blur, directions
    s = blur.slab_support(obj.psf, blk)
    return directions.mg_step(obj, x[s.z_lo:s.z_hi + 1], s.z_lo, blk, d_mem)


def test_cauchy_step_without_memory():
    """d_mem = 0: the step is -alpha g, alpha = g'g / g'A g."""
    from paper_2002_02328_b200 import objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, _ = _problem()
    blk = SliceBlock(3, 5)
    n = blk.count(obj.dims)
    st = _step(obj, x, blk, np.zeros(n))
    g = objective.grad_block(obj, x, blk)
    Ag = objective.MajorantOperator(obj, x, blk, 0).apply(g)
    alpha = (g @ g) / (g @ Ag)
    assert st.ncols == 1
    np.testing.assert_allclose(st.increment, -alpha * g, rtol=1e-10)


def test_parallel_memory_column_gives_cauchy_step():
    """d_mem parallel to g: the 2x2 Gram is singular, the pseudo-inverse
    drops the null direction and the step is still the Cauchy step."""
    from paper_2002_02328_b200 import objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, _ = _problem()
    blk = SliceBlock(0, 2)
    g = objective.grad_block(obj, x, blk)
    st = _step(obj, x, blk, -0.3 * g)
    Ag = objective.MajorantOperator(obj, x, blk, 0).apply(g)
    alpha = (g @ g) / (g @ Ag)
    np.testing.assert_allclose(st.increment, -alpha * g, rtol=1e-8, atol=1e-12 * np.abs(g).max())


def test_two_column_step_minimises_the_model_on_the_subspace():
    """The increment minimises Q over span{-g, d} (checked against the exact
    2x2 solve on host-built Gram entries and against a perturbation grid)."""
    from paper_2002_02328_b200 import objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, rng = _problem()
    blk = SliceBlock(3, 5)
    n = blk.count(obj.dims)
    d = 0.05 * rng.standard_normal(n)
    st = _step(obj, x, blk, d)
    g = objective.grad_block(obj, x, blk)
    maj = objective.MajorantOperator(obj, x, blk, 0)
    B = np.stack([-g, d], axis=1)
    AB = np.stack([maj.apply(B[:, 0]), maj.apply(B[:, 1])], axis=1)
    G = B.T @ AB
    c = -np.linalg.solve(0.5 * (G + G.T), B.T @ g)
    assert st.ncols == 2
    np.testing.assert_allclose(st.increment, B @ c, rtol=1e-9)
    rows = x[blk.z_lo:blk.z_hi + 1].ravel()
    q0 = objective.majorant_Q(maj, rows + st.increment)
    for du in (1e-3, -1e-3):
        for dv in (1e-3, -1e-3):
            q = objective.majorant_Q(maj, rows + B @ (c + np.array([du, dv])))
            assert q >= q0 - 1e-12 * abs(q0)


@pytest.mark.parametrize("k", [3, 5, 7, 9])
def test_block_step_descends_for_every_tap_width(k):
    from paper_2002_02328_b200 import objective
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x, _ = _problem(dims=(24, 20, 16), kdims=(k, k, 5))
    f0 = objective.eval_f(obj, x)
    for blk in (SliceBlock(0, 3), SliceBlock(4, 9), SliceBlock(10, 15)):
        st = _step(obj, x, blk, np.zeros(blk.count(obj.dims)))
        xn = x.copy()
        xn[blk.z_lo:blk.z_hi + 1] += st.increment.reshape(xn[blk.z_lo:blk.z_hi + 1].shape)
        assert objective.eval_f(obj, xn) < f0
