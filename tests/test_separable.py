"""Separable-PSF fast path: rank-one detection on the
host, and on the GPU the C-ABI bd3mg_sep_correlate_* against the oracle's
dense correlation (the reference contract, _core.pyx:17-96)."""

import numpy as np
import pytest

from paper_2002_02328_b200 import blur, separable
from paper_2002_02328_b200.volume import Dims3


def test_detects_axis_aligned_gaussians_only():
    dims = Dims3(16, 12, 10)
    psf = blur.depth_variant_stack(dims, (5, 5, 7), (0.8, 2.0), (1.0, 2.5))
    f = separable.factor_stack(psf)
    assert f is not None
    u, v, w = f
    assert u.shape == (10, 7) and v.shape == (10, 5) and w.shape == (10, 5)
    rot = blur.generate_psf_stack(dims, blur.KernelDims(5, 5, 7), seed=3)  # random phi, theta
    assert separable.factor_stack(rot) is None
    with pytest.raises(ValueError, match="not separable"):
        separable.SeparableStack.from_psf(rot)
    with pytest.raises(ValueError, match="kx == ky"):
        separable.SeparableStack.from_psf(blur.depth_variant_stack(dims, (3, 5, 7), (0.8, 2.0), (1.0, 2.5)))


@pytest.mark.gpu
@pytest.mark.parametrize("k,kz", [(3, 5), (5, 11), (7, 15), (9, 21)])
@pytest.mark.parametrize("nx", [48, 37])
def test_matches_dense_oracle(k, kz, nx, oracle_mod):
    import torch
    dims = Dims3(nx, 29, 40)
    psf = blur.depth_variant_stack(dims, (k, k, kz), (0.8, 2.0), (1.0, 2.5))
    sep = separable.SeparableStack.from_psf(psf)
    rng = np.random.Generator(np.random.Philox(k * 100 + nx))
    x = rng.uniform(-1, 1, dims.shape)
    for adj, want in ((False, oracle_mod.H(psf.kernels, x)), (True, oracle_mod.Ht(psf.kernels, x))):
        got = sep.correlate_rows(torch.from_numpy(x).cuda(), 0, 0, dims.nz - 1, adjoint=adj).cpu().numpy()
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
        got32 = sep.correlate_rows(torch.from_numpy(x).cuda().float(), 0, 0, dims.nz - 1, adjoint=adj)
        assert np.linalg.norm(got32.double().cpu().numpy() - want) <= 1e-5 * np.linalg.norm(want)


@pytest.mark.gpu
def test_rows_of_a_fragment_and_adjoint_identity(oracle_mod):
    import torch
    dims = Dims3(40, 33, 50)
    psf = blur.depth_variant_stack(dims, (5, 5, 11), (0.8, 2.0), (1.0, 2.5))
    sep = separable.SeparableStack.from_psf(psf)
    rng = np.random.Generator(np.random.Philox(7))
    x = rng.uniform(0, 1, dims.shape)
    z0, z1 = 13, 38  # fragment planes 13..38: zero outside, as the reference
    frag = x[z0:z1 + 1]
    for adj in (False, True):
        fn = oracle_mod.Ht_rows if adj else oracle_mod.H_rows
        for lo, hi in ((0, 49), (20, 31), (40, 49), (0, 3)):
            want = fn(psf.kernels, frag, z0, lo, hi)
            got = sep.correlate_rows(torch.from_numpy(frag).cuda(), z0, lo, hi, adjoint=adj).cpu().numpy()
            assert np.linalg.norm(got - want) <= 1e-12 * max(np.linalg.norm(want), 1e-300)
            # fp32 (nx = 40: the TMA-fed 2-D filter, boxes offset by the fragment origin)
            got32 = sep.correlate_rows(torch.from_numpy(frag).cuda().float(), z0, lo, hi, adjoint=adj)
            assert np.linalg.norm(got32.double().cpu().numpy() - want) <= 1e-5 * max(np.linalg.norm(want), 1e-300)
    y = rng.uniform(0, 1, dims.shape)
    hx = sep.apply_H(x)
    hty = sep.apply_Ht(y)
    assert abs(np.vdot(hx, y) - np.vdot(x, hty)) <= 1e-12 * abs(np.vdot(hx, y))


@pytest.mark.gpu
@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_variants_bitwise_equal(dt, monkeypatch):
    """Every depth-FIR / 2-D filter variant (csrc/separable.cu probe knobs)
    computes the same sums in the same order: results are bitwise equal."""
    import torch
    dims = Dims3(64, 40, 48)
    psf = blur.depth_variant_stack(dims, (7, 7, 15), (0.8, 2.0), (1.0, 2.5))
    sep = separable.SeparableStack.from_psf(psf)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(dims.shape, dtype=getattr(torch, dt), device="cuda", generator=g)
    for adj in (False, True):
        ref = None
        for xy, zv in (("1", "8160"), ("2", "8160"), ("2", "8161"), ("2", "8080"), ("2", "8081"),
                       ("2", "16081"), ("2", "16161"), ("3", "16161"), ("3", "8160"), ("5", "16161")):
            monkeypatch.setenv("BD3MG_SEP_XY", xy)
            monkeypatch.setenv("BD3MG_SEP_Z", zv)
            got = sep.correlate_rows(x[5:40], 5, 9, 33, adjoint=adj)
            if ref is None:
                ref = got
            assert torch.equal(got, ref), (adj, xy, zv)
