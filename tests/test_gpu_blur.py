"""GPU parity of H / H^T (sm_100a kernels through the C ABI) against the
reference's own outputs (tests/golden/blur.npz, made by the reference) and
the reference test suite's properties (reference tests/test_blur.py)."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


def _psf(blur, kernels):
    nz, kz, ky, kx = kernels.shape
    return blur.PsfStack((1, 1, nz), (kx, ky, kz), kernels)


def _psf_for(blur, kernels, shape):
    nz, ny, nx = shape
    _, kz, ky, kx = kernels.shape
    return blur.PsfStack((nx, ny, nz), (kx, ky, kz), kernels)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def cases():
    return golden("blur")


def test_forward_adjoint_match_reference(cases):
    from paper_2002_02328_b200 import blur
    for name, c in cases.items():
        psf = _psf_for(blur, c["kernels"], c["x"].shape)
        np.testing.assert_allclose(blur.apply_H(psf, c["x"]), c["Hx"], rtol=1e-12, atol=1e-13, err_msg=name)
        np.testing.assert_allclose(blur.apply_Ht(psf, c["v"]), c["Htv"], rtol=1e-12, atol=1e-13, err_msg=name)
        assert rel(blur.apply_H(psf, c["x"]), c["Hx"]) <= 1e-12


def test_rows_match_reference(cases):
    from paper_2002_02328_b200 import blur
    for name, c in cases.items():
        psf = _psf_for(blur, c["kernels"], c["x"].shape)
        lo, hi, f0, f1 = (int(v) for v in c["rows"])
        np.testing.assert_allclose(blur.apply_H_rows(psf, c["x"][f0:f1 + 1], f0, lo, hi), c["Hrows"],
                                   rtol=1e-12, atol=1e-13, err_msg=name)
        np.testing.assert_allclose(blur.apply_Ht_rows(psf, c["v"][f0:f1 + 1], f0, lo, hi), c["Htrows"],
                                   rtol=1e-12, atol=1e-13, err_msg=name)


def test_against_oracle_random_shapes(oracle_mod, rng):
    """Tiled (square ky=kx) and generic paths, odd sizes, partial tiles."""
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    for dims, kd in [((70, 67, 13), (3, 3, 3)), ((65, 130, 9), (5, 5, 11)), ((131, 7, 6), (7, 7, 5)),
                     ((19, 90, 7), (9, 9, 3)), ((17, 23, 8), (3, 5, 3)), ((5, 6, 9), (1, 1, 1)),
                     ((1, 40, 5), (1, 3, 3)), ((64, 64, 4), (11, 11, 3))]:
        psf = blur.generate_psf_stack(Dims3(*dims), blur.KernelDims(*kd), seed=sum(dims))
        x = rng.standard_normal(Dims3(*dims).shape)
        want = oracle_mod.H(psf.kernels, x)
        assert rel(blur.apply_H(psf, x), want) <= 1e-13, (dims, kd)
        want_t = oracle_mod.Ht(psf.kernels, x)
        assert rel(blur.apply_Ht(psf, x), want_t) <= 1e-13, (dims, kd)


def test_dirac_is_identity_bitwise(rng):
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    for kd in [(3, 3, 3), (5, 5, 5), (1, 1, 1), (3, 5, 3)]:
        psf = blur.dirac_stack(Dims3(6, 5, 4), blur.KernelDims(*kd))
        x = rng.standard_normal((4, 5, 6))
        assert np.array_equal(blur.apply_H(psf, x), x)
        assert np.array_equal(blur.apply_Ht(psf, x), x)


def test_slab_restriction_bitwise(rng):
    """reference tests/test_blur.py:139-147: rows from a slab == full rows."""
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3, SliceBlock
    for dims, kd in [((8, 8, 12), (3, 3, 3)), ((70, 40, 30), (5, 5, 11)), ((9, 7, 10), (3, 5, 5))]:
        psf = blur.generate_psf_stack(Dims3(*dims), blur.KernelDims(*kd), seed=5)
        x = rng.standard_normal(Dims3(*dims).shape)
        full = blur.apply_H(psf, x)
        fullt = blur.apply_Ht(psf, x)
        nz = dims[2]
        for blk in (SliceBlock(nz // 2, nz // 2 + 1), SliceBlock(0, 1), SliceBlock(nz - 2, nz - 1)):
            s = blur.slab_support(psf, blk)
            rows = blur.apply_H_rows(psf, x[s.z_lo:s.z_hi + 1], s.z_lo, blk.z_lo, blk.z_hi)
            assert np.array_equal(rows, full[blk.z_lo:blk.z_hi + 1])
            rows = blur.apply_Ht_rows(psf, x[s.z_lo:s.z_hi + 1], s.z_lo, blk.z_lo, blk.z_hi)
            assert np.array_equal(rows, fullt[blk.z_lo:blk.z_hi + 1])


def test_adjoint_identity(rng):
    """<Hx, v> == <x, H^T v> (reference tests/test_blur.py:96-105)."""
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    for trial in range(5):
        psf = blur.generate_psf_stack(Dims3(40, 33, 12), blur.KernelDims(5, 5, 7), seed=trial)
        x = rng.standard_normal((12, 33, 40))
        v = rng.standard_normal((12, 33, 40))
        lhs = np.vdot(blur.apply_H(psf, x), v)
        rhs = np.vdot(x, blur.apply_Ht(psf, v))
        assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(x) * np.linalg.norm(v)


def test_linearity_and_zero(rng):
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    psf = blur.generate_psf_stack(Dims3(7, 6, 5), blur.KernelDims(3, 3, 5), seed=8)
    x, y = rng.standard_normal((5, 6, 7)), rng.standard_normal((5, 6, 7))
    np.testing.assert_allclose(blur.apply_H(psf, 1.7 * x - 0.4 * y),
                               1.7 * blur.apply_H(psf, x) - 0.4 * blur.apply_H(psf, y), rtol=1e-12, atol=1e-14)
    assert not blur.apply_H(psf, np.zeros((5, 6, 7))).any()
    assert not blur.apply_Ht(psf, np.zeros((5, 6, 7))).any()


def test_fp32_within_1e5(oracle_mod, rng):
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    psf = blur.depth_variant_stack(Dims3(256, 96, 24), blur.KernelDims(5, 5, 11), (0.8, 2.0), (1.5, 2.5))
    x = rng.uniform(0, 1, (24, 96, 256))
    xt = torch.from_numpy(x).cuda().float()
    got = blur.apply_H(psf, xt).double().cpu().numpy()
    assert rel(got, oracle_mod.H(psf.kernels, x)) <= 1e-5
    got = blur.apply_Ht(psf, xt).double().cpu().numpy()
    assert rel(got, oracle_mod.Ht(psf.kernels, x)) <= 1e-5


def test_device_tensor_roundtrip(rng):
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    psf = blur.generate_psf_stack(Dims3(9, 8, 6), blur.KernelDims(3, 3, 3), seed=1)
    x = rng.standard_normal((6, 8, 9))
    out = blur.apply_H(psf, torch.from_numpy(x).cuda())
    assert out.is_cuda and out.dtype == torch.float64
    assert np.array_equal(out.cpu().numpy(), blur.apply_H(psf, x))


def test_errors():
    from paper_2002_02328_b200 import blur, kernels
    from paper_2002_02328_b200.volume import Dims3
    psf = blur.generate_psf_stack(Dims3(6, 6, 4), blur.KernelDims(3, 3, 3), seed=0)
    with pytest.raises(ValueError, match="dims"):
        blur.apply_H(psf, np.zeros((4, 6, 7)))
    with pytest.raises(ValueError):
        kernels.depthvar_correlate(np.zeros((4, 6, 6)), psf.kernels, 0, 0, 4)  # row 4 outside stack
    with pytest.raises(ValueError, match="dtype"):
        kernels.depthvar_correlate(np.zeros((4, 6, 6), dtype=np.float32), psf.kernels, 0, 0, 3)


def test_host_capi_dropin_matches_device(cases):
    """kernels.depthvar_correlate[_adjoint]: the host-buffer C entry points a
    ctypes binding of the reference would call."""
    from paper_2002_02328_b200 import kernels
    for name, c in cases.items():
        k = c["kernels"]
        nz = c["x"].shape[0]
        np.testing.assert_allclose(kernels.depthvar_correlate(c["x"], k, 0, 0, nz - 1), c["Hx"], rtol=1e-12,
                                   atol=1e-13, err_msg=name)
        np.testing.assert_allclose(kernels.depthvar_correlate_adjoint(c["v"], k, 0, 0, nz - 1), c["Htv"],
                                   rtol=1e-12, atol=1e-13, err_msg=name)
    assert kernels.USING_COMPILED and kernels.backend_name() == "cuda-sm100a"
