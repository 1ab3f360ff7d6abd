"""Host-buffer C-ABI entry points (the reference-facing plugin calls used by
the end-to-end measurement) agree with the device-resident paths."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1obj():
    from paper_2002_02328_b200 import configs, objective
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    return objective.Objective(psf, y, params), x0, cfg


def test_host_worker_step_matches_device(c1obj):
    from paper_2002_02328_b200 import blur, directions
    from paper_2002_02328_b200.host import HostProblem
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x0, cfg = c1obj
    hp = HostProblem(obj)
    rng = np.random.default_rng(1)
    for blk in (SliceBlock(0, 7), SliceBlock(8, 15), SliceBlock(16, 23)):
        s = blur.slab_support(obj.psf, blk)
        dm = 0.01 * rng.standard_normal(blk.count(obj.dims))
        info = np.zeros(16)
        got = hp.mg_direction(x0[s.z_lo:s.z_hi + 1], s.z_lo, blk, dm, info)
        want = directions.mg_step(obj, x0[s.z_lo:s.z_hi + 1], s.z_lo, blk, dm)
        assert np.array_equal(got, want.increment)
        assert int(info[7]) == want.ncols
    hp.close()


def test_host_sweep_matches_device_sweeper(c1obj):
    from paper_2002_02328_b200 import runtime
    from paper_2002_02328_b200.host import HostProblem, pinned_empty
    obj, x0, cfg = c1obj
    eng = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64)
    hp = HostProblem(obj)
    x = pinned_empty(x0.shape)
    x[...] = x0
    dm = pinned_empty(x0.shape)
    dm[...] = 0
    for _ in range(4):
        eng.sweep()
        t = hp.jacobi_sweep(x, dm, eng.blocks)
        assert t[4] == pytest.approx(eng.f(), rel=1e-14)
    assert np.array_equal(x, eng.x.cpu().numpy())
    assert np.array_equal(dm, eng.prev.cpu().numpy())
    hp.close()


def test_host_sweep_fp32(c1obj):
    from paper_2002_02328_b200 import runtime
    from paper_2002_02328_b200.host import HostProblem
    obj, x0, cfg = c1obj
    eng = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64)
    hp = HostProblem(obj, dtype="f32")
    x, dm = x0.copy(), np.zeros_like(x0)
    for _ in range(4):
        eng.sweep()
        hp.jacobi_sweep(x, dm, eng.blocks)
    ref = eng.x.cpu().numpy()
    assert np.linalg.norm(x - ref) <= 1e-5 * np.linalg.norm(ref)
    hp.close()


def test_host_sweep_session_mode(c1obj):
    """dmem=None keeps the memory store on the device: same iterates."""
    from paper_2002_02328_b200 import runtime
    from paper_2002_02328_b200.host import HostProblem
    obj, x0, cfg = c1obj
    eng = runtime.JacobiSweeper(obj, x0, cfg.block_height, torch.float64)
    hp = HostProblem(obj)
    x = x0.copy()
    for _ in range(4):
        eng.sweep()
        hp.jacobi_sweep(x, None, eng.blocks)
    assert np.array_equal(x, eng.x.cpu().numpy())
    hp.close()


@pytest.mark.parametrize("h,pinned,dt", [(5, False, "f64"), (8, True, "f64"), (3, True, "f64"), (8, True, "f32"),
                                         (5, False, "f32")])
def test_pipelined_session_sweep_bitwise(h, pinned, dt):
    """>= 4 back-to-back blocks over the whole volume take the pipelined host
    path (two halves, transfers overlapped): iterate bitwise that of the
    device sweep, recorder terms equal to rounding; BD3MG_NO_PIPELINE=1 path
    agrees."""
    from paper_2002_02328_b200 import blur, objective, runtime
    from paper_2002_02328_b200.host import HostProblem
    from paper_2002_02328_b200.volume import Dims3
    dims = Dims3(64, 48, 40)
    psf = blur.depth_variant_stack(dims, (5, 5, 11), (0.8, 2.0), (1.5, 2.5))
    rng = np.random.Generator(np.random.Philox(11))
    y = rng.uniform(0, 1, dims.shape)
    x0 = rng.uniform(0, 1, dims.shape)
    obj = objective.Objective(psf, y, objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2))
    eng = runtime.JacobiSweeper(obj, x0, h, torch.float64 if dt == "f64" else torch.float32)
    assert eng.nblocks >= 4
    hp = HostProblem(obj, dtype=dt)
    if pinned:  # page-locked x: calls after the first replay one captured CUDA graph
        from paper_2002_02328_b200.host import pinned_empty
        x = pinned_empty(x0.shape)
        x[...] = x0
    else:
        x = x0.copy()
    terms = np.zeros(7)
    for _ in range(4):
        eng.sweep()
        hp.jacobi_sweep(x, None, eng.blocks, terms=terms)
        ref = eng.terms.cpu().numpy()
        np.testing.assert_allclose(terms[:5], ref[:5], rtol=1e-13 if dt == "f64" else 1e-6)
    assert np.array_equal(x, eng.x.double().cpu().numpy())
    hp.close()


def test_host_handle_serialises_concurrent_worker_threads(c1obj):
    """The reference's live engine calls its core from several worker
    threads at once (runtime.py:188-200).  Calls on one HostProblem handle
    share its stream and buffers, so the library serialises them (per-handle
    mutex): 8 threads x 6 calls each must give exactly the sequential
    results (concurrent calls used to race on the uploads)."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.host import HostProblem
    from paper_2002_02328_b200.volume import SliceBlock
    obj, x0, cfg = c1obj
    hp = HostProblem(obj)
    rng = np.random.default_rng(7)
    jobs = []
    for i in range(48):
        blk = (SliceBlock(0, 7), SliceBlock(8, 15), SliceBlock(16, 23))[i % 3]
        s = blur.slab_support(obj.psf, blk)
        xs = x0[s.z_lo:s.z_hi + 1] * (1.0 + 0.01 * i)
        jobs.append((xs, s.z_lo, blk, 0.01 * rng.standard_normal(blk.count(obj.dims))))
    want = [hp.mg_direction(*j) for j in jobs]
    with ThreadPoolExecutor(max_workers=8) as pool:
        got = list(pool.map(lambda j: hp.mg_direction(*j), jobs))
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    hp.close()
