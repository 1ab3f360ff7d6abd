"""Oracle parity of the dense kernels at the BASELINE PSF geometries and
volume sizes (reference contract: _core.pyx:17-96, objective.py:159-187,
directions.py:57-94).

* 7x7x15 (C3/C4) and 9x9x21 (C5) stacks, fp64 <= 1e-12 and fp32 <= 1e-5
  (north_star tolerances), on volumes whose x/y extents leave ragged tiles
  (nx = 45, 64, 200): H, H^T, fragments with a depth offset, the fused
  gradient, one fused block step (gram / increment), and the fused
  block-Jacobi sweep (RESID, GRAD, dual-input GRAM2, solve, update).
* full C2 size (256x256x64 fp64): H, H^T and grad f against the oracle.
* C5 geometry with byte offsets past 2^31 (1024x1024x540 fp32 and
  1024x1024x300 fp64): rows read at the far end of a full-size field must be
  bit-equal to the same rows from a small re-based fragment, and a cropped
  oracle check pins the values; a full-size fp32 Jacobi sweep is bit-equal
  to the same sweep split over two virtual ranks whose local slabs start at
  small offsets.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REG = dict(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2)


def rel(a, b):
    a = a.double().cpu().numpy() if torch.is_tensor(a) else np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


GEOMS = {
    "7x7x15": ((7, 7, 15), (1.0, 3.0), (1.5, 2.5)),   # C3 / C4 family
    "9x9x21": ((9, 9, 21), (1.0, 4.0), (2.0, 3.5)),   # C5 family
}


def _problem(geom, nx, ny, nz, seed, rotated=False):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3
    kd, sxy, sz = GEOMS[geom]
    dims = Dims3(nx, ny, nz)
    if rotated:
        psf = blur.generate_psf_stack(dims, blur.KernelDims(*kd), seed=seed)
    else:
        psf = blur.depth_variant_stack(dims, kd, sxy, sz)
    rng = np.random.Generator(np.random.Philox(seed))
    y = rng.uniform(0, 1, dims.shape)
    x = rng.uniform(-0.1, 1.1, dims.shape)
    obj = objective.Objective(psf, y, objective.RegParams(**REG))
    return obj, x


@pytest.fixture(scope="module")
def geom_cases(oracle_mod):
    """Oracle H, H^T, grad f per (geometry, nx): computed once, shared by
    both precisions."""
    out = {}
    for geom in GEOMS:
        for nx, ny, nz, rot in [(45, 53, 46, False), (64, 64, 48, True), (200, 37, 44, False)]:
            obj, x = _problem(geom, nx, ny, nz, seed=nx + ny, rotated=rot)
            crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, **REG)
            k = obj.psf.kernels
            out[(geom, nx)] = dict(obj=obj, x=x, H=oracle_mod.H(k, x), Ht=oracle_mod.Ht(k, x), g=crit.grad(x),
                                   crit=crit)
    return out


@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("nx", [45, 64, 200])
@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 1e-5)])
def test_H_Ht_grad_at_baseline_geometries(geom, nx, dtype, tol, geom_cases):
    from paper_2002_02328_b200 import blur, objective
    c = geom_cases[(geom, nx)]
    obj, x = c["obj"], c["x"]
    xt = torch.from_numpy(x).cuda().to(dtype)
    assert rel(blur.apply_H(obj.psf, xt), c["H"]) <= tol
    assert rel(blur.apply_Ht(obj.psf, xt), c["Ht"]) <= tol
    assert rel(objective.grad_f(obj, xt), c["g"]) <= tol


@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 1e-5)])
def test_rows_from_offset_fragments(geom, dtype, tol, geom_cases, oracle_mod):
    """Rows from a fragment that starts mid-volume (global depths, zero
    outside the fragment): kz-deep tap walks cut by the fragment edges."""
    from paper_2002_02328_b200 import blur
    c = geom_cases[(geom, 200)]
    obj, x = c["obj"], c["x"]
    k = obj.psf.kernels
    kz = obj.psf.kdims.kz
    for f0, f1, lo, hi in [(3, 3 + kz + 4, 5, 5 + kz), (10, 43, 12, 40), (0, 20, 0, 30)]:
        frag = x[f0:f1 + 1]
        ft = torch.from_numpy(frag).cuda().to(dtype)
        assert rel(blur.apply_H_rows(obj.psf, ft, f0, lo, hi), oracle_mod.H_rows(k, frag, f0, lo, hi)) <= tol
        assert rel(blur.apply_Ht_rows(obj.psf, ft, f0, lo, hi), oracle_mod.Ht_rows(k, frag, f0, lo, hi)) <= tol


@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-10), (torch.float32, 1e-5)])
def test_block_step_at_baseline_geometries(geom, dtype, tol, geom_cases, oracle_mod):
    """One fused mg step (gradient, forward-only Gram, 2x2 solve) on an
    interior and an edge block vs the oracle's reference-arithmetic step."""
    from paper_2002_02328_b200 import blur, directions
    from paper_2002_02328_b200.volume import SliceBlock
    c = geom_cases[(geom, 64)]
    obj, x, crit = c["obj"], c["x"], c["crit"]
    rng = np.random.Generator(np.random.Philox(11))
    for lo, hi in [(20, 27), (0, 9), (40, 47)]:
        blk = SliceBlock(lo, hi)
        s = blur.slab_support(obj.psf, blk)
        d_mem = 0.01 * rng.standard_normal(blk.count(obj.dims))
        slab = x[s.z_lo:s.z_hi + 1]
        want = oracle_mod.mg_step(crit, slab, s.z_lo, lo, hi, d_mem)
        got = directions.mg_step(obj, torch.from_numpy(slab).cuda().to(dtype), s.z_lo, blk,
                                 torch.from_numpy(d_mem).cuda().to(dtype))
        assert got.ncols == want.ncols == 2
        assert rel(np.asarray(got.gram), want.gram) <= tol
        inc = got.increment
        assert rel(inc, want.increment) <= tol


@pytest.mark.parametrize("geom", list(GEOMS))
@pytest.mark.parametrize("nx,h", [(45, 8), (64, 16)])
def test_jacobi_sweeps_at_baseline_geometries(geom, nx, h, oracle_mod):
    """Fused block-Jacobi sweeps (the bench step) vs the oracle's bp3mg
    barrier with workers = B: fp64 <= 1e-12, fp32 <= 1e-5."""
    from paper_2002_02328_b200 import runtime
    obj, x0 = _problem(geom, nx, 41, 48, seed=7 + nx)
    x0 = np.clip(x0, 0, 1)
    B = -(-48 // h)
    sweeps = 2
    crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, **REG)
    want, _, _ = oracle_mod.run_bp3mg(crit, x0, B, h, max_updates=sweeps * B)
    for dtype, tol in [(torch.float64, 1e-12), (torch.float32, 1e-5)]:
        eng = runtime.JacobiSweeper(obj, x0, h, dtype)
        for _ in range(sweeps):
            eng.sweep()
        eng.check()
        assert rel(eng.x, want) <= tol, dtype


def test_cyclic_sweep_at_c5_geometry(oracle_mod):
    """The reference's deterministic cyclic order (one block per step) on
    the 9x9x21 stack in fp64 vs the oracle's simulated engine, workers = 1."""
    from paper_2002_02328_b200 import runtime
    obj, x0 = _problem("9x9x21", 48, 40, 50, seed=5)
    x0 = np.clip(x0, 0, 1)
    h = 10
    B = 5
    crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, **REG)
    want, log, _ = oracle_mod.run_bd3mg(crit, x0, 1, h, max_updates=2 * B)
    res = runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=1, block_height=h, tol=1e-30,
                                                 max_updates=2 * B, engine="simulated"))
    assert rel(res.x_final, want) <= 1e-9
    np.testing.assert_allclose([e.f_value for e in res.log], [f for _, _, f, _ in log], rtol=1e-9)


# ---------------------------------------------------------------------------
def test_full_c2_fp64_vs_oracle(oracle_mod):
    """The headline volume itself: 256x256x64 fp64, PSF 5x5x11 (C2)."""
    from paper_2002_02328_b200 import blur, configs, objective
    cfg = configs.CONFIGS["C2"]
    psf = blur.depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
    rng = np.random.Generator(np.random.Philox(2))
    x = rng.uniform(0, 1, cfg.dims.shape)
    y = oracle_mod.H(psf.kernels, rng.uniform(0, 1, cfg.dims.shape)) + 0.02 * rng.standard_normal(cfg.dims.shape)
    params = objective.RegParams(lam=cfg.lam, eta=cfg.eta, kappa=cfg.kappa, delta=cfg.delta)
    obj = objective.Objective(psf, y, params)
    crit = oracle_mod.Criterion(psf.kernels, y, cfg.lam, cfg.eta, cfg.kappa, cfg.delta)
    xt = torch.from_numpy(x).cuda()
    assert rel(blur.apply_H(psf, xt), oracle_mod.H(psf.kernels, x)) <= 1e-12
    assert rel(blur.apply_Ht(psf, xt), oracle_mod.Ht(psf.kernels, x)) <= 1e-12
    assert rel(objective.grad_f(obj, xt), crit.grad(x)) <= 1e-12
    f_want = crit.value(x)
    assert abs(objective.eval_f(obj, xt) - f_want) <= 1e-12 * abs(f_want)


# ---------------------------------------------------------------------------
def _big_problem(nz, dtype, geom="9x9x21"):
    from paper_2002_02328_b200 import blur, objective
    from paper_2002_02328_b200.volume import Dims3
    kd, sxy, sz = GEOMS[geom]
    dims = Dims3(1024, 1024, nz)
    psf = blur.depth_variant_stack(dims, kd, sxy, sz)
    g = torch.Generator(device="cuda").manual_seed(1234)
    x = torch.rand(dims.shape, generator=g, device="cuda", dtype=dtype)
    y = torch.rand(dims.shape, generator=g, device="cuda", dtype=dtype)
    obj = objective.Objective(psf, y, objective.RegParams(lam=5e-3, eta=1e-1, kappa=0.05, delta=1e-2))
    return obj, x


@pytest.mark.parametrize("nz,dtype,tol", [(540, torch.float32, 1e-5), (300, torch.float64, 1e-12)])
def test_c5_geometry_offsets_past_2gib(nz, dtype, tol, oracle_mod):
    """Rows read at byte offsets > 2^31 inside one full-size field."""
    from paper_2002_02328_b200 import blur, objective
    obj, x = _big_problem(nz, dtype)
    plane_bytes = 1024 * 1024 * x.element_size()
    lo, hi = nz - 12, nz - 3
    assert lo * plane_bytes > 2**31
    kz = obj.psf.kdims.kz
    f0 = lo - kz
    frag = x[f0:].clone()  # re-based copy: small offsets
    for adjoint in (False, True):
        full = blur.correlate_rows(obj.psf, x, 0, lo, hi, adjoint)
        small = blur.correlate_rows(obj.psf, frag, f0, lo, hi, adjoint)
        assert torch.equal(full, small), adjoint
    # gradient rows of a block at the far end: full field vs re-based slab
    g_full, w_full = objective.grad_rows_device(obj, x, 0, lo, hi)
    g_small, w_small = objective.grad_rows_device(obj, frag, f0, lo, hi)
    assert torch.equal(g_full, g_small) and torch.equal(w_full, w_small)
    # values: a cropped oracle check of the top 96 image rows (exact rows
    # are y < 96 - ry; the crop edge only perturbs the rows past that)
    ry = (obj.psf.kdims.ky - 1) // 2
    crop = x[f0:, :96, :].double().cpu().numpy()
    k = obj.psf.kernels
    want = oracle_mod.H_rows(k, crop, f0, lo, lo + 1)
    got = blur.correlate_rows(obj.psf, x, 0, lo, lo + 1, False)[:, :96 - ry].double().cpu().numpy()
    assert rel(got, want[:, :96 - ry]) <= tol
    want_t = oracle_mod.Ht_rows(k, crop, f0, hi - 1, hi)
    got_t = blur.correlate_rows(obj.psf, x, 0, hi - 1, hi, True)[:, :96 - ry].double().cpu().numpy()
    assert rel(got_t, want_t[:, :96 - ry]) <= tol


def test_c5_geometry_sweep_bitwise_vs_rebased_shards():
    """A full-size fp32 Jacobi sweep (1024x1024x520, 9x9x21, 64-plane blocks)
    whose fields cross 2^31 bytes equals, bit for bit, the same sweep split
    over two virtual ranks (local slabs re-based at small offsets)."""
    from paper_2002_02328_b200 import runtime
    from paper_2002_02328_b200.distributed import ShardedJacobi
    obj, x = _big_problem(520, torch.float32)
    x0 = x.double().cpu().numpy()
    del x
    single = runtime.JacobiSweeper(obj, x0, 64, torch.float32)
    shards = [ShardedJacobi(obj, x0, 64, torch.float32, rank=r, world=2, halo="p2p") for r in range(2)]
    bases = {r: s.peer.ptr for r, s in enumerate(shards)}
    for s in shards:
        s.peer.connect(bases)
    for _ in range(2):
        single.sweep()
        for s in shards:
            s.local_sweep()
    single.check()
    full = torch.cat([s.x[s.o_lo - s.l_lo:s.o_hi - s.l_lo + 1] for s in shards])
    assert torch.equal(full, single.x)
    assert not torch.equal(single.x, torch.from_numpy(x0).cuda().float())
    for s in shards:
        s.close()
