"""Full-solve parity on BASELINE config C1 (64x64x24 fp64, PSF 5x5x11,
3 blocks of 8): the GPU runtime against the reference's own trajectories
(tests/golden/c1.npz) -- objective log and final iterate within 1e-9
relative after 50 (and 150) block updates of the deterministic cyclic
schedule, the block-Jacobi barrier mode and the seeded async engine."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    return golden("c1")


@pytest.fixture(scope="module")
def problem(c1):
    from paper_2002_02328_b200 import blur, configs, objective
    from paper_2002_02328_b200.volume import add_gaussian_noise, init_uniform
    cfg = configs.CONFIGS["C1"]
    k = c1["kernels"]
    psf = blur.depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
    assert np.array_equal(psf.kernels, k)  # generator is bitwise the reference's
    truth = configs.truth_of(cfg)
    # H(truth) through the reference-identical oracle so y is bitwise the golden y
    from oracle import oracle as O
    O.core("c", threads=8)
    y = add_gaussian_noise(O.H(k, truth), cfg.noise, cfg.seed + 2)
    import hashlib
    assert hashlib.sha256(y.tobytes()).hexdigest() == str(c1["y_sha"])
    x0 = init_uniform(cfg.dims, float(np.max(y)), cfg.seed + 3)
    assert hashlib.sha256(x0.tobytes()).hexdigest() == str(c1["x0_sha"])
    p = objective.RegParams(lam=cfg.lam, eta=cfg.eta, kappa=cfg.kappa, delta=cfg.delta)
    return objective.Objective(psf, y, p), x0, cfg


def _check(res, c1, tag, tol=1e-9):
    f = np.array([e.f_value for e in res.log])
    assert [e.k for e in res.log] == list(c1[f"{tag}_k"])
    assert np.max(np.abs(f - c1[f"{tag}_f"]) / np.abs(c1[f"{tag}_f"])) <= tol
    assert res.grant_log == list(c1[f"{tag}_grants"])
    assert [ev.staleness for ev in res.trace] == list(c1[f"{tag}_stale"])
    x = res.x_final
    assert abs(np.linalg.norm(x) - float(c1[f"{tag}_norm"])) <= tol * float(c1[f"{tag}_norm"])
    s = c1[f"{tag}_sample"]
    assert np.linalg.norm(x.ravel()[::97] - s) <= tol * np.linalg.norm(s)


def test_cyclic_50_updates(problem, c1):
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    res = runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=1, block_height=8, tol=1e-30,
                                                 max_updates=50, engine="simulated"))
    _check(res, c1, "cyc")
    assert res.stop_reason == "budget"


def test_cyclic_150_updates_full_iterate(problem, c1, oracle_mod):
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    res = runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=1, block_height=8, tol=1e-30,
                                                 max_updates=150, engine="simulated"))
    _check(res, c1, "cyc150")
    crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, cfg.lam, cfg.eta, cfg.kappa, cfg.delta)
    x_ref, _, _ = oracle_mod.run_bd3mg(crit, x0, 1, 8, max_updates=150)
    assert np.linalg.norm(res.x_final - x_ref) <= 1e-9 * np.linalg.norm(x_ref)


def test_barrier_jacobi(problem, c1):
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    res = runtime.run(obj, x0, runtime.RunConfig(method="bp3mg", workers=3, block_height=8, tol=1e-30,
                                                 max_updates=24, engine="simulated"))
    _check(res, c1, "jac")


def test_async_two_workers(problem, c1):
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    res = runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=2, block_height=8, tol=1e-30,
                                                 max_updates=12, engine="simulated", seed=5))
    _check(res, c1, "async")
    assert res.tau_hat == max(c1["async_stale"])


def test_barrier_partial_cycle_budget(problem, oracle_mod):
    """workers < blocks and a budget ending mid-cycle: the per-update
    recorder semantics (runtime.py:126-141) on the non-fused apply path."""
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    res = runtime.run(obj, x0, runtime.RunConfig(method="bp3mg", workers=2, block_height=8, tol=1e-30,
                                                 max_updates=7, engine="simulated"))
    crit = oracle_mod.Criterion(obj.psf.kernels, obj.y, cfg.lam, cfg.eta, cfg.kappa, cfg.delta)
    x_ref, log, _ = oracle_mod.run_bp3mg(crit, x0, 2, 8, max_updates=7)
    assert [e.k for e in res.log] == [e[0] for e in log]
    np.testing.assert_allclose([e.f_value for e in res.log], [e[2] for e in log], rtol=1e-10)
    assert np.linalg.norm(res.x_final - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


def test_tolerance_stop_and_descent(problem):
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    res = runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=1, block_height=8, tol=1e-2,
                                                 max_updates=3000, engine="simulated"))
    assert res.stop_reason == "tolerance"
    f = [e.f_value for e in res.log]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(f, f[1:]))


def test_fp32_solve_tracks_fp64(problem):
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    r64 = runtime.run(obj, x0, runtime.RunConfig(method="bp3mg", workers=3, block_height=8, tol=1e-30,
                                                 max_updates=30))
    r32 = runtime.run(obj, x0, runtime.RunConfig(method="bp3mg", workers=3, block_height=8, tol=1e-30,
                                                 max_updates=30, dtype="f32"))
    f64 = np.array([e.f_value for e in r64.log])
    f32 = np.array([e.f_value for e in r32.log])
    assert np.max(np.abs(f32 - f64) / f64) <= 1e-4


def test_live_engine_descends(problem):
    from paper_2002_02328_b200 import runtime
    obj, x0, cfg = problem
    res = runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=2, block_height=8, tol=1e-30,
                                                 max_updates=30, engine="live"))
    assert res.log and res.log[-1].f_value < res.log[0].f_value
    assert len(res.trace) == res.log[-1].k
