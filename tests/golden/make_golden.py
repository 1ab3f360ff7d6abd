"""Generate the golden vectors that pin the oracle, FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    make -C oracle ref          # reference Cython core -> oracle/_ref
    python tests/golden/make_golden.py

Imports the unmodified reference package from /root/reference/pkg/src with
its compiled core (oracle/_ref/_core*.so, built from the reference's own
_core.pyx) and records inputs + outputs as .npz fixtures.  The fixtures are
committed; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import importlib.util
import sys
import sysconfig
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")


def load_reference():
    core = ROOT / "oracle" / "_ref" / ("_core" + sysconfig.get_config_var("EXT_SUFFIX"))
    if core.exists():
        spec = importlib.util.spec_from_file_location("bd3mg._core", core)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        sys.modules["bd3mg._core"] = mod
    sys.path.insert(0, str(REF_SRC))
    import bd3mg  # noqa: F401
    from bd3mg import blur, directions, kernels, objective, runtime, volume
    return blur, directions, kernels, objective, runtime, volume


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def philox(seed):
    return np.random.Generator(np.random.Philox(seed))


def blur_cases(blur, kernels, volume):
    cases = {}
    specs = [  # (dims (nx,ny,nz), kdims (kx,ky,kz), seed)
        ((10, 9, 8), (5, 3, 5), 6),
        ((8, 8, 6), (3, 5, 3), 2),
        ((12, 8, 12), (3, 3, 3), 5),
        ((33, 21, 9), (5, 5, 5), 7),
        ((37, 35, 14), (5, 5, 11), 8),
        ((24, 22, 10), (7, 7, 7), 9),
        ((21, 19, 12), (9, 9, 5), 10),
        ((6, 5, 4), (1, 1, 3), 1),
    ]
    for i, (dims, kd, seed) in enumerate(specs):
        psf = blur.generate_psf_stack(volume.Dims3(*dims), blur.KernelDims(*kd), seed=seed)
        rng = philox(100 + i)
        shape = (dims[2], dims[1], dims[0])
        x = rng.standard_normal(shape)
        v = rng.standard_normal(shape)
        nz = dims[2]
        lo, hi = nz // 3, max(nz // 3, (2 * nz) // 3)
        f0, f1 = max(0, lo - kd[2]), min(nz - 1, hi + kd[2] - 1)
        cases[f"blur{i}"] = dict(
            kernels=psf.kernels, params=psf.params, x=x, v=v,
            Hx=blur.apply_H(psf, x), Htv=blur.apply_Ht(psf, v),
            rows=np.array([lo, hi, f0, f1]),
            Hrows=blur.apply_H_rows(psf, x[f0:f1 + 1], f0, lo, hi),
            Htrows=blur.apply_Ht_rows(psf, v[f0:f1 + 1], f0, lo, hi),
            backend=np.array(kernels.backend_name()))
    return cases


def objective_cases(blur, directions, objective, volume):
    cases = {}
    specs = [  # (dims, kdims, blocks, params)
        ((6, 6, 4), (3, 3, 3), [(0, 3), (1, 2), (3, 3)], dict()),
        ((8, 7, 10), (3, 3, 5), [(4, 5), (0, 0), (9, 9), (0, 9)], dict(lam=0.07)),
        ((20, 18, 24), (5, 5, 11), [(0, 7), (8, 15), (16, 23)],
         dict(lam=1e-2, delta=1e-2, eta=1e-1, kappa=0.05)),
        ((9, 1, 5), (3, 1, 3), [(1, 3)], dict()),
        ((1, 7, 5), (1, 3, 3), [(2, 2)], dict()),
    ]
    for i, (dims, kd, blocks, pk) in enumerate(specs):
        d3 = volume.Dims3(*dims)
        ranges = blur.ParamRanges(sigma1=(0.6, 1.1), sigma2=(0.6, 1.1), sigma3=(0.6, 1.1))
        psf = blur.generate_psf_stack(d3, blur.KernelDims(*kd), ranges, 3 + i)
        truth = volume.phantom(d3, 7 + i)
        y = volume.add_gaussian_noise(blur.apply_H(psf, truth), 0.05, 11 + i)
        params = objective.RegParams(**pk)
        obj = objective.Objective(psf, y, params)
        rng = philox(200 + i)
        x = rng.uniform(-0.2, 1.2, d3.shape)
        case = dict(kernels=psf.kernels, y=y, x=x,
                    reg=np.array([params.lam, params.eta, params.kappa, params.delta,
                                  params.x_min, params.x_max]),
                    f=np.array(objective.eval_f(obj, x)), grad=objective.grad_f(obj, x),
                    blocks=np.array(blocks))
        for j, (lo, hi) in enumerate(blocks):
            blk = volume.SliceBlock(lo, hi)
            slab = blur.slab_support(psf, blk)
            frag = x[slab.z_lo:slab.z_hi + 1]
            n = blk.count(d3)
            vj = rng.standard_normal(n)
            dmem = 0.01 * rng.standard_normal(n)
            maj = objective.MajorantOperator(obj, frag, blk, slab.z_lo)
            g = objective.grad_block(obj, frag, blk, slab.z_lo)
            info = directions.subspace_step(g, dmem, maj.apply)
            info0 = directions.subspace_step(g, np.zeros(n), maj.apply)
            case.update({
                f"b{j}_gblock": g, f"b{j}_v": vj, f"b{j}_Av": maj.apply(vj), f"b{j}_omega": maj.omega,
                f"b{j}_dmem": dmem, f"b{j}_inc": info.increment, f"b{j}_gram": info.gram,
                f"b{j}_rhs": info.rhs, f"b{j}_coeffs": info.coeffs, f"b{j}_inc0": info0.increment,
                f"b{j}_gram0": info0.gram,
            })
        cases[f"obj{i}"] = case
    return cases


def c1_case(blur, objective, runtime, volume):
    """BASELINE config C1 run by the reference (cyclic bd3mg and bp3mg)."""
    sys.path.insert(0, str(ROOT))
    from paper_2002_02328_b200 import configs

    cfg = configs.CONFIGS["C1"]
    nz = cfg.dims.nz
    kd = blur.KernelDims(*cfg.kdims)
    stack = np.empty((nz, kd.kz, kd.ky, kd.kx))
    par = np.empty((nz, 5))
    for z in range(nz):
        t = z / (nz - 1)
        sxy = cfg.sigma_xy[0] + (cfg.sigma_xy[1] - cfg.sigma_xy[0]) * t
        sz = cfg.sigma_z[0] + (cfg.sigma_z[1] - cfg.sigma_z[0]) * t
        stack[z] = blur.gaussian_kernel(kd, sxy, sxy, sz, 0.0, 0.0)
        par[z] = (sxy, sxy, sz, 0.0, 0.0)
    psf = blur.PsfStack(volume.Dims3(*cfg.dims), kd, stack, par)
    truth = configs.truth_of(cfg)
    y = volume.add_gaussian_noise(blur.apply_H(psf, truth), cfg.noise, cfg.seed + 2)
    x0 = volume.init_uniform(volume.Dims3(*cfg.dims), float(np.max(y)), cfg.seed + 3)
    params = objective.RegParams(lam=cfg.lam, eta=cfg.eta, kappa=cfg.kappa, delta=cfg.delta)
    obj = objective.Objective(psf, y, params)
    # large arrays are pinned by SHA-256 + norms + a strided sample (the
    # oracle reproduces them bitwise); the kernel stack is stored in full
    out = dict(kernels=stack, y_sha=np.array(sha(y)), x0_sha=np.array(sha(x0)), y_sample=y.ravel()[::97],
               truth_sum=np.array(truth.sum()),
               reg=np.array([params.lam, params.eta, params.kappa, params.delta, 0.0, 1.0]))

    def record(tag, r):
        out.update({f"{tag}_sha": np.array(sha(r.x_final)), f"{tag}_norm": np.array(np.linalg.norm(r.x_final)),
                    f"{tag}_sample": r.x_final.ravel()[::97], f"{tag}_k": np.array([e.k for e in r.log]),
                    f"{tag}_f": np.array([e.f_value for e in r.log]), f"{tag}_grants": np.array(r.grant_log),
                    f"{tag}_stale": np.array([ev.staleness for ev in r.trace])})

    record("cyc", runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=1, block_height=8, tol=1e-30,
                                                         max_updates=cfg.iterations, engine="simulated")))
    record("cyc150", runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=1, block_height=8,
                                                            tol=1e-30, max_updates=150, engine="simulated")))
    record("jac", runtime.run(obj, x0, runtime.RunConfig(method="bp3mg", workers=3, block_height=8, tol=1e-30,
                                                         max_updates=24, engine="simulated")))
    record("async", runtime.run(obj, x0, runtime.RunConfig(method="bd3mg", workers=2, block_height=8,
                                                           tol=1e-30, max_updates=12, engine="simulated",
                                                           seed=5)))
    return out


def ablation_cases(blur, directions, objective, volume):
    """The ablation directions and the Lipschitz estimate (directions.py:97-168,
    objective.py:301-375) as the reference computes them."""
    import warnings
    out = {}
    for i, (dims, kd, seed) in enumerate([((12, 10, 16), (3, 3, 5), 3), ((9, 11, 12), (5, 5, 3), 4)]):
        d3 = volume.Dims3(*dims)
        ranges = blur.ParamRanges(sigma1=(0.6, 1.1), sigma2=(0.6, 1.1), sigma3=(0.6, 1.1))
        psf = blur.generate_psf_stack(d3, blur.KernelDims(*kd), ranges, seed)
        truth = volume.phantom(d3, 20 + i)
        y = volume.add_gaussian_noise(blur.apply_H(psf, truth), 0.05, 30 + i)
        params = objective.RegParams(lam=1e-2, eta=1e-1, kappa=0.05, delta=1e-2)
        obj = objective.Objective(psf, y, params)
        rng = philox(300 + i)
        x = rng.uniform(-0.2, 1.2, d3.shape)
        L = objective.lipschitz_estimate(obj)
        case = dict(kernels=psf.kernels, y=y, x=x, reg=np.array([params.lam, params.eta, params.kappa, params.delta,
                                                                  params.x_min, params.x_max]),
                    rho=np.array(objective.rho_hth_estimate(psf)),
                    rho3=np.array(objective.rho_hth_estimate(psf, iters=3, seed=1)),
                    norm_bound=np.array(objective.operator_norm_bound(psf)), L=np.array(L))
        for j, (lo, hi) in enumerate([(4, 7), (0, 2)]):
            blk = volume.SliceBlock(lo, hi)
            slab = blur.slab_support(psf, blk)
            frag = x[slab.z_lo:slab.z_hi + 1]
            n = blk.count(d3)
            dmem = 0.01 * rng.standard_normal(n)
            g = objective.grad_block(obj, frag, blk, slab.z_lo)
            maj = objective.MajorantOperator(obj, frag, blk, slab.z_lo)
            case[f"b{j}_blk"] = np.array([lo, hi])
            case[f"b{j}_dmem"] = dmem
            case[f"b{j}_gd"] = directions.gd_direction(obj, frag, slab.z_lo, blk, L)
            case[f"b{j}_cg"] = directions.cg_direction(obj, frag, slab.z_lo, blk, dmem, L)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                case[f"b{j}_mm"] = directions.mm_direction(obj, frag, slab.z_lo, blk, cg_tol=1e-8, cg_maxit=200)
            for tag, tol, maxit in (("conv", 1e-10, 400), ("budget", 1e-12, 4)):
                xs, conv, iters, relres = directions.cg_solve(maj.apply, -g, tol, maxit)
                case[f"b{j}_cg_{tag}_x"] = xs
                case[f"b{j}_cg_{tag}_meta"] = np.array([float(conv), float(iters), relres, tol, float(maxit)])
        out[f"abl{i}"] = case
    return out


def io_cases(blur, volume):
    """Container files written by the reference's own writers
    (volume.py:104-114, blur.py:201-211) plus the arrays they hold."""
    d = OUT / "io"
    d.mkdir(exist_ok=True)
    vol = philox(41).uniform(-2.0, 3.0, (3, 4, 5))          # (nz, ny, nx)
    volume.write_volume(vol, d / "vol_5x4x3.bd3mgvol")
    idx = np.arange(8, dtype=np.float64).reshape(2, 2, 2)
    volume.write_volume(idx, d / "vol_2x2x2.bd3mgvol")
    psf = blur.generate_psf_stack(volume.Dims3(6, 5, 4), blur.KernelDims(3, 3, 5), seed=7)
    blur.write_psf(psf, d / "psf_6x5x4_k3x3x5.bd3mgpsf")
    np.savez_compressed(d / "io.npz", vol=vol, idx=idx, psf_kernels=psf.kernels, psf_params=psf.params)


def main():
    blur, directions, kernels, objective, runtime, volume = load_reference()
    if "--only-io" in sys.argv:
        io_cases(blur, volume)
        return
    print("reference backend:", kernels.backend_name())
    if "--only-ablation" in sys.argv:
        ab = ablation_cases(blur, directions, objective, volume)
        np.savez_compressed(OUT / "ablation.npz", **{f"{c}/{k}": v for c, d in ab.items() for k, v in d.items()})
        return
    cases = {}
    cases.update(blur_cases(blur, kernels, volume))
    np.savez_compressed(OUT / "blur.npz", **{f"{c}/{k}": v for c, d in cases.items() for k, v in d.items()})
    oc = objective_cases(blur, directions, objective, volume)
    np.savez_compressed(OUT / "objective.npz", **{f"{c}/{k}": v for c, d in oc.items() for k, v in d.items()})
    ab = ablation_cases(blur, directions, objective, volume)
    np.savez_compressed(OUT / "ablation.npz", **{f"{c}/{k}": v for c, d in ab.items() for k, v in d.items()})
    if "--only-ablation" in sys.argv:
        return
    c1 = c1_case(blur, objective, runtime, volume)
    np.savez_compressed(OUT / "c1.npz", **c1)
    io_cases(blur, volume)
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
