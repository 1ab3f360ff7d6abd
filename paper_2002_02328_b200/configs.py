"""BASELINE.json workload configurations C1-C5 as seeded synthetic inputs.

No public dataset is used: the paper's FlyBrain/Aneurysm volumes are not
available, so every config is a seeded ellipsoid phantom blurred by the
depth-variant Gaussian PSF family of BASELINE.json, plus i.i.d. Gaussian
noise, with x0 ~ U[0, max(y)] (reference cli.py:152-156).  All draws are
numpy Philox streams, so the oracle and the GPU path consume identical
arrays.  The BASELINE regulariser has no axial weight; the reference's
mandatory kappa takes its default 0.05 (objective.py:53).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .volume import Dims3, add_gaussian_noise, ellipsoid_phantom, init_uniform


@dataclass(frozen=True)
class Config:
    name: str
    dims: Dims3                 # (nx, ny, nz)
    kdims: tuple[int, int, int]  # (kx, ky, kz)
    sigma_xy: tuple[float, float]
    sigma_z: tuple[float, float]
    n_ellipsoids: int
    amplitude: str
    noise: float
    lam: float
    delta: float
    eta: float
    kappa: float
    block_height: int
    dtype: str                  # "f64" / "f32"
    iterations: int
    seed: int = 0


CONFIGS = {
    # CPU-oracle size: 3 blocks of 8, cyclic schedule, 50 iterations
    "C1": Config("C1", Dims3(64, 64, 24), (5, 5, 11), (0.8, 2.0), (1.5, 2.5), 40, "uniform", 0.02,
                 1e-2, 1e-2, 1e-1, 0.05, 8, "f64", 50),
    # single-GPU operator bench (fp64 headline; fp32 variant below)
    "C2": Config("C2", Dims3(256, 256, 64), (5, 5, 11), (0.8, 2.0), (1.5, 2.5), 40, "uniform", 0.02,
                 1e-2, 1e-2, 1e-1, 0.05, 8, "f64", 10),
    "C2f32": Config("C2f32", Dims3(256, 256, 64), (5, 5, 11), (0.8, 2.0), (1.5, 2.5), 40, "uniform", 0.02,
                    1e-2, 1e-2, 1e-1, 0.05, 8, "f32", 10),
    # microscopy-scale, sync cyclic, 8 blocks of 16
    "C3": Config("C3", Dims3(512, 512, 128), (7, 7, 15), (1.0, 3.0), (1.5, 2.5), 200, "gamma", 0.01,
                 1e-2, 1e-2, 1e-1, 0.05, 16, "f32", 200),
    # async: 32 blocks of 8
    "C4": Config("C4", Dims3(512, 512, 256), (7, 7, 15), (1.0, 3.0), (1.5, 2.5), 200, "gamma", 0.01,
                 1e-2, 1e-2, 1e-1, 0.05, 8, "f32", 200),
    # large scaling sweep: 8 blocks of 64
    "C5": Config("C5", Dims3(1024, 1024, 512), (9, 9, 21), (1.0, 4.0), (2.0, 3.5), 400, "gamma", 0.01,
                 5e-3, 1e-2, 1e-1, 0.05, 64, "f32", 500),
}


def depth_variant_params(nz: int, sigma_xy: tuple[float, float], sigma_z: tuple[float, float]) -> np.ndarray:
    """BASELINE.json PSF family, one (sigma1, sigma2, sigma3, phi, theta)
    record per output plane: axis-aligned, sigma_xy and sigma_z linear in
    t = z/(nz-1).  Torch-free, shared by the GPU arm (blur.depth_variant_stack)
    and bench.py's reference arm (which builds the kernels with the
    reference's own gaussian_kernel)."""
    params = np.empty((nz, 5))
    for z in range(nz):
        t = z / (nz - 1) if nz > 1 else 0.0
        sxy = sigma_xy[0] + (sigma_xy[1] - sigma_xy[0]) * t
        sz = sigma_z[0] + (sigma_z[1] - sigma_z[0]) * t
        params[z] = (sxy, sxy, sz, 0.0, 0.0)
    return params


def truth_of(cfg: Config) -> np.ndarray:
    return ellipsoid_phantom(cfg.dims, cfg.n_ellipsoids, cfg.seed + 1, cfg.amplitude)


def make_problem(cfg: Config | str, y_from=None):
    """(psf, truth, y, x0, params) for a config.  ``y_from(psf, truth)``
    computes H(truth) (defaults to the GPU apply_H)."""
    from .blur import apply_H, depth_variant_stack
    from .objective import RegParams

    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    psf = depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
    truth = truth_of(cfg)
    if y_from is None and cfg.dtype == "f32":
        # fp32 configs: the observation is blurred in fp32 on the GPU (the fp64
        # H of C5 alone is ~1.7 TFLOP); every consumer reads this same y
        import torch
        y_from = lambda p, t: apply_H(p, torch.from_numpy(t).cuda().float()).double().cpu().numpy()
    blurred = (y_from or apply_H)(psf, truth)
    y = add_gaussian_noise(blurred, cfg.noise, cfg.seed + 2)
    x0 = init_uniform(cfg.dims, float(np.max(y)), cfg.seed + 3)
    params = RegParams(lam=cfg.lam, eta=cfg.eta, kappa=cfg.kappa, delta=cfg.delta, x_min=0.0, x_max=1.0)
    return psf, truth, y, x0, params
