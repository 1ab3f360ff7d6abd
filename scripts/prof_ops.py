"""Small driver for ncu captures of single operators at BASELINE C2 size.

    python scripts/prof_ops.py [H|Ht|step] [f64|f32] [reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2002_02328_b200 import blur, configs, objective, runtime

op = sys.argv[1] if len(sys.argv) > 1 else "H"
dt = torch.float64 if (sys.argv[2] if len(sys.argv) > 2 else "f64") == "f64" else torch.float32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = configs.CONFIGS["C2"]
psf = blur.depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
x = torch.rand(cfg.dims.shape, dtype=dt, device="cuda")
out = torch.empty_like(x)
if op in ("H", "Ht"):
    for _ in range(reps):
        blur.correlate_rows(psf, x, 0, 0, cfg.dims.nz - 1, op == "Ht", out=out)
else:
    y = torch.rand(cfg.dims.shape, dtype=torch.float64).numpy()
    obj = objective.Objective(psf, y, objective.RegParams(lam=cfg.lam, eta=cfg.eta, kappa=cfg.kappa, delta=cfg.delta))
    eng = runtime.JacobiSweeper(obj, x, cfg.block_height, dt)
    for _ in range(reps):
        eng.sweep()
torch.cuda.synchronize()
print("done", op)
