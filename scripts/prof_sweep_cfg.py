"""Sweeps of a named config (for ncu launch lists):
    python scripts/prof_sweep_cfg.py C3 [reps] [jacobi|cyclic|incremental]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_02328_b200 import configs, objective, runtime

cfg = configs.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dt = torch.float64 if cfg.dtype == "f64" else torch.float32
psf, truth, y, x0, params = configs.make_problem(cfg)
mode = sys.argv[3] if len(sys.argv) > 3 else "jacobi"
obj = objective.Objective(psf, y, params)
if mode == "cyclic":
    eng = runtime.CyclicSweeper(obj, x0, cfg.block_height, dt)
else:
    eng = runtime.JacobiSweeper(obj, x0, cfg.block_height, dt, incremental=mode == "incremental", refresh_every=0)
for _ in range(reps):
    eng.sweep()
torch.cuda.synchronize()
print("done", cfg.name)
