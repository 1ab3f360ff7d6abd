"""H on a named config (for ncu):  python scripts/prof_h_cfg.py C3 [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_02328_b200 import blur, configs

cfg = configs.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dt = torch.float64 if cfg.dtype == "f64" else torch.float32
psf = blur.depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
x = torch.rand(cfg.dims.shape, dtype=dt, device="cuda")
out = torch.empty_like(x)
for _ in range(reps):
    blur.correlate_rows(psf, x, 0, 0, cfg.dims.nz - 1, False, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    blur.correlate_rows(psf, x, 0, 0, cfg.dims.nz - 1, False, out=out)
e.record()
torch.cuda.synchronize()
t = s.elapsed_time(e) / reps / 1e3
print(f"{cfg.name} H {t * 1e3:.3f} ms {blur.flops_H(cfg.dims, psf.kdims) / t / 1e12:.2f} TFLOP/s")
