"""CUDA-event timing of single operators at C2 size (no profiler).

    python scripts/time_ops.py [f64|f32]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_02328_b200 import blur, configs

dt = torch.float64 if (sys.argv[1] if len(sys.argv) > 1 else "f64") == "f64" else torch.float32
cfg = configs.CONFIGS["C2"]
psf = blur.depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
x = torch.rand(cfg.dims.shape, dtype=dt, device="cuda")
out = torch.empty_like(x)
fl = blur.flops_H(cfg.dims, psf.kdims)
for adj in (False, True):
    for _ in range(3):
        blur.correlate_rows(psf, x, 0, 0, cfg.dims.nz - 1, adj, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(20):
        blur.correlate_rows(psf, x, 0, 0, cfg.dims.nz - 1, adj, out=out)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20
    print(f"{'Ht' if adj else 'H '} {t * 1e3:8.1f} us  {fl / t / 1e9:6.2f} TFLOP/s")
