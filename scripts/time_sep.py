"""Separable-PSF fast path timing vs the dense kernels (python scripts/time_sep.py C2 [C5 ...])."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_02328_b200 import blur, configs, separable

peak = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))["hbm_gbs"]
for name in sys.argv[1:] or ["C2"]:
    cfg = configs.CONFIGS[name]
    dt = torch.float64 if cfg.dtype == "f64" else torch.float32
    psf = blur.depth_variant_stack(cfg.dims, cfg.kdims, cfg.sigma_xy, cfg.sigma_z)
    sep = separable.SeparableStack.from_psf(psf)
    x = torch.rand(cfg.dims.shape, dtype=dt, device="cuda")
    out = torch.empty_like(x)
    nz = cfg.dims.nz
    nbytes = separable.bytes_H(cfg.dims, x.element_size())
    for adj in (False, True):
        for label, fn in (("dense", lambda: blur.correlate_rows(psf, x, 0, 0, nz - 1, adj, out=out)),
                          ("sep", lambda: sep.correlate_rows(x, 0, 0, nz - 1, adjoint=adj, out=out))):
            for _ in range(3):
                fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for _ in range(10):
                fn()
            e.record()
            torch.cuda.synchronize()
            t = s.elapsed_time(e) / 10 / 1e3
            print(f"{name} {'Ht' if adj else 'H '} {label:5s} {t * 1e6:9.1f} us  {nbytes / t / 1e9:7.0f} GB/s "
                  f"({nbytes / t / 1e9 / peak:.2f} of HBM)")
