"""Run one H case in a fresh process: python scripts/tma_probe.py nx ny nz k [dtype]."""
import subprocess
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def one(nx, ny, nz, k, dt):
    import numpy as np
    import torch
    from paper_2002_02328_b200 import blur
    from paper_2002_02328_b200.volume import Dims3
    psf = blur.generate_psf_stack(Dims3(nx, ny, nz), blur.KernelDims(k, k, 3), seed=1)
    x = torch.rand((nz, ny, nx), dtype=torch.float64 if dt == "f64" else torch.float32, device="cuda")
    out = blur.correlate_rows(psf, x, 0, 0, nz - 1, False)
    torch.cuda.synchronize()
    print("ok", float(out.sum()))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(*map(int, sys.argv[1:5]), sys.argv[5] if len(sys.argv) > 5 else "f64")
    else:
        for case in ["12 8 12 3", "12 8 12 5", "256 256 8 3", "256 256 8 5", "256 8 8 5", "8 256 8 5", "40 136 8 5",
                     "36 132 8 5", "34 130 8 3", "64 64 8 3", "64 64 8 5", "48 48 8 5", "256 256 8 7", "256 256 8 9",
                     "12 8 12 5 f32", "256 256 8 5 f32", "256 256 8 3 f32"]:
            r = subprocess.run([sys.executable, __file__, *case.split()], capture_output=True, text=True, timeout=120)
            print(case, "->", (r.stdout.strip().splitlines() or ["?"])[-1] if r.returncode == 0 else "FAIL " + (r.stderr.strip().splitlines() or ["?"])[-1][:80], flush=True)
