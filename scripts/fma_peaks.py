"""FMA-pipe peaks: DFMA, FFMA and packed FFMA2 (python scripts/fma_peaks.py)."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2002_02328_b200 import _native as N

out = torch.empty(148 * 8 * 256, dtype=torch.float64, device="cuda")
for name, dt in (("f64 DFMA", 0), ("f32 FFMA", 1), ("f32 FFMA2", 2)):
    fl = ctypes.c_double()
    best = 0.0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        N.check(N.lib.bd3mg_fma_probe(dt, 148 * 8, 4000, out.data_ptr(), ctypes.byref(fl), None))
        e.record()
        torch.cuda.synchronize()
        best = max(best, fl.value / (s.elapsed_time(e) * 1e-3) / 1e12)
    print(f"{name}: {best:.1f} TFLOP/s")
