"""Run each golden blur case through H / H^T with a sync after every call."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
from conftest import golden
from paper_2002_02328_b200 import blur

for name, c in golden("blur").items():
    nz, ny, nx = c["x"].shape
    k = c["kernels"]
    psf = blur.PsfStack((nx, ny, nz), (k.shape[3], k.shape[2], k.shape[1]), k)
    for adj in (False, True):
        print(name, c["x"].shape, k.shape, "adj" if adj else "fwd", flush=True)
        out = blur.correlate_rows(psf, torch.from_numpy(c["x"]).cuda(), 0, 0, nz - 1, adj)
        torch.cuda.synchronize()
        ref = c["Htv"] if adj else c["Hx"]
        src = c["v"] if adj else c["x"]
        out = blur.correlate_rows(psf, torch.from_numpy(src).cuda(), 0, 0, nz - 1, adj).cpu().numpy()
        print("   err", np.abs(out - ref).max(), flush=True)
