"""Per-item timeline of the persistent sweep (BD3MG_PK_TRACE=1): runs a few
C2 sweeps, dumps the last one's item records to gpurun_out/pk_trace.npz and
prints a per-type summary (count, mean run time, mean dependency wait,
first start / last end relative to the sweep start).

    BD3MG_PK_TRACE=1 python scripts/pk_trace.py [CONFIG]
"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("BD3MG_PK_TRACE", "1")
os.environ.setdefault("BD3MG_PK", "1")

from paper_2002_02328_b200 import _native as N, configs, objective, runtime  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = configs.CONFIGS[name]
psf, truth, y, x0, params = configs.make_problem(cfg)
obj = objective.Objective(psf, y, params)
dt = torch.float64 if cfg.dtype == "f64" else torch.float32
eng = runtime.JacobiSweeper(obj, x0, cfg.block_height, dt)
for _ in range(4):
    eng.sweep()
torch.cuda.synchronize()
n = C.c_int64()
N.check(N.lib.bd3mg_pk_trace(None, 0, C.byref(n)))
buf = np.zeros((n.value, 4), dtype=np.uint64)
N.check(N.lib.bd3mg_pk_trace(buf.ctypes.data, n.value, C.byref(n)))
t0 = buf[:, 0].min()
deq = (buf[:, 0] - t0) / 1e3
go = (buf[:, 1] - t0) / 1e3
end = (buf[:, 2] - t0) / 1e3
meta = buf[:, 3]
sm = (meta >> 48).astype(int)
typ = ((meta >> 40) & 0xff).astype(int)
blk = ((meta >> 32) & 0xff).astype(int)
z = ((meta >> 16) & 0xffff).astype(int)
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
np.savez(out / f"pk_trace_{name}.npz", deq=deq, go=go, end=end, sm=sm, type=typ, b=blk, z=z)
names = ["GREG", "RESID", "GRAD", "RG", "GRAM", "SOLVE", "UPD", "RED"]
print(f"{name}: {n.value} items, sweep span {end.max():.1f} us")
for t in range(8):
    m = typ == t
    if not m.any():
        continue
    run = end[m] - go[m]
    wait = go[m] - deq[m]
    print(f"{names[t]:6s} n={m.sum():6d} run mean {run.mean():7.2f} us  sum {run.sum():9.0f}  wait mean {wait.mean():6.2f} "
          f"sum {wait.sum():8.0f}  first {deq[m].min():7.1f}  last end {end[m].max():7.1f}")
busy = (end - go).sum()
print(f"slot-time busy {busy:.0f} us of {444 * end.max():.0f} ({busy / (444 * end.max()):.2f}); waits {(go - deq).sum():.0f} us")
