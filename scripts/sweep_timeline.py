"""Kernel timeline of graph-replayed block-Jacobi sweeps (torch.profiler / CUPTI):
    python scripts/sweep_timeline.py C2 [sweeps] [jacobi|cyclic]
Prints, per kernel of the last replayed sweep, start / end relative to the sweep's first kernel and the
stream it ran on: shows what actually overlaps inside the captured graph (ncu serialises launches)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2002_02328_b200 import configs, objective, runtime

cfg = configs.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dt = torch.float64 if cfg.dtype == "f64" else torch.float32
psf, truth, y, x0, params = configs.make_problem(cfg)
obj = objective.Objective(psf, y, params)
mode = sys.argv[3] if len(sys.argv) > 3 else "jacobi"
eng = (runtime.CyclicSweeper if mode == "cyclic" else runtime.JacobiSweeper)(obj, x0, cfg.block_height, dt)
import os
eng.sweep()
if not os.environ.get("TIMELINE_EAGER"):
    eng.capture()
for _ in range(3):
    eng.sweep()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(reps):
        eng.sweep()
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name]
ev.sort(key=lambda e: e.time_range.start)
# split into sweeps by the large gaps of the host synchronize
sweeps, cur = [], []
for e in ev:
    if cur and e.time_range.start - max(x.time_range.end for x in cur) > 50:
        sweeps.append(cur)
        cur = []
    cur.append(e)
sweeps.append(cur)
last = sweeps[-1]
t0 = min(e.time_range.start for e in last)
print(f"# {cfg.name}: {len(sweeps)} sweeps traced; last sweep: {len(last)} kernels, "
      f"{max(e.time_range.end for e in last) - t0:.1f} us")
print("| start us | end us | dur us | stream | kernel |")
print("|---:|---:|---:|---:|---|")
for e in last:
    name = e.name.replace("bd3mg::", "").replace("void ", "")[:70]
    stream = getattr(e, "stream", None)
    print(f"| {e.time_range.start - t0:.1f} | {e.time_range.end - t0:.1f} | {e.time_range.end - e.time_range.start:.1f} | "
          f"{stream if stream is not None else ''} | `{name}` |")
