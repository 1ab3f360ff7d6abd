"""Does an HBM-bound smem-free kernel overlap the FP64 correlation?  H on
stream A, a torch elementwise pass (no shared memory) over ~100 MB on
stream B: serial vs concurrent time (C2 fp64)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_02328_b200 import blur, configs, objective  # noqa: E402

cfg = configs.CONFIGS["C2"]
psf, truth, y, x0, params = configs.make_problem(cfg)
x = torch.from_numpy(x0).cuda()
out = torch.empty_like(x)
a = torch.rand(3 * x.numel(), dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def h():
    with torch.cuda.stream(sa):
        blur.apply_H(psf, x)


def ew():
    with torch.cuda.stream(sb):
        a.mul_(1.0000001)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def both():
    h()
    ew()


def serial():
    h()
    torch.cuda.synchronize()
    ew()
    torch.cuda.synchronize()


print(f"H alone {t(h):.1f} us, elementwise alone {t(ew):.1f} us, serial {t(serial):.1f} us, concurrent {t(both):.1f} us")
