"""Variant probe for the separable-PSF fast path (csrc/separable.cu): times
full-volume H / H^T for each depth-FIR (BD3MG_SEP_Z) and 2-D filter
(BD3MG_SEP_XY) variant at the C2 / C3 / C5 shapes, and checks every variant
is bitwise equal to the first (same sums, same order).  Writes one JSON line
per (config, direction, variant) to stdout."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2002_02328_b200 import blur, separable  # noqa: E402
from paper_2002_02328_b200.volume import Dims3  # noqa: E402

SHAPES = {"C2": ((256, 256, 64), 5, 11, torch.float64), "C3": ((512, 512, 128), 7, 15, torch.float32),
          "C5": ((1024, 1024, 512), 9, 21, torch.float32)}
VARIANTS = [("1", "8160"), ("2", "8160"), ("2", "8161"), ("2", "8080"), ("2", "8081"), ("2", "16081"),
            ("2", "16161"), ("3", "16161"), ("3", "8160"), ("5", "16161")]


def main():
    peak = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))["hbm_gbs"]
    names = sys.argv[1:] or list(SHAPES)
    variants = VARIANTS
    if os.environ.get("SEP_PROBE_VARIANT"):  # e.g. "2:16161" (one variant, for ncu captures)
        variants = [tuple(os.environ["SEP_PROBE_VARIANT"].split(":"))]
    for name in names:
        (nx, ny, nz), k, kz, dt = SHAPES[name]
        dims = Dims3(nx, ny, nz)
        sep = separable.SeparableStack.from_psf(blur.depth_variant_stack(dims, (k, k, kz), (0.8, 2.0), (1.0, 2.5)))
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand(dims.shape, dtype=dt, device="cuda", generator=g)
        out = torch.empty_like(x)
        nbytes = separable.bytes_H(dims, x.element_size())
        for adj in (False, True):
            ref = None
            for xy, zv in variants:
                os.environ["BD3MG_SEP_XY"], os.environ["BD3MG_SEP_Z"] = xy, zv
                for _ in range(3):
                    sep.correlate_rows(x, 0, 0, nz - 1, adjoint=adj, out=out)
                torch.cuda.synchronize()
                if ref is None:
                    ref = out.clone()
                same = bool(torch.equal(out, ref))
                reps = 20 if name != "C5" else 8
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(reps):
                    sep.correlate_rows(x, 0, 0, nz - 1, adjoint=adj, out=out)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e) / reps
                print(json.dumps({"config": name, "adjoint": adj, "xy": xy, "z": zv, "ms": round(ms, 4),
                                  "gbs": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / peak, 3),
                                  "bitwise_equal_to_first": same}), flush=True)


if __name__ == "__main__":
    main()
