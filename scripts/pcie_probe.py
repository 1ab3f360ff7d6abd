"""PCIe probe for the e2e host sweep: pinned H2D / D2H / both directions at
once for one C2 field (33.5 MB), and the session-mode host sweep's time per
call at the pipeline group count given by BD3MG_PIPELINE_GROUPS."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def bw():
    n = 256 * 256 * 64
    h_in = torch.empty(n, dtype=torch.float64, pin_memory=True).fill_(1.0)
    h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.float64, device="cuda")
    d_out = torch.ones(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name in ("h2d", "d2h", "both"):
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(20):
                if name in ("h2d", "both"):
                    with torch.cuda.stream(s1):
                        d_in.copy_(h_in, non_blocking=True)
                if name in ("d2h", "both"):
                    with torch.cuda.stream(s2):
                        h_out.copy_(d_out, non_blocking=True)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 20
        res[name] = {"ms": dt * 1e3, "gbs_per_dir": n * 8 / dt / 1e9}
    return res


def sweep():
    from paper_2002_02328_b200 import configs, objective
    from paper_2002_02328_b200.host import HostProblem, pinned_empty
    from paper_2002_02328_b200.runtime import scheduler
    cfg = configs.CONFIGS[os.environ.get("CFG", "C2")]
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    hp = HostProblem(obj, cfg.dtype, 0)
    blocks = scheduler.partition_blocks(cfg.dims.nz, cfg.block_height)
    x = pinned_empty(x0.shape)
    x[...] = x0
    for _ in range(3):
        hp.jacobi_sweep(x, None, blocks)
    t0 = time.perf_counter()
    for _ in range(20):
        hp.jacobi_sweep(x, None, blocks)
    dt = (time.perf_counter() - t0) / 20
    return {"groups": os.environ.get("BD3MG_PIPELINE_GROUPS", "default"), "ms": dt * 1e3,
            "block_it_s": len(blocks) / dt}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    out = {"sweep": sweep()}
    if "--bw" in sys.argv:
        out["bw"] = bw()
    print(json.dumps(out))
