"""BASELINE config C4 (512 x 512 x 256 fp32, 32 blocks of 8 planes): objective
against block-iterations for the three schedules, and against wall-clock
projected from measured per-update device times on one B200.

  * sync   : block-Jacobi sweeps (every block at a common anchor per cycle)
  * cyclic : the reference's deterministic single-worker order
  * async  : 8 virtual ranks (4 blocks each) on peer halo rings, a seeded
             random schedule that keeps every rank within the delay bound 2

The async ranks run on one GPU, so their wall-clock is projected: 8 ranks
run concurrently on 8 GPUs, so the time for U updates is U/8 of the
measured per-update time (halo rings included; the all-rank barrier-free
schedule has no other cost).  The sync projection uses the measured
per-rank sweep time of the 8-way layout (scripts/scaling_projection.py
method).  Output: one JSON object on stdout.

    python scripts/convergence_c4.py [sweeps]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2002_02328_b200 import configs, objective, runtime  # noqa: E402
from paper_2002_02328_b200.distributed import (AsyncShard, RingHub, RingPlan, ShardedJacobi,  # noqa: E402
                                               SlabLayout, cuda_block_step, ring_slots)


def f_of(obj, x):
    return float(objective.eval_terms(obj, x)[4].item())


def main():
    sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cfg = configs.CONFIGS["C4"]
    dtype = torch.float32
    psf, truth, y, x0, params = configs.make_problem(cfg)
    obj = objective.Objective(psf, y, params)
    B = -(-cfg.dims.nz // cfg.block_height)
    out = {"config": "C4 512x512x256 fp32, 32 blocks x 8 planes, PSF 7x7x15", "f0": f_of(obj, torch.from_numpy(x0).cuda().float())}

    # sync (block-Jacobi) and cyclic: f after every sweep of B block-iterations
    for name, eng in (("sync", runtime.JacobiSweeper(obj, x0, cfg.block_height, dtype)),
                      ("cyclic", runtime.CyclicSweeper(obj, x0, cfg.block_height, dtype))):
        eng.sweep()
        eng.capture()
        fs, its = [], []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(sweeps):
            eng.sweep()
            torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / sweeps
        # replay from x0 for the curve (the timing loop above moved the iterate)
        eng2 = (runtime.JacobiSweeper if name == "sync" else runtime.CyclicSweeper)(obj, x0, cfg.block_height, dtype)
        for k in range(sweeps + 1):
            eng2.sweep()
            if k > 0 or name == "cyclic":
                fs.append(eng2.f())
                its.append((k if name == "sync" else k + 1) * B)
        out[name] = {"block_iterations": its, "f": fs, "ms_per_sweep_1gpu": dt * 1e3}

    # sync at 8 GPUs: per-rank sweep time of the 8-way layout (slowest rank)
    shards = [ShardedJacobi(obj, x0, cfg.block_height, dtype, rank=r, world=8, halo="p2p") for r in range(8)]
    bases = {r: s.peer.ptr for r, s in enumerate(shards)}
    for s in shards:
        s.peer.connect(bases)
    for s in shards:
        s.local_sweep()
    for s in shards:
        s.capture()
    rank_ms = []
    for s in shards:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            s.local_sweep()
        torch.cuda.synchronize()
        rank_ms.append((time.perf_counter() - t0) / 5 * 1e3)
    for s in shards:
        s.close()
    del shards
    out["sync"]["ms_per_sweep_8gpu_projected"] = max(rank_ms)

    # async: 8 virtual ranks on peer halo rings, bounded random schedule
    lay = SlabLayout.build(cfg.dims.nz, cfg.kdims[2], cfg.block_height, 8)
    xs, z0s = [], []
    for r in range(8):
        lo, hi = lay.local(r)
        xs.append(torch.from_numpy(np.ascontiguousarray(x0[lo:hi + 1])).cuda().float())
        z0s.append(lo)
    hub, rings = RingHub.local(RingPlan(lay, ring_slots(2)), xs, z0s)
    step = cuda_block_step(obj, dtype)
    ranks = [AsyncShard(lay, r, xs[r], torch.zeros_like(xs[r]), rings[r], step, 2) for r in range(8)]
    rng = np.random.default_rng(0)
    fs, its = [], []
    torch.cuda.synchronize()
    t_upd = 0.0
    for sweep in range(sweeps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(B):  # one sweep's worth of updates, enqueued without host syncs
            lo_t = min(s.t for s in ranks)
            ready = [s for s in ranks if s.t - lo_t < 2]
            rng.choice(ready).update()
        torch.cuda.synchronize()
        t_upd += time.perf_counter() - t0
        full = torch.cat([s.x[s.o_lo - s.l_lo:s.o_hi - s.l_lo + 1] for s in ranks])
        fs.append(f_of(obj, full))
        its.append((sweep + 1) * B)
    st = [v for s in ranks for v in s.staleness]
    hub.close()
    out["async"] = {"block_iterations": its, "f": fs, "ms_per_update_1gpu": t_upd / (sweeps * B) * 1e3,
                    "staleness_max": int(max(st)), "staleness_mean": float(np.mean(st)),
                    "ms_per_32_updates_8gpu_projected": t_upd / (sweeps * B) * 1e3 * B / 8}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
