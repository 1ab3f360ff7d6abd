"""Projected multi-GPU scaling from MEASURED per-rank sweep times on one B200.

This run has one GPU, so the N>1 sweeps cannot be timed end to end.  What
can be measured is the device work every rank does per synchronous sweep:
each virtual rank of the sharded layout (distributed.ShardedJacobi with the
p2p halo path: inbox unpack + fused sweep with the mirror stores, captured
as the same CUDA graph a real rank replays) is timed alone on this GPU.  A
synchronous sweep at P GPUs takes max over ranks of that time plus the
recorder all-reduce (7 doubles), which is NOT included.

  strong: efficiency(P) = T(1) / (P * max_r T_r)   (the config split over P)
  weak:   efficiency(P) = T(1) / max_r T_r         (the config per GPU)

    python scripts/scaling_projection.py [C2 C3 C5 ...] > out.json
"""
import dataclasses
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2002_02328_b200 import configs, objective, runtime  # noqa: E402
from paper_2002_02328_b200.distributed import ShardedJacobi  # noqa: E402
from paper_2002_02328_b200.volume import Dims3  # noqa: E402

FLUSH = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timed(fn, steps=5, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(steps):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / steps


def ranks_ms(obj, x0, h, dtype, P, exposed=False):
    """Per-rank sweep time (p2p graph: inbox unpack + mirrored sweep).  With
    `exposed`, also the same rank's plain sweep (no unpack, no mirror stores):
    the difference is the halo exchange work left on the rank's stream (here
    the mirror stores hit local HBM instead of NVLink)."""
    shards = [ShardedJacobi(obj, x0, h, dtype, rank=r, world=P, halo="p2p") for r in range(P)]
    bases = {r: s.peer.ptr for r, s in enumerate(shards)}
    for s in shards:
        s.peer.connect(bases)
    for s in shards:  # one eager sweep each, then the per-parity graphs
        s.local_sweep()
    for s in shards:
        s.capture()
    out = [timed(s.local_sweep) for s in shards]
    plain = None
    if exposed:
        plain = []
        for s in shards:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                s.peer, peer = None, s.peer
                s._launch(0)
                s.peer = peer
            plain.append(timed(g.replay))
    for s in shards:
        s.close()
    del shards
    torch.cuda.empty_cache()
    return (out, plain) if exposed else out


def main():
    names = sys.argv[1:] or ["C2", "C3", "C5"]
    res = {"method": __doc__.strip().splitlines()[0], "excluded": "recorder all-reduce of 7 doubles per sweep",
           "exposed_halo": "p2p rank sweep minus the same sweep without inbox unpack and mirror stores",
           "configs": {}}
    for name in names:
        cfg = configs.CONFIGS[name]
        dtype = torch.float64 if cfg.dtype == "f64" else torch.float32
        psf, truth, y, x0, params = configs.make_problem(cfg)
        obj = objective.Objective(psf, y, params)
        one = runtime.JacobiSweeper(obj, x0, cfg.block_height, dtype)
        one.sweep()
        one.capture()
        t1 = timed(one.sweep)
        del one
        torch.cuda.empty_cache()
        B = -(-cfg.dims.nz // cfg.block_height)
        entry = {"T1_ms": t1, "blocks": B, "strong": {}, "weak": {}}
        for P in (2, 4, 8):
            if P > B:
                continue
            ms, plain = ranks_ms(obj, x0, cfg.block_height, dtype, P, exposed=True)
            entry["strong"][P] = {"rank_ms": ms, "max_ms": max(ms), "efficiency": t1 / (P * max(ms)),
                                  "plain_rank_ms": plain,
                                  "exposed_halo_us": [1e3 * (a - b) for a, b in zip(ms, plain)]}
        if name == "C2":  # bench.py's default N>1 mode: the config per GPU
            for P in (2, 4, 8):
                wc = dataclasses.replace(cfg, name=f"C2x{P}", dims=Dims3(cfg.dims.nx, cfg.dims.ny, cfg.dims.nz * P))
                wpsf, _, wy, wx0, wpar = configs.make_problem(wc)
                wobj = objective.Objective(wpsf, wy, wpar)
                ms = ranks_ms(wobj, wx0, cfg.block_height, dtype, P)
                entry["weak"][P] = {"rank_ms": ms, "max_ms": max(ms), "efficiency": t1 / max(ms)}
        res["configs"][name] = entry
        print(json.dumps({name: entry}), file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
