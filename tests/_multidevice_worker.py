"""Worker of tests/test_gpu_multidevice.py, launched by torchrun with one
rank per GPU (rank r on device r, NCCL): the sharded block-Jacobi sweep
(update-kernel NVLink mirror stores into cudaIpc-mapped peer inboxes, and
the NCCL-message transport) and the asynchronous engine (peer halo rings)
on distinct devices.  Rank 0 writes the results to the path in argv[1]."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2002_02328_b200 import configs, objective  # noqa: E402
from paper_2002_02328_b200.distributed import AsyncEngine, ShardedJacobi  # noqa: E402


def main():
    out = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg, y_from=lambda p, t: __import__("oracle.oracle",
                                                                                          fromlist=["H"]).H(p.kernels, t))
    obj = objective.Objective(psf, y, params)
    res = {}
    for halo in ("p2p", "nccl"):
        eng = ShardedJacobi(obj, x0, 4, torch.float64, halo=halo)
        eng.sweep()
        eng.capture()
        for _ in range(5):
            eng.sweep()
        torch.cuda.synchronize()
        owned = eng.x[eng.o_lo - eng.l_lo:eng.o_hi - eng.l_lo + 1].cpu()
        parts = [None] * world
        dist.all_gather_object(parts, (eng.o_lo, owned.numpy()))
        res[halo] = np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0])])
        res[halo + "_f"] = float(eng.terms[4].item())
        eng.close()
    a = AsyncEngine(obj, x0, 4, torch.float64, max_delay=2, halo="p2p")
    for _ in range(6):
        a.sweep()
    a.finish()
    torch.cuda.synchronize()
    st = a.shard.staleness
    parts = [None] * world
    dist.all_gather_object(parts, (a.layout.owned(rank)[0], a.x[a.layout.owned(rank)[0] - a.layout.local(rank)[0]:
                                                              a.layout.owned(rank)[1] - a.layout.local(rank)[0] + 1]
                                   .cpu().numpy(), max(st) if st else 0))
    res["async"] = np.concatenate([p for _, p, _ in sorted(parts, key=lambda t: t[0])])
    res["async_stale_max"] = max(s for _, _, s in parts)
    if rank == 0:
        np.savez(out, **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
