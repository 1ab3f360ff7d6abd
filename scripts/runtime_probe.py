"""Throughput of the reference-API driver runtime.run at C2 (bd3mg one worker,
bp3mg 8 workers, live engine 4 workers):  python scripts/runtime_probe.py"""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_2002_02328_b200 import configs, objective, runtime
psf, truth, y, x0, params = configs.make_problem("C2")
obj = objective.Objective(psf, y, params)
for method, workers, engine in (("bd3mg", 1, "simulated"), ("bp3mg", 8, "simulated"), ("bd3mg", 4, "live")):
    cfg = runtime.RunConfig(method=method, workers=workers, block_height=8, tol=1e-30, max_updates=16, engine=engine)
    runtime.run(obj, x0, cfg)
    torch.cuda.synchronize()
    cfg = runtime.RunConfig(method=method, workers=workers, block_height=8, tol=1e-30, max_updates=160, engine=engine)
    t0 = time.perf_counter()
    res = runtime.run(obj, x0, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(method, workers, engine, f"{160/dt:.0f} block-it/s", len(res.log))
