"""Multi-GPU paths on DISTINCT devices (skipped on a one-GPU box): rank r on
device r over NCCL, launched by torchrun.  The sharded block-Jacobi sweep --
cross-device cudaIpc inboxes with peer access and the update kernel's
NVLink mirror stores, and the NCCL-message transport -- must equal the
single-GPU sweep bit for bit; the asynchronous engine must respect its
delay bound and descend (reference semantics: runtime.py:244-292)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("world", [2])
def test_sharded_and_async_on_distinct_devices(world, tmp_path, oracle_mod):
    from paper_2002_02328_b200 import configs, objective, runtime
    out = tmp_path / "md.npz"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", str(ROOT / "tests" / "_multidevice_worker.py"),
           str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert f"nranks {world}" in (res.stdout + res.stderr)  # the NCCL communicator spans the ranks
    got = np.load(out)
    cfg = configs.CONFIGS["C1"]
    psf, truth, y, x0, params = configs.make_problem(cfg, y_from=lambda p, t: oracle_mod.H(p.kernels, t))
    obj = objective.Objective(psf, y, params)
    eng = runtime.JacobiSweeper(obj, x0, 4, torch.float64)
    for _ in range(6):
        eng.sweep()
    single = eng.x.cpu().numpy()
    assert np.array_equal(got["p2p"], single)
    assert np.array_equal(got["nccl"], single)
    assert int(got["async_stale_max"]) <= 2
    f0 = objective.eval_f(obj, x0)
    assert objective.eval_f(obj, got["async"]) < f0
