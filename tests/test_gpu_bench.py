"""bench.py's N>1 path end to end on the one GPU of the test box: two
torchrun ranks on device 0 (BD3MG_BENCH_ONE_GPU=1: gloo for the host-side
collectives, cudaIpc-mapped halo inboxes / rings on the same device).  The
ranks' kernels never wait on one another; every cross-rank ordering is a
host synchronisation.  Checks that rank 0 prints one well-formed JSON line
with the p2p halo path active."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("extra", [[], ["--mode", "async", "--quick"]])
def test_bench_two_ranks_one_gpu(extra):
    env = dict(os.environ, BD3MG_BENCH_ONE_GPU="1", OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", *extra]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["halo"].startswith("p2p"), d["halo"]
    if not extra:
        assert d["e2e"]["value"] > 0 and d["scaling"] == "weak"
        assert "roofline" in d and d["gpu_launches"] > 0
    else:
        assert d["async"]["staleness_max"] <= d["async"]["max_delay_bound"]
