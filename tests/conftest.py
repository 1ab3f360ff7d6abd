import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    """Dict of cases from tests/golden/<name>.npz ('case/key' -> array)."""
    raw = np.load(GOLDEN / f"{name}.npz")
    out = {}
    for k in raw.files:
        if "/" in k:
            c, kk = k.split("/", 1)
            out.setdefault(c, {})[kk] = raw[k]
        else:
            out[k] = raw[k]
    return out


@pytest.fixture(scope="session")
def oracle_mod():
    """The CPU oracle (test infrastructure), built on demand."""
    import subprocess
    lib = ROOT / "oracle" / "liboracle_bd3mg.so"
    if not lib.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True, capture_output=True)
    from oracle import oracle
    oracle.core("c", threads=8)
    return oracle


@pytest.fixture
def rng():
    return np.random.default_rng(42)
