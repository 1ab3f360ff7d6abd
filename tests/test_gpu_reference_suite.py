"""The reference's own test suite (pkg/tests: test_blur, test_objective,
test_directions, test_scheduler, test_volume) run on the B200 through the
INTEGRATION.md ctypes binding (scripts/run_reference_suite.py).  Needs the
reference install in baseline/_ref (git-ignored; it travels to the GPU box
with the snapshot); skipped when absent."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "ref_tests").exists(), reason="baseline/_ref absent")
def test_reference_suite_passes_on_cuda_core():
    res = subprocess.run([sys.executable, str(ROOT / "scripts" / "run_reference_suite.py")], capture_output=True,
                         text=True, timeout=1800, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    assert "active core: bd3mg._b200" in res.stdout
