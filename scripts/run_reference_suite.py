#!/usr/bin/env python
"""Run the reference's OWN test suite on the B200 through the INTEGRATION.md
binding.

* takes the unmodified reference installed in baseline/_ref (``pip install
  --target``) and its tests (baseline/_ref/ref_tests,
  copied from pkg/tests; both git-ignored, both travel to the GPU box);
* builds a scratch copy of the package with exactly the maintainer's change
  of INTEGRATION.md section 1: ``integration/_b200.py`` dropped in as
  ``bd3mg/_b200.py`` and the ``BD3MG_B200`` switch added to ``bd3mg/kernels.py``;
* runs pytest on the reference tests with ``BD3MG_B200=1``; a probe plugin
  asserts the binding is the active core and records how many kernels the
  library launched (proof the suite ran on the GPU).

    python scripts/run_reference_suite.py [--log FILE] [pytest args...]

Exit status is pytest's (0 = every reference test passed on the CUDA core).
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
LIB = ROOT / "paper_2002_02328_b200" / "_lib" / "libbd3mg_b200.so"

SWITCH_ANCHOR = "if not _force_fallback:\n"
SWITCH = ('if os.environ.get("BD3MG_B200", "") not in ("", "0"):\n'
          "    from . import _b200 as _impl  # libbd3mg_b200.so (INTEGRATION.md section 1)\n"
          "    USING_COMPILED = True\n"
          "elif not _force_fallback:\n")

PROBE = '''
import ctypes, os, sys

def pytest_sessionfinish(session, exitstatus):
    k = sys.modules.get("bd3mg.kernels")
    impl = getattr(k, "_impl", None)
    name = getattr(impl, "__name__", None)
    lib = ctypes.CDLL(os.environ["BD3MG_B200_LIB"])
    lib.bd3mg_launch_count.restype = ctypes.c_longlong
    n = lib.bd3mg_launch_count()
    print(f"\\n[b200-probe] active core: {name}; backend_name(): {k.backend_name() if k else None}; "
          f"libbd3mg_b200 kernel launches in this process: {n}")
    if name != "bd3mg._b200" or n == 0:
        print("[b200-probe] FAIL: the reference suite did not run on the B200 core")
        session.exitstatus = 3
'''


def stage(dst: Path) -> Path:
    pkg = dst / "bd3mg"
    shutil.copytree(REF / "bd3mg", pkg, ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(ROOT / "integration" / "_b200.py", pkg / "_b200.py")
    kp = pkg / "kernels.py"
    src = kp.read_text()
    if SWITCH_ANCHOR not in src:
        raise SystemExit("reference kernels.py changed: switch anchor not found")
    kp.write_text(src.replace(SWITCH_ANCHOR, SWITCH, 1))
    tests = dst / "tests"
    shutil.copytree(REF / "ref_tests", tests, ignore=shutil.ignore_patterns("__pycache__"))
    (dst / "b200_probe.py").write_text(PROBE)
    return tests


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--log", default=None)
    args, rest = ap.parse_known_args()
    if not (REF / "bd3mg").exists() or not (REF / "ref_tests").exists():
        print("baseline/_ref (reference install + ref_tests) is absent", file=sys.stderr)
        return 4
    if not LIB.exists():
        print(f"{LIB} is not built", file=sys.stderr)
        return 4
    with tempfile.TemporaryDirectory(prefix="bd3mg_b200_suite_") as tmp:
        tmp = Path(tmp)
        tests = stage(tmp)
        env = dict(os.environ, BD3MG_B200="1", BD3MG_B200_LIB=str(LIB),
                   PYTHONPATH=os.pathsep.join([str(tmp), str(tests)]))
        env.pop("BD3MG_NO_EXT", None)
        cmd = [sys.executable, "-m", "pytest", str(tests), "-p", "b200_probe", "-q", "-rfE",
               "-o", "cache_dir=" + str(tmp / ".pytest_cache"), *rest]
        res = subprocess.run(cmd, cwd=tmp, env=env, capture_output=True, text=True)
        out = res.stdout + res.stderr
        print(out)
        if args.log:
            Path(args.log).parent.mkdir(parents=True, exist_ok=True)
            Path(args.log).write_text("$ BD3MG_B200=1 " + " ".join(cmd[1:]) + "\n" + out)
        return res.returncode


if __name__ == "__main__":
    sys.exit(main())
