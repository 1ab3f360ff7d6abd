"""bench.py --impl reference (the reference arm the driver runs) on the CPU:
one JSON line with the contract's keys, the faster reference backend named."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env,
                         cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "block-it/s"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert "backend" in cb["sample"]


def test_reference_arm_is_import_clean():
    """The reference arm never maps the product library or torch (VERDICT r1:
    its native_so_loaded listed libbd3mg_b200.so through an import
    side-effect): run it in-process and inspect sys.modules."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--config','C1','--steps','1',"
            "'--warmup','1']; runpy.run_path('bench.py', run_name='__main__'); "
            "bad=[m for m in sys.modules if m=='torch' or m.startswith('paper_2002_02328_b200._native') "
            "or m in ('paper_2002_02328_b200.blur','paper_2002_02328_b200.objective')]; "
            "assert not bad, bad; print('CLEAN')")
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "CLEAN" in res.stdout
