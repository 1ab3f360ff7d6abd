"""The C-ABI library loads without a GPU and exports every entry point the
header declares (no compute calls here)."""

import ctypes
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "bd3mg_b200.h"
LIB = ROOT / "paper_2002_02328_b200" / "_lib" / "libbd3mg_b200.so"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bd3mg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert "bd3mg_depthvar_correlate_f64" in names
    assert "bd3mg_depthvar_correlate_adjoint_f64" in names
    assert "bd3mg_mg_steps" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(str(LIB))
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (bd3mg_\w+)", out))
    assert set(declared()) <= exported


def test_binding_covers_header():
    from paper_2002_02328_b200 import _native
    assert set(_native.EXPORTS) == set(declared())
    assert _native.lib.bd3mg_version().startswith(b"bd3mg_b200")


def test_error_path_without_gpu():
    """Argument validation runs before any CUDA call and maps to ValueError."""
    import pytest

    from paper_2002_02328_b200 import _native as N
    rc = N.lib.bd3mg_depthvar_correlate_f64(None, 4, 4, 4, None, 4, 2, 3, 3, 0, 0, 3, None, None)
    assert rc == N.BD3MG_EINVAL
    with pytest.raises(ValueError, match="odd"):
        N.check(rc)
    g = N.Geom(4, 4, 4, 3, 3, 3, N.BD3MG_F64)
    assert N.lib.bd3mg_grad_rows_ws_bytes(ctypes.byref(g), 0, 3) > 0
    assert N.lib.bd3mg_grad_rows_ws_bytes(ctypes.byref(g), 2, 9) == ctypes.c_size_t(-1).value


def test_sm100a_code_present():
    """The library carries sm_100a SASS with TMA and FP64 FMA in the
    correlation kernels (evidence of the Blackwell path)."""
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UTMALDG" in out and "DFMA" in out
