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


def test_sharded_fp32_workspace_sizing():
    """Regression: an fp32 rank whose residual rows split around its recorder
    rows into odd-length jobs (two-plane kernel) needs more partial rows than
    one job; the size query must see the same split as the call (it once
    measured with a null recorder pointer and came out 3 KB short)."""
    import ctypes as C

    from paper_2002_02328_b200 import _native as N
    from paper_2002_02328_b200.distributed import SlabLayout
    g = N.Geom(512, 512, 128, 7, 7, 15, N.BD3MG_F32)
    lay = SlabLayout.build(128, 15, 16, 8)
    bl = lay.owned_blocks(1)
    (o_lo, o_hi), (l_lo, l_hi) = lay.owned(1), lay.local(1)
    barr = (C.c_int64 * 2)(bl[0].z_lo, bl[0].z_hi)
    with_rec = N.Sweep(1 << 30, 1 << 31, l_lo, l_hi - l_lo + 1, barr, 1, o_lo, o_hi, 1 << 32, None)
    no_rec = N.Sweep(1 << 30, 1 << 31, l_lo, l_hi - l_lo + 1, barr, 1, 0, -1, None, None)
    a = N.lib.bd3mg_jacobi_sweep_ws_bytes(C.byref(g), C.byref(with_rec))
    b = N.lib.bd3mg_jacobi_sweep_ws_bytes(C.byref(g), C.byref(no_rec))
    assert a >= 82051328 and a > b


def test_peer_and_flag_entry_points_validate_without_a_gpu():
    """Argument checks of the multi-GPU entry points return EINVAL before any
    CUDA call (runnable on the CPU-only host)."""
    import ctypes as C

    from paper_2002_02328_b200 import _native as N
    flags = (N.Flag * (N.MAX_FLAGS + 1))()
    assert N.lib.bd3mg_publish(flags, N.MAX_FLAGS + 1, None) == N.BD3MG_EINVAL
    assert N.lib.bd3mg_publish(None, 1, None) == N.BD3MG_EINVAL
    assert N.lib.bd3mg_publish(flags, 0, None) == N.BD3MG_OK  # nothing to publish
    dev = C.c_void_p()
    assert N.lib.bd3mg_host_register(None, 4096, C.byref(dev)) == N.BD3MG_EINVAL
    handle = (C.c_ubyte * N.IPC_HANDLE_BYTES)()
    assert N.lib.bd3mg_peer_alloc(0, C.byref(dev), handle) == N.BD3MG_EINVAL
    assert N.lib.bd3mg_peer_open(None, C.byref(dev)) == N.BD3MG_EINVAL
    g = N.Geom(16, 16, 8, 3, 3, 3, N.BD3MG_F64)
    r = N.Reg(1e-2, 1e-1, 0.05, 1e-2, 0.0, 1.0)
    assert N.lib.bd3mg_mg_steps_incremental(C.byref(g), C.byref(r), None, None, None, 1, None, None, None, None,
                                            0, None) == N.BD3MG_EINVAL
    assert N.lib.bd3mg_eval_f_resid(C.byref(g), C.byref(r), None, None, None, None, None, 0, None) == N.BD3MG_EINVAL
    assert b"null" in N.lib.bd3mg_last_error()


def test_integration_stub_mirrors_cython_buffer_errors():
    """integration/_b200.py (the maintainer's binding)
    raises the reference core's buffer errors -- type, message, order -- for
    every malformed input the Cython typed memoryviews reject (compared
    with the reference core compiled in oracle/_ref when present; no GPU
    work: every case fails before the foreign call)."""
    import importlib.util
    import os

    import numpy as np
    import pytest

    lib = ROOT / "paper_2002_02328_b200" / "_lib" / "libbd3mg_b200.so"
    if not lib.exists():
        pytest.skip("library not built")
    os.environ["BD3MG_B200_LIB"] = str(lib)
    spec = importlib.util.spec_from_file_location("_b200_stub", ROOT / "integration" / "_b200.py")
    stub = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(stub)
    k = np.ones((4, 3, 3, 3)) / 27
    x = np.zeros((4, 5, 6))
    ro = x.copy()
    ro.flags.writeable = False
    ro_str = x[:, :, ::2]
    ro_str.flags.writeable = False
    cases = [(x.astype(np.float32), k), (x, k.astype(np.float32)), (x[:, :, ::2], k), (np.asfortranarray(x), k),
             (x[0], k), (x.tolist(), k), (x.astype(np.int64), k), (x, k[0]), (ro, k), (ro_str, k),
             (x[0].astype(np.float32), k), (x.astype(np.float16), k), (x.astype(">f8"), k),
             (x.astype(np.complex128), k), (x.astype(np.uint8), k), (x.astype(np.bool_), k), (b"abc", k),
             (x.astype(np.float32), k[0]), (x, k[:, :, :, ::2])]
    want = None
    if (ROOT / "oracle" / "_ref").exists():
        from oracle import oracle as O
        if O.ref_core_available():
            want = O._RefCore().mod
    for frag, ker in cases:
        for name in ("depthvar_correlate", "depthvar_correlate_adjoint"):
            with pytest.raises((ValueError, TypeError, BufferError)) as got:
                getattr(stub, name)(frag, ker, 0, 0, 3)
            if want is not None:
                with pytest.raises((ValueError, TypeError, BufferError)) as ref:
                    getattr(want, name)(frag, ker, 0, 0, 3)
                assert type(got.value) is type(ref.value) and str(got.value) == str(ref.value), (
                    str(got.value), str(ref.value))
    # negative extent: numpy's error, as the reference's np.zeros
    with pytest.raises(ValueError, match="negative dimensions"):
        stub.depthvar_correlate(x, k, 0, 3, 0)
    assert stub.depthvar_correlate(x, k, 0, 3, 2).shape == (0, 5, 6)
