"""ctypes binding of the C ABI in ``include/bd3mg_b200.h``.

The library is the only compute backend: if it is missing this module raises
at import time (there is no CPU fallback on the product path).  Build it with
``python -m paper_2002_02328_b200.build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("BD3MG_LIB") or Path(__file__).resolve().parent / "_lib" / "libbd3mg_b200.so")

BD3MG_OK, BD3MG_EINVAL, BD3MG_ECUDA, BD3MG_EWORKSPACE, BD3MG_ENONFINITE, BD3MG_EFORMAT, BD3MG_EIO = range(7)
BD3MG_F64, BD3MG_F32 = 0, 1
INFO_DOUBLES = 16
MAX_TASKS_IN_PLACE = 32  # bd3mg_mg_steps: in-place calls are one launch of <= 32 tasks
EVAL_DOUBLES = 7

# every symbol the header declares (checked by tests/test_capi_symbols.py)
EXPORTS = (
    "bd3mg_last_error", "bd3mg_version", "bd3mg_launch_count", "bd3mg_set_device", "bd3mg_get_device",
    "bd3mg_depthvar_correlate_f64", "bd3mg_depthvar_correlate_adjoint_f64",
    "bd3mg_depthvar_correlate_f32", "bd3mg_depthvar_correlate_adjoint_f32",
    "bd3mg_depthvar_correlate_host_f64", "bd3mg_depthvar_correlate_adjoint_host_f64",
    "bd3mg_grad_rows_ws_bytes", "bd3mg_grad_rows",
    "bd3mg_eval_f_ws_bytes", "bd3mg_eval_f", "bd3mg_eval_rows_ws_bytes", "bd3mg_eval_rows",
    "bd3mg_omega_rows", "bd3mg_majorant_apply_ws_bytes", "bd3mg_majorant_apply",
    "bd3mg_cg_solve_ws_bytes", "bd3mg_cg_solve", "bd3mg_power_hth_ws_bytes", "bd3mg_power_hth", "bd3mg_pk_trace",
    "bd3mg_pk_launches",
    "bd3mg_mg_steps_ws_bytes", "bd3mg_mg_steps", "bd3mg_apply_increment",
    "bd3mg_jacobi_sweep_ws_bytes", "bd3mg_jacobi_cache_elems", "bd3mg_jacobi_sweep",
    "bd3mg_jacobi_sweep_mirrored", "bd3mg_jacobi_sweep_incremental", "bd3mg_mg_steps_incremental_ws_bytes",
    "bd3mg_mg_steps_incremental", "bd3mg_eval_f_resid", "bd3mg_mg_steps_mirrored", "bd3mg_host_register", "bd3mg_host_unregister",
    "bd3mg_publish", "bd3mg_peer_alloc", "bd3mg_peer_open", "bd3mg_peer_close", "bd3mg_peer_free",
    "bd3mg_problem_create", "bd3mg_problem_destroy", "bd3mg_problem_mg_direction_host",
    "bd3mg_problem_jacobi_sweep_host",
    "bd3mg_fma_probe",
    "bd3mg_payload_read_device", "bd3mg_payload_write_device", "bd3mg_field_nonfinite",
    "bd3mg_sep_correlate_f64", "bd3mg_sep_correlate_f32",
)


class Geom(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("kx", C.c_int32), ("ky", C.c_int32), ("kz", C.c_int32), ("dtype", C.c_int32)]


class Reg(C.Structure):
    _fields_ = [("lam", C.c_double), ("eta", C.c_double), ("kappa", C.c_double),
                ("delta", C.c_double), ("x_min", C.c_double), ("x_max", C.c_double)]


class Task(C.Structure):
    _fields_ = [("frag", C.c_void_p), ("frag_z0", C.c_int64), ("nzf", C.c_int64),
                ("z_lo", C.c_int64), ("z_hi", C.c_int64), ("d_mem", C.c_void_p),
                ("inc_out", C.c_void_p), ("x_rows", C.c_void_p), ("dmem_rows", C.c_void_p)]


class Sweep(C.Structure):
    _fields_ = [("x", C.c_void_p), ("dmem", C.c_void_p), ("frag_z0", C.c_int64), ("nzf", C.c_int64),
                ("blocks", C.POINTER(C.c_int64)), ("nblocks", C.c_int), ("rec_lo", C.c_int64),
                ("rec_hi", C.c_int64), ("snap", C.c_void_p), ("hd_cache", C.c_void_p)]


class Mirror(C.Structure):
    _fields_ = [("z_lo", C.c_int64), ("z_hi", C.c_int64), ("dst", C.c_void_p)]


IPC_HANDLE_BYTES = 64
MAX_FLAGS = 16


class Flag(C.Structure):
    _fields_ = [("word", C.c_void_p), ("value", C.c_int64)]


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[bd3mg_b200 status {code}] {msg}")
        self.code = code


_i64, _vp, _dp, _sz = C.c_int64, C.c_void_p, C.POINTER(C.c_double), C.c_size_t


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"CUDA library {LIB_PATH} is not built; run `python -m paper_2002_02328_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    corr = [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _vp]
    for name in ("bd3mg_depthvar_correlate_f64", "bd3mg_depthvar_correlate_adjoint_f64",
                 "bd3mg_depthvar_correlate_f32", "bd3mg_depthvar_correlate_adjoint_f32"):
        getattr(lib, name).argtypes = corr + [_vp]
    for name in ("bd3mg_depthvar_correlate_host_f64", "bd3mg_depthvar_correlate_adjoint_host_f64"):
        getattr(lib, name).argtypes = corr
    G, R, T = C.POINTER(Geom), C.POINTER(Reg), C.POINTER(Task)
    lib.bd3mg_last_error.restype = C.c_char_p
    lib.bd3mg_version.restype = C.c_char_p
    lib.bd3mg_launch_count.restype = C.c_longlong
    lib.bd3mg_set_device.argtypes = [C.c_int]
    lib.bd3mg_get_device.argtypes = [C.POINTER(C.c_int)]
    lib.bd3mg_grad_rows_ws_bytes.argtypes = [G, _i64, _i64]
    lib.bd3mg_grad_rows_ws_bytes.restype = _sz
    lib.bd3mg_grad_rows.argtypes = [G, R, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_eval_f_ws_bytes.argtypes = [G]
    lib.bd3mg_eval_f_ws_bytes.restype = _sz
    lib.bd3mg_eval_f.argtypes = [G, R, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_eval_rows_ws_bytes.argtypes = [G, _i64, _i64]
    lib.bd3mg_eval_rows_ws_bytes.restype = _sz
    lib.bd3mg_eval_rows.argtypes = [G, R, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_omega_rows.argtypes = [G, R, _vp, _i64, _i64, _i64, _i64, _vp, _vp]
    lib.bd3mg_majorant_apply_ws_bytes.argtypes = [G, _i64, _i64]
    lib.bd3mg_majorant_apply_ws_bytes.restype = _sz
    lib.bd3mg_majorant_apply.argtypes = [G, R, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp]
    lib.bd3mg_cg_solve_ws_bytes.argtypes = [G, _i64, _i64]
    lib.bd3mg_cg_solve_ws_bytes.restype = _sz
    lib.bd3mg_cg_solve.argtypes = [G, R, _vp, _vp, _vp, _i64, _i64, C.c_double, C.c_int32, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_pk_trace.argtypes = [_vp, _i64, C.POINTER(C.c_int64)]
    lib.bd3mg_pk_launches.restype = C.c_longlong
    lib.bd3mg_power_hth_ws_bytes.argtypes = [G]
    lib.bd3mg_power_hth_ws_bytes.restype = _sz
    lib.bd3mg_power_hth.argtypes = [G, _vp, _vp, C.c_int32, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_mg_steps_ws_bytes.argtypes = [G, T, C.c_int]
    lib.bd3mg_mg_steps_ws_bytes.restype = _sz
    lib.bd3mg_mg_steps.argtypes = [G, R, _vp, _vp, T, C.c_int, _vp, _vp, _sz, _vp]
    S = C.POINTER(Sweep)
    lib.bd3mg_jacobi_sweep_ws_bytes.argtypes = [G, S]
    lib.bd3mg_jacobi_sweep_ws_bytes.restype = _sz
    lib.bd3mg_jacobi_cache_elems.argtypes = [G, S]
    lib.bd3mg_jacobi_cache_elems.restype = C.c_int64
    lib.bd3mg_jacobi_sweep.argtypes = [G, R, _vp, _vp, S, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_jacobi_sweep_mirrored.argtypes = [G, R, _vp, _vp, S, C.POINTER(Mirror), C.c_int, _vp, _vp, _vp, _sz,
                                                _vp]
    lib.bd3mg_jacobi_sweep_incremental.argtypes = [G, R, _vp, _vp, S, _vp, C.c_int, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_mg_steps_incremental_ws_bytes.argtypes = [G, T, C.c_int]
    lib.bd3mg_mg_steps_incremental_ws_bytes.restype = _sz
    lib.bd3mg_mg_steps_incremental.argtypes = [G, R, _vp, _vp, T, C.c_int, C.POINTER(C.c_void_p), _vp, _vp, _vp, _sz,
                                               _vp]
    lib.bd3mg_eval_f_resid.argtypes = [G, R, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
    lib.bd3mg_mg_steps_mirrored.argtypes = [G, R, _vp, _vp, T, C.c_int, C.POINTER(Mirror), C.c_int, _vp, _vp, _sz,
                                            _vp]
    lib.bd3mg_host_register.argtypes = [_vp, _sz, C.POINTER(C.c_void_p)]
    lib.bd3mg_host_unregister.argtypes = [_vp]
    lib.bd3mg_publish.argtypes = [C.POINTER(Flag), C.c_int, _vp]
    lib.bd3mg_peer_alloc.argtypes = [_sz, C.POINTER(C.c_void_p), _vp]
    lib.bd3mg_peer_open.argtypes = [_vp, C.POINTER(C.c_void_p)]
    lib.bd3mg_peer_close.argtypes = [_vp]
    lib.bd3mg_peer_free.argtypes = [_vp]
    lib.bd3mg_apply_increment.argtypes = [C.c_int32, _vp, _vp, _vp, _i64, _vp]
    lib.bd3mg_problem_create.argtypes = [G, R, _vp, _vp, C.c_int, C.POINTER(C.c_void_p)]
    lib.bd3mg_problem_destroy.argtypes = [_vp]
    lib.bd3mg_problem_mg_direction_host.argtypes = [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp]
    lib.bd3mg_problem_jacobi_sweep_host.argtypes = [_vp, _vp, _vp, _i64, _i64, C.POINTER(C.c_int64), C.c_int,
                                                    _vp, _vp]
    lib.bd3mg_fma_probe.argtypes = [C.c_int32, C.c_int32, C.c_int32, _vp, _dp, _vp]
    lib.bd3mg_payload_read_device.argtypes = [C.c_char_p, _i64, _i64, _vp, C.c_int32, _vp]
    lib.bd3mg_payload_write_device.argtypes = [C.c_char_p, _vp, _i64, C.c_int32, _vp]
    lib.bd3mg_field_nonfinite.argtypes = [_vp, _i64, C.c_int32, C.POINTER(C.c_int32), _vp]
    for name in ("bd3mg_sep_correlate_f64", "bd3mg_sep_correlate_f32"):
        getattr(lib, name).argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64,
                                       _i64, _vp, C.c_int32, _vp]
    return lib


lib = _load()


def check(rc: int) -> None:
    """Map a status to the reference's exception types."""
    if rc == BD3MG_OK:
        return
    msg = (lib.bd3mg_last_error() or b"").decode()
    if rc == BD3MG_EINVAL:
        raise ValueError(msg)
    if rc == BD3MG_ENONFINITE:
        raise ValueError(msg or "non-finite gradient")
    if rc == BD3MG_EFORMAT:
        from .volume import FormatError
        raise FormatError(msg)
    if rc == BD3MG_EIO:
        raise OSError(msg)
    raise NativeError(rc, msg)


def ws_bytes(n: int) -> int:
    if n == C.c_size_t(-1).value:
        check(BD3MG_EINVAL)
    return n
