"""Device plumbing: torch owns device memory and streams; the C ABI computes.

Public functions accept numpy arrays (host, float64 -- the reference
contract) or torch tensors.  numpy in -> numpy out (copied through the
device); CUDA tensors stay on the device and keep their dtype (float64 or
float32).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _native as N

DTYPES = {torch.float64: N.BD3MG_F64, torch.float32: N.BD3MG_F32}


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("bd3mg_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def is_tensor(a) -> bool:
    return isinstance(a, torch.Tensor)


def to_device(a, dtype: torch.dtype = torch.float64, device=None) -> torch.Tensor:
    """Contiguous CUDA tensor of ``dtype`` (copies only when needed)."""
    if is_tensor(a):
        t = a
        if not t.is_cuda:
            t = t.to(device or default_device())
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return torch.from_numpy(arr).to(device or default_device(), non_blocking=False).to(dtype)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


_bound = threading.local()


def bind(device: int) -> None:
    """Point the library's own CUDA runtime at `device` for this thread
    (it links cudart statically, so torch.cuda.set_device alone is not its
    state)."""
    if getattr(_bound, "dev", None) != device:
        N.check(N.lib.bd3mg_set_device(device))
        _bound.dev = device


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream or torch.cuda.current_stream()
    bind(s.device.index if s.device.index is not None else torch.cuda.current_device())
    return s.cuda_stream


_ws_lock = threading.Lock()
_ws: dict[tuple[int, int], torch.Tensor] = {}


def workspace(nbytes: int, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Grow-only scratch buffer, one per (device, stream) so stream-ordered
    reuse is race-free."""
    s = stream or torch.cuda.current_stream()
    key = (s.device.index if s.device.index is not None else torch.cuda.current_device(), s.cuda_stream)
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=s.device)
            _ws[key] = buf
        return buf


def geom(dims, kdims, dtype: torch.dtype) -> N.Geom:
    nx, ny, nz = dims
    kx, ky, kz = kdims
    return N.Geom(nx, ny, nz, kx, ky, kz, DTYPES[dtype])


def reg(p) -> N.Reg:
    return N.Reg(p.lam, p.eta, p.kappa, p.delta, p.x_min, p.x_max)


def byref(s):
    return C.byref(s)
