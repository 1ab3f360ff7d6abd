"""Volume and block types plus the seeded input generators.

Mirrors the type layer of the reference (`pkg/src/bd3mg/volume.py:35-94`):
a volume is a C-contiguous array of shape ``(nz, ny, nx)`` with x fastest,
blocks are inclusive z-slice ranges.  The stochastic helpers draw from numpy's
Philox counter-based generator so the oracle and the CUDA path consume
bitwise-identical arrays (`volume.py:176-178`, `:222-239`).

The ellipsoid phantom is not in the reference (its phantom is
blobs/spheres/boxes); it is the BASELINE.json generator for configs C1-C5.
"""

from __future__ import annotations

import math
import os
import struct
from contextlib import contextmanager
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np


VOLUME_MAGIC = b"BD3MGVOL"
FORMAT_VERSION = 1
HEADER_BYTES = 8 + 4 + 12


class FormatError(ValueError):
    """A binary container violated the volume/PSF format (reference `volume.py:31-32`)."""


class Dims3(NamedTuple):
    """Voxel counts per axis (reference `volume.py:35-54`)."""

    nx: int
    ny: int
    nz: int

    @property
    def shape(self) -> tuple[int, int, int]:
        return (self.nz, self.ny, self.nx)

    @property
    def count(self) -> int:
        return self.nx * self.ny * self.nz

    def validate(self) -> "Dims3":
        if min(self) < 1:
            raise ValueError(f"dimensions must be >= 1, got {self}")
        return self


@dataclass(frozen=True)
class SliceBlock:
    """Inclusive depth range [z_lo, z_hi] (reference `volume.py:57-79`)."""

    z_lo: int
    z_hi: int

    def __post_init__(self):
        if not (0 <= self.z_lo <= self.z_hi):
            raise ValueError(f"invalid slice range [{self.z_lo}, {self.z_hi}]")

    @property
    def height(self) -> int:
        return self.z_hi - self.z_lo + 1

    def count(self, dims: Dims3) -> int:
        return dims.nx * dims.ny * self.height

    def check_within(self, dims: Dims3) -> "SliceBlock":
        if self.z_hi >= dims.nz:
            raise ValueError(f"block {self} exceeds nz={dims.nz}")
        return self


def dims_of(vol) -> Dims3:
    nz, ny, nx = tuple(vol.shape)
    return Dims3(int(nx), int(ny), int(nz))


def check_volume(vol) -> np.ndarray:
    """float64, C-order, 3-D, finite (reference `volume.py:87-94`)."""
    arr = np.ascontiguousarray(vol, dtype=np.float64)
    if arr.ndim != 3:
        raise ValueError(f"volume must be 3-dimensional, got shape {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValueError("volume contains non-finite entries")
    return arr


@contextmanager
def _as_stream(source, mode):
    if hasattr(source, "read") or hasattr(source, "write"):
        yield source
    else:
        with open(source, mode) as fh:
            yield fh


def _read_exact(fh, n: int, what: str) -> bytes:
    buf = fh.read(n)
    if len(buf) != n:
        raise FormatError(f"truncated {what}: expected {n} bytes, got {len(buf)}")
    return buf


def _read_header(fh, magic_want: bytes, version_want: int) -> tuple[int, int, int]:
    magic = _read_exact(fh, 8, "header")
    if magic != magic_want:
        raise FormatError(f"bad magic {magic!r}")
    (version,) = struct.unpack("<I", _read_exact(fh, 4, "header"))
    if version != version_want:
        raise FormatError(f"unsupported version {version}")
    nx, ny, nz = struct.unpack("<III", _read_exact(fh, 12, "header"))
    if min(nx, ny, nz) < 1:
        raise FormatError(f"invalid dimensions ({nx}, {ny}, {nz})")
    return nx, ny, nz


def _payload_extent(path, offset: int, nbytes: int) -> None:
    """Truncation / trailing-data checks of a file payload from its size
    (the order and wording of reference `volume.py:138-141`)."""
    have = os.stat(path).st_size - offset
    if have < nbytes:
        raise FormatError(f"truncated payload: expected {nbytes} bytes, got {max(have, 0)}")
    if have > nbytes:
        raise FormatError("payload length mismatch: trailing data")


def _is_device_tensor(vol) -> bool:
    return type(vol).__module__.startswith("torch") and getattr(vol, "is_cuda", False)


def write_volume(vol, sink) -> None:
    """BD3MGVOL container: 8-byte magic, u32 version, u32 nx/ny/nz, float64
    payload, little-endian (reference `volume.py:104-114`).

    A CUDA tensor (float64 or float32) written to a path streams straight
    from device memory through the native payload writer; the finiteness check
    runs on the device first, so a rejected volume creates no file."""
    if _is_device_tensor(vol) and not (hasattr(sink, "read") or hasattr(sink, "write")):
        from . import _native as N
        import ctypes

        if vol.dim() != 3:
            raise ValueError(f"volume must be 3-dimensional, got shape {tuple(vol.shape)}")
        import torch

        t = vol.contiguous()
        if t.dtype not in (torch.float64, torch.float32):
            t = t.double()
        dt = N.BD3MG_F64 if t.dtype == torch.float64 else N.BD3MG_F32
        stream = torch.cuda.current_stream(t.device).cuda_stream
        bad = ctypes.c_int32(0)
        with torch.cuda.device(t.device):
            N.check(N.lib.bd3mg_field_nonfinite(t.data_ptr(), t.numel(), dt, ctypes.byref(bad), stream))
            if bad.value:
                raise ValueError("volume contains non-finite entries")
            nz, ny, nx = t.shape
            with open(sink, "wb") as fh:
                fh.write(VOLUME_MAGIC)
                fh.write(struct.pack("<I", FORMAT_VERSION))
                fh.write(struct.pack("<III", nx, ny, nz))
            N.check(N.lib.bd3mg_payload_write_device(os.fsencode(sink), t.data_ptr(), t.numel(), dt, stream))
        return
    arr = check_volume(vol)
    d = dims_of(arr)
    with _as_stream(sink, "wb") as fh:
        fh.write(VOLUME_MAGIC)
        fh.write(struct.pack("<I", FORMAT_VERSION))
        fh.write(struct.pack("<III", d.nx, d.ny, d.nz))
        fh.write(arr.astype("<f8", copy=False).tobytes())


def read_volume(source, device=None, dtype=None):
    """Inverse of :func:`write_volume` with the reference's distinct errors
    for bad magic, version mismatch, truncation, trailing data and a
    non-finite payload (reference `volume.py:124-145`).

    ``device=None``: a float64 numpy array, as the reference returns.
    ``device="cuda"`` (or a torch device) with a path: the payload streams
    file -> pinned chunks -> device through ``bd3mg_payload_read_device`` into
    a CUDA tensor of ``dtype`` (torch.float64 default, or torch.float32,
    narrowed on the device after the float64 finiteness check)."""
    if device is None:
        with _as_stream(source, "rb") as fh:
            nx, ny, nz = _read_header(fh, VOLUME_MAGIC, FORMAT_VERSION)
            n = nx * ny * nz
            payload = _read_exact(fh, 8 * n, "payload")
            if fh.read(1):
                raise FormatError("payload length mismatch: trailing data")
        data = np.frombuffer(payload, dtype="<f8").astype(np.float64)
        if not np.isfinite(data).all():
            raise FormatError("non-finite payload")
        return np.ascontiguousarray(data.reshape(nz, ny, nx))
    import torch

    dtype = torch.float64 if dtype is None else dtype
    if dtype not in (torch.float64, torch.float32):
        raise ValueError(f"device volumes are float64 or float32, got {dtype}")
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    if hasattr(source, "read"):  # a stream: parse on the host, then upload
        return torch.from_numpy(read_volume(source)).to(dev).to(dtype)
    from . import _native as N

    with open(source, "rb") as fh:
        nx, ny, nz = _read_header(fh, VOLUME_MAGIC, FORMAT_VERSION)
    n = nx * ny * nz
    _payload_extent(source, HEADER_BYTES, 8 * n)
    out = torch.empty((nz, ny, nx), dtype=dtype, device=dev)
    dt = N.BD3MG_F64 if dtype == torch.float64 else N.BD3MG_F32
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        N.check(N.lib.bd3mg_payload_read_device(os.fsencode(source), HEADER_BYTES, n, out.data_ptr(), dt, stream))
    return out


def philox(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def add_gaussian_noise(vol, sigma: float, seed: int) -> np.ndarray:
    """vol + sigma * N(0,1) i.i.d. (reference `volume.py:222-229`)."""
    base = np.asarray(vol, dtype=np.float64)
    if sigma < 0:
        raise ValueError("sigma must be nonnegative")
    if sigma == 0:
        return base.copy()
    return base + sigma * philox(seed).standard_normal(base.shape)


def init_uniform(dims: Dims3, upper: float, seed: int) -> np.ndarray:
    """U[0, upper] i.i.d. (reference `volume.py:232-239`)."""
    dims = Dims3(*dims).validate()
    if upper < 0:
        raise ValueError("upper must be nonnegative")
    if upper == 0:
        return np.zeros(dims.shape)
    return philox(seed).uniform(0.0, upper, dims.shape)


def snr_db(reference, estimate) -> float:
    """20 log10(||ref|| / ||est - ref||) (reference `volume.py:148-161`)."""
    ref = np.asarray(reference, dtype=np.float64)
    est = np.asarray(estimate, dtype=np.float64)
    if ref.shape != est.shape:
        raise ValueError(f"shape mismatch {ref.shape} vs {est.shape}")
    rn = float(np.linalg.norm(ref))
    if rn == 0.0:
        raise ValueError("reference volume has zero norm")
    en = float(np.linalg.norm(est - ref))
    return math.inf if en == 0.0 else 20.0 * math.log10(rn / en)


def rel_dist(x, x_star) -> float:
    """||x - x*|| / ||x*|| (reference `volume.py:164-173`)."""
    a = np.asarray(x, dtype=np.float64)
    b = np.asarray(x_star, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch {a.shape} vs {b.shape}")
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        raise ValueError("x_star has zero norm")
    return float(np.linalg.norm(a - b)) / bn


def ellipsoid_phantom(dims: Dims3, n: int, seed: int, amplitude: str = "uniform",
                      axis_frac=(0.05, 0.2)) -> np.ndarray:
    """Sum of ``n`` axis-aligned solid ellipsoids (BASELINE configs C1-C5).

    Centres ~ U over the volume, semi-axes ~ U[axis_frac]*extent + 1 voxel,
    amplitudes ~ U[0,1] (``amplitude="uniform"``) or Gamma(2, 0.25)
    (``"gamma"``, the Poisson-like spread of C3/C4).  Built plane by plane so
    the 1024x1024x512 config does not need a full-volume meshgrid.
    """
    dims = Dims3(*dims).validate()
    rng = philox(seed)
    nz, ny, nx = dims.shape
    extent = np.array([nz, ny, nx], dtype=np.float64)
    centres = rng.uniform(0.0, 1.0, (n, 3)) * (extent - 1)
    axes = rng.uniform(axis_frac[0], axis_frac[1], (n, 3)) * extent + 1.0
    if amplitude == "uniform":
        amps = rng.uniform(0.0, 1.0, n)
    elif amplitude == "gamma":
        amps = rng.gamma(2.0, 0.25, n)
    else:
        raise ValueError(f"unknown amplitude law {amplitude!r}")
    vol = np.zeros(dims.shape)
    for (cz, cy, cx), (az, ay, ax), amp in zip(centres, axes, amps):
        z0 = max(0, int(math.floor(cz - az)))
        z1 = min(nz - 1, int(math.ceil(cz + az)))
        # bounding box in y, x (mask evaluated only there)
        y0, y1 = max(0, int(math.floor(cy - ay))), min(ny - 1, int(math.ceil(cy + ay)))
        x0, x1 = max(0, int(math.floor(cx - ax))), min(nx - 1, int(math.ceil(cx + ax)))
        yy = np.arange(y0, y1 + 1, dtype=np.float64)[:, None]
        xx = np.arange(x0, x1 + 1, dtype=np.float64)[None, :]
        q = ((yy - cy) / ay) ** 2 + ((xx - cx) / ax) ** 2
        for z in range(z0, z1 + 1):
            tz = ((z - cz) / az) ** 2
            if tz > 1.0:
                continue
            vol[z, y0:y1 + 1, x0:x1 + 1][q <= 1.0 - tz] += amp
    return vol
