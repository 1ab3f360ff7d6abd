"""BD3MGVOL payloads straight between files and device memory through the
C ABI (bd3mg_payload_read_device / _write_device / bd3mg_field_nonfinite):
bitwise against the reference-written files and the host path, across the
16 MiB chunk boundary, with the reference's error behaviour."""

import struct
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2002_02328_b200.volume import FormatError, read_volume, write_volume

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "io"
CHUNK = (16 << 20) // 8  # elements per pinned chunk


def test_device_read_matches_reference_files():
    arrays = np.load(GOLD / "io.npz")
    for name, key in (("vol_5x4x3.bd3mgvol", "vol"), ("vol_2x2x2.bd3mgvol", "idx")):
        t = read_volume(GOLD / name, device="cuda")
        assert t.is_cuda and t.dtype == torch.float64
        assert np.array_equal(t.cpu().numpy(), arrays[key])
        t32 = read_volume(GOLD / name, device="cuda", dtype=torch.float32)
        assert np.array_equal(t32.cpu().numpy(), arrays[key].astype(np.float32))


def test_device_write_reproduces_reference_bytes(tmp_path):
    arrays = np.load(GOLD / "io.npz")
    write_volume(torch.from_numpy(arrays["vol"]).cuda(), tmp_path / "v")
    assert (tmp_path / "v").read_bytes() == (GOLD / "vol_5x4x3.bd3mgvol").read_bytes()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_multi_chunk_round_trip(dtype, tmp_path):
    nz, ny, nx = 6, 417, 2011  # 5.03 M voxels: two full chunks + a ragged tail
    assert nz * ny * nx > 2 * CHUNK and (nz * ny * nx) % CHUNK
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand((nz, ny, nx), dtype=dtype, device="cuda", generator=g) * 4 - 1
    write_volume(x, tmp_path / "x")
    assert (tmp_path / "x").stat().st_size == 24 + 8 * x.numel()
    host = read_volume(tmp_path / "x")                      # reference-format host reader
    assert np.array_equal(host, x.double().cpu().numpy())
    back = read_volume(tmp_path / "x", device="cuda", dtype=dtype)
    assert torch.equal(back, x)


def test_device_read_errors(tmp_path):
    n = 2 * CHUNK + 17
    vals = np.zeros(n)
    vals[CHUNK + 5] = np.nan  # in the second chunk
    p = tmp_path / "nan"
    p.write_bytes(b"BD3MGVOL" + struct.pack("<I", 1) + struct.pack("<III", n, 1, 1) + vals.tobytes())
    for dt in (torch.float64, torch.float32):
        with pytest.raises(FormatError, match="non-finite payload"):
            read_volume(p, device="cuda", dtype=dt)
    raw = p.read_bytes()
    (tmp_path / "short").write_bytes(raw[:-8])
    with pytest.raises(FormatError, match=f"truncated payload: expected {8 * n} bytes, got {8 * n - 8}"):
        read_volume(tmp_path / "short", device="cuda")
    (tmp_path / "long").write_bytes(raw + b"\0")
    with pytest.raises(FormatError, match="trailing data"):
        read_volume(tmp_path / "long", device="cuda")
    with pytest.raises(OSError):
        read_volume(tmp_path / "missing", device="cuda")


def test_device_write_rejects_non_finite(tmp_path):
    x = torch.zeros((3, 4, 5), dtype=torch.float32, device="cuda")
    x[2, 3, 4] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        write_volume(x, tmp_path / "bad")
    assert not (tmp_path / "bad").exists()
