"""BD3MGVOL / BD3MGPSF containers on the host path, pinned to files written by
the reference's own writers (tests/golden/io, made by make_golden.py), and the
error behaviour of reference tests/test_volume.py:15-81."""

import io
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2002_02328_b200 import blur
from paper_2002_02328_b200.volume import FORMAT_VERSION, VOLUME_MAGIC, FormatError, read_volume, write_volume

GOLD = Path(__file__).resolve().parent / "golden" / "io"


@pytest.fixture(scope="module")
def arrays():
    return np.load(GOLD / "io.npz")


def test_reference_files_read_bitwise(arrays):
    assert np.array_equal(read_volume(GOLD / "vol_5x4x3.bd3mgvol"), arrays["vol"])
    assert np.array_equal(read_volume(GOLD / "vol_2x2x2.bd3mgvol"), arrays["idx"])
    psf = blur.read_psf(GOLD / "psf_6x5x4_k3x3x5.bd3mgpsf")
    assert psf.dims == (6, 5, 4) and psf.kdims == (3, 3, 5)
    assert np.array_equal(psf.kernels, arrays["psf_kernels"])
    assert np.array_equal(psf.params, arrays["psf_params"])


def test_writers_reproduce_reference_bytes(arrays, tmp_path):
    write_volume(arrays["vol"], tmp_path / "v")
    assert (tmp_path / "v").read_bytes() == (GOLD / "vol_5x4x3.bd3mgvol").read_bytes()
    buf = io.BytesIO()
    write_volume(arrays["idx"], buf)
    assert buf.getvalue() == (GOLD / "vol_2x2x2.bd3mgvol").read_bytes()
    psf = blur.PsfStack((6, 5, 4), (3, 3, 5), arrays["psf_kernels"], arrays["psf_params"])
    blur.write_psf(psf, tmp_path / "p")
    assert (tmp_path / "p").read_bytes() == (GOLD / "psf_6x5x4_k3x3x5.bd3mgpsf").read_bytes()


def test_smallest_volume_layout():
    buf = io.BytesIO()
    write_volume(np.full((1, 1, 1), 0.5), buf)
    raw = buf.getvalue()
    assert len(raw) == 32  # reference test_volume.py:15-24 (SPEC's 29 is wrong)
    assert raw[:8] == VOLUME_MAGIC and struct.unpack("<I", raw[8:12])[0] == FORMAT_VERSION
    assert struct.unpack("<III", raw[12:24]) == (1, 1, 1) and struct.unpack("<d", raw[24:])[0] == 0.5


def _header(nx=2, ny=2, nz=2, magic=VOLUME_MAGIC, version=FORMAT_VERSION):
    return magic + struct.pack("<I", version) + struct.pack("<III", nx, ny, nz)


@pytest.mark.parametrize("raw, msg", [
    (b"BD3MGXXX" + bytes(16), "bad magic"),
    (_header(version=2), "unsupported version 2"),
    (_header() + bytes(8 * 7), "truncated payload: expected 64 bytes, got 56"),
    (_header() + bytes(8 * 8 + 1), "payload length mismatch: trailing data"),
    (_header(nx=0), "invalid dimensions (0, 2, 2)"),
    (b"BD3MG", "truncated header: expected 8 bytes, got 5"),
    (_header(1, 1, 1) + struct.pack("<d", float("nan")), "non-finite payload"),
])
def test_read_errors(raw, msg, tmp_path):
    with pytest.raises(FormatError, match=msg.replace("(", r"\(").replace(")", r"\)")):
        read_volume(io.BytesIO(raw))
    p = tmp_path / "f"
    p.write_bytes(raw)
    with pytest.raises(FormatError):
        read_volume(p)


def test_write_rejects_non_finite(tmp_path):
    vol = np.zeros((2, 2, 2))
    vol[1, 1, 1] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        write_volume(vol, tmp_path / "bad")
    assert not (tmp_path / "bad").exists()


def test_psf_errors(arrays):
    good = (GOLD / "psf_6x5x4_k3x3x5.bd3mgpsf").read_bytes()
    bad_k = good[:24] + struct.pack("<III", 3, 4, 5) + good[36:]
    with pytest.raises(FormatError, match=r"invalid kernel dimensions \(3, 4, 5\)"):
        blur.read_psf(io.BytesIO(bad_k))
    with pytest.raises(FormatError, match="truncated kernel payload"):
        blur.read_psf(io.BytesIO(good[:-8]))
    with pytest.raises(FormatError, match="truncated parameter records"):
        blur.read_psf(io.BytesIO(good[:40]))
    with pytest.raises(FormatError, match="trailing data"):
        blur.read_psf(io.BytesIO(good + b"\0"))
    with pytest.raises(FormatError, match="bad magic"):
        blur.read_psf(io.BytesIO(b"BD3MGVOL" + good[8:]))
