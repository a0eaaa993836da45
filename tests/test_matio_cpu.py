"""CRUTVMAT format handling (matio.py:24, 60-83) -- no GPU needed."""

import struct

import numpy as np
import pytest

from paper_1906_04572_b200 import matio


def test_roundtrip_and_layout(tmp_path):
    a = np.random.Generator(np.random.PCG64(1)).standard_normal((7, 5))
    p = tmp_path / "a.bin"
    matio.write_matrix_bin(p, a)
    raw = p.read_bytes()
    assert raw[:8] == b"CRUTVMAT"
    assert struct.unpack("<QQ", raw[8:24]) == (7, 5)
    assert np.array_equal(np.frombuffer(raw[24:], dtype="<f8").reshape(7, 5), a)
    assert matio.read_header(p) == (7, 5)
    assert np.array_equal(matio.read_matrix_bin(p), a)


def test_header_errors(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOTAMAT!" + bytes(16))
    with pytest.raises(ValueError, match="bad magic"):
        matio.read_header(p)
    p.write_bytes(b"CRUTVMAT" + bytes(5))
    with pytest.raises(ValueError, match="truncated header"):
        matio.read_header(p)
    p.write_bytes(b"CRUTVMAT" + struct.pack("<QQ", 0, 3))
    with pytest.raises(ValueError, match="implausible"):
        matio.read_header(p)
    p.write_bytes(b"CRUTVMAT" + struct.pack("<QQ", 4, 3) + bytes(8 * 11))
    with pytest.raises(ValueError, match="truncated payload"):
        matio.read_header(p)
