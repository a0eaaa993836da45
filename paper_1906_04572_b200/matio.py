"""CRUTVMAT binary matrix files streamed into the device path.

The reference's binary format (/root/reference/pkg/src/corutv/matio.py:24,
60-83): 8-byte magic ``CRUTVMAT``, two little-endian uint64 dimensions
(rows, cols), then the entries as little-endian float64, row-major.  The
reference reads the whole payload into memory and caps files at 1e9
entries (matio.py:78).  :func:`corutv_file` instead streams the rows from
disk through the library's pinned staging buffers straight into the device
(``corutv_decompose_stream``): the read of one ~1 GiB row chunk overlaps
the H2D copy and the first sketch sweeps of the previous one, so a 34 GB
(C3) or 68 GB (C5) matrix never has to fit in host memory.
"""

from __future__ import annotations

import ctypes
import os
import struct
import sys

import numpy as np

from . import _device as dev
from . import _lib
from .sketch import _VARIANT_CODE, CorUtvFactors, PassCounter, SketchConfig, pcg_state

__all__ = ["MAGIC", "read_header", "write_matrix_bin", "read_matrix_bin", "corutv_file"]

MAGIC = b"CRUTVMAT"   # matio.py:24
HEADER_BYTES = 24


def read_header(path) -> tuple[int, int]:
    """(rows, cols) of a CRUTVMAT file, with the reference's checks
    (matio.py:70-79) except the in-memory 1e9-entry cap; the payload length
    is checked against the file size."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
        header = fh.read(16)
    if len(header) != 16:
        raise ValueError(f"{path}: truncated header")
    rows, cols = struct.unpack("<QQ", header)
    if rows < 1 or cols < 1:
        raise ValueError(f"{path}: implausible dimensions {rows}x{cols}")
    if os.path.getsize(path) < HEADER_BYTES + 8 * rows * cols:
        raise ValueError(f"{path}: truncated payload")
    return int(rows), int(cols)


def write_matrix_bin(path, a) -> None:
    """matio.py:60-66."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ValueError(f"a must be 2-D, got shape {a.shape}")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<QQ", a.shape[0], a.shape[1]))
        fh.write(a.astype("<f8").tobytes())


def read_matrix_bin(path) -> np.ndarray:
    """matio.py:69-83 (in-memory read, with the reference's 1e9 cap)."""
    rows, cols = read_header(path)
    if rows * cols > 10**9:
        raise ValueError(f"{path}: implausible dimensions {rows}x{cols}")
    data = np.fromfile(path, dtype="<f8", count=rows * cols, offset=HEADER_BYTES)
    return data.astype(float).reshape(rows, cols)


class _RowReader:
    """read_rows callback: pread rows [row0, row0 + rows) into the library's
    pinned staging buffer (GIL released by the I/O)."""

    def __init__(self, path, cols):
        if sys.byteorder != "little":  # pragma: no cover
            raise OSError("CRUTVMAT streaming assumes a little-endian host")
        self.fd = os.open(path, os.O_RDONLY)
        self.cols = cols
        self.error = None
        self.fn = _lib.READ_ROWS_FN(self._read)

    def _read(self, user, row0, rows, dst, ld):  # noqa: ARG002
        try:
            if ld != self.cols:
                raise ValueError("unexpected staging leading dimension")
            nbytes = 8 * rows * self.cols
            view = memoryview((ctypes.c_char * nbytes).from_address(dst)).cast("B")
            off, pos = HEADER_BYTES + 8 * row0 * self.cols, 0
            while pos < nbytes:
                got = os.preadv(self.fd, [view[pos:]], off + pos)
                if got <= 0:
                    raise OSError(f"short read at byte {off + pos}")
                pos += got
            return 0
        except Exception as exc:  # surfaced as CORUTV_ERR_IO
            self.error = exc
            return 1

    def close(self):
        os.close(self.fd)


def corutv_file(path, cfg: SketchConfig, counter: PassCounter | None = None, omega=None) -> CorUtvFactors:
    """corutv (sketch.py:182-208) of the matrix stored in a CRUTVMAT file,
    streamed from disk to the device (the matrix never sits in host
    memory).  Factors come back as numpy arrays, bit-identical to
    ``corutv(read_matrix_bin(path), cfg)``."""
    torch = dev.torch_mod()
    m, n = read_header(path)
    if m < n:
        raise ValueError(f"corutv requires rows >= cols, got {m}x{n}")
    cfg.validated_for(m, n)
    ell = cfg.ell
    device = torch.device("cuda", torch.cuda.current_device())
    ld_dev = n + (n & 1)
    a_dev = torch.empty((m, ld_dev), dtype=torch.float64, device=device)
    u = torch.empty((m, ell), dtype=torch.float64, device=device)
    t = torch.empty((ell, ell), dtype=torch.float64, device=device)
    v = torch.empty((n, ell), dtype=torch.float64, device=device)
    perm = torch.empty((ell,), dtype=torch.int64, device=device)
    om = None
    if omega is not None:
        from .sketch import _omega_device
        om = _omega_device(omega, n, ell, cfg.seed, a_dev)
    passes = ctypes.c_int64(0)
    h = _lib.handle(device.index)
    reader = _RowReader(path, n)
    try:
        try:
            h.call("corutv_decompose_stream", reader.fn, None, m, n, dev.ptr(a_dev), ld_dev, ell, cfg.q_power,
                   _VARIANT_CODE[cfg.variant], None if om is None else dev.ptr(om),
                   None if om is not None else pcg_state(cfg.seed), dev.ptr(u), dev.ptr(t), dev.ptr(v),
                   dev.ptr(perm), ctypes.byref(passes))
        except OSError as exc:
            if reader.error is not None:
                raise OSError(f"{path}: {reader.error}") from reader.error
            raise exc
    finally:
        reader.close()
    if counter is not None:
        counter.add(passes.value)
    del a_dev
    return CorUtvFactors(u=u.cpu().numpy(), t=t.cpu().numpy(), v=v.cpu().numpy(), ell=ell,
                         q_power=cfg.q_power, variant=cfg.variant, perm=perm.cpu().numpy())
