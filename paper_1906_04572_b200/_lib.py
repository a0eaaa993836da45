"""ctypes binding of the C-ABI in include/corutv_b200.h.

The shared library ``libcorutv_b200.so`` is built in-tree (``python
__graft_entry__.py`` or ``python -m paper_1906_04572_b200.build``).  There
is no fallback: if the library or a CUDA device is missing, every device
entry point raises :class:`DeviceUnavailable` loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import ConvergenceError, CorutvError

LIB_NAME = "libcorutv_b200.so"
# CORUTV_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = Path(os.environ["CORUTV_LIB"]).resolve() if os.environ.get("CORUTV_LIB") else \
    Path(__file__).resolve().parent / LIB_NAME

OK, ERR_SHAPE, ERR_NONFINITE, ERR_CUDA, ERR_COMM, ERR_CONVERGENCE, ERR_ARG, ERR_NOMEM, ERR_IO = range(9)
EXACT_D, APPROX_D = 0, 1

c_double_p = ctypes.POINTER(ctypes.c_double)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                ctypes.c_void_p)
READ_ROWS_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_void_p, ctypes.c_int64)

# name -> (restype, argtypes); mirrors include/corutv_b200.h
_VP, _I64, _I32, _D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
SIGNATURES = {
    "corutv_version": (_I32, []),
    "corutv_create": (_I32, [_I32, _VP, ctypes.POINTER(_VP)]),
    "corutv_destroy": (None, [_VP]),
    "corutv_set_stream": (_I32, [_VP, _VP]),
    "corutv_last_error": (ctypes.c_char_p, [_VP]),
    "corutv_set_comm": (_I32, [_VP, ALLREDUCE_FN, _VP, _I32, _I32]),
    "corutv_decompose": (_I32, [_VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _VP, _VP, _VP, _VP,
                                _VP, c_int64_p]),
    "corutv_decompose_seeded": (_I32, [_VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _VP, _VP, _VP,
                                       _VP, _VP, c_int64_p]),
    "corutv_gaussian": (_I32, [_VP, _VP, _I64, _I64, _VP, _I64]),
    "corutv_decompose_stream": (_I32, [_VP, READ_ROWS_FN, _VP, _I64, _I64, _VP, _I64, _I32, _I32, _I32, _VP,
                                       _VP, _VP, _VP, _VP, _VP, c_int64_p]),
    "corutv_sor_svd_host": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _I64, _I32, _I32, _I32, _VP, _VP, _VP,
                                   _VP, _VP, c_int64_p]),
    "corutv_tsr_svd_host": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _I64, _I32, _VP, _VP, _VP, _VP, _VP,
                                   _VP, _VP, c_int64_p]),
    "corutv_upload": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _I64]),
    "corutv_download": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _I64]),
    "corutv_jacobi_svd": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _VP, _VP]),
    "corutv_jacobi_svd_warm": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _I64, _D, _I32, _VP, _VP, _VP]),
    "corutv_lowrank_error_rank": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _VP, _VP, _I32, _I32, c_double_p]),
    "corutv_qrcp": (_I32, [_VP, _VP, _I64, _I64, _VP, _VP, _VP]),
    "corutv_qrcp_mn": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP]),
    "corutv_svt": (_I32, [_VP, _VP, _I64, _I64, _I64, _D, _I32, _VP, _I64, _VP, _VP, _VP, _VP,
                          ctypes.POINTER(_I32)]),
    "corutv_sor_svd": (_I32, [_VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _VP, _VP, _VP, _VP, _VP,
                              c_int64_p]),
    "corutv_tsr_svd": (_I32, [_VP, _VP, _I64, _I64, _I64, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                              c_int64_p]),
    "corutv_decompose_host": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _I64, _I32, _I32, _I32, _VP, _VP,
                                     _VP, _VP, _VP, _VP, c_int64_p]),
    "corutv_decompose_truncated": (_I32, [_VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _VP, _VP, _D,
                                          _VP, _VP, _VP, _VP, c_int64_p, ctypes.POINTER(_I32)]),
    "corutv_alm_update": (_I32, [_VP, _VP, _VP, _VP, _VP, _I64, _I64, _VP, _VP, _VP, _I32, _I32,
                                 _D, _D, _D, c_double_p, c_int64_p]),
    "corutv_lowrank": (_I32, [_VP, _VP, _VP, _VP, _I64, _I64, _I32, _I32, _VP]),
    "corutv_spectral_norm": (_I32, [_VP, _VP, _I64, _I64, _I64, _D, _I32, c_double_p,
                                    ctypes.POINTER(_I32)]),
    "corutv_singular_values": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP]),
    "corutv_sumsq": (_I32, [_VP, _VP, _I64, _I64, _I64, c_double_p]),
    "corutv_count_nonfinite": (_I32, [_VP, _VP, _I64, _I64, _I64, c_int64_p]),
    "corutv_shrink": (_I32, [_VP, _VP, _I64, _I64, _I64, _D, _VP, _I64]),
    "corutv_set_global_rows": (_I32, [_VP, _I64]),
    "corutv_nccl_unique_id": (_I32, [_VP]),
    "corutv_nccl_comm_create": (_I32, [_I32, _VP, _I32, _I32, ctypes.POINTER(_VP)]),
    "corutv_nccl_comm_destroy": (_I32, [_VP]),
    "corutv_set_nccl": (_I32, [_VP, _VP, _I32, _I32]),
    "corutv_lowrank_error": (_I32, [_VP, _VP, _I64, _I64, _I64, _VP, _VP, _VP, _I32, c_double_p]),
    "corutv_gemm": (_I32, [_VP, _I32, _I64, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _I64]),
    "corutv_profile_begin": (_I32, [_VP]),
    "corutv_profile_end": (_I32, [_VP, c_double_p, c_int64_p]),
}


class DeviceUnavailable(CorutvError):
    """The sm_100a library or a CUDA device is missing (no CPU fallback)."""


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load and type the shared library (does not need a GPU)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise DeviceUnavailable(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(status: int, handle=None, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception types (errors.py)."""
    if status == OK:
        return
    msg = ""
    if handle is not None:
        raw = load_library().corutv_last_error(handle)
        msg = raw.decode() if raw else ""
    text = f"{what}: {msg}" if what else msg
    if status in (ERR_SHAPE, ERR_NONFINITE, ERR_ARG):
        raise ValueError(msg or text)
    if status == ERR_CONVERGENCE:
        raise ConvergenceError(text)
    if status == ERR_IO:
        raise OSError(text)
    raise CorutvError(f"{text} (status {status})")


class Handle:
    """One native handle per (thread, device); bound to torch's current
    stream at each call."""

    def __init__(self, device: int):
        import torch

        if not torch.cuda.is_available():
            raise DeviceUnavailable("no CUDA device: the CoR-UTV B200 path has no CPU fallback")
        self.lib = load_library()
        self.device = device
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            check(self.lib.corutv_create(device, None, ctypes.byref(h)), None, "corutv_create")
        self.ptr = h
        self._comm_keepalive = None

    def bind_stream(self):
        import torch

        s = torch.cuda.current_stream(self.device).cuda_stream
        self.lib.corutv_set_stream(self.ptr, ctypes.c_void_p(s))

    def call(self, name, *args):
        self.bind_stream()
        status = getattr(self.lib, name)(self.ptr, *args)
        check(status, self.ptr, name)

    def __del__(self):
        try:
            if getattr(self, "ptr", None):
                self.lib.corutv_destroy(self.ptr)
        except Exception:
            pass


_tls = threading.local()


def handle(device: int | None = None) -> Handle:
    """Per-thread handle for ``device`` (default: torch's current device)."""
    import torch

    if device is None:
        if not torch.cuda.is_available():
            raise DeviceUnavailable("no CUDA device: the CoR-UTV B200 path has no CPU fallback")
        device = torch.cuda.current_device()
    cache = getattr(_tls, "handles", None)
    if cache is None:
        cache = _tls.handles = {}
    h = cache.get(device)
    if h is None:
        h = cache[device] = Handle(device)
    return h
