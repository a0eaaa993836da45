"""Host <-> device marshalling shared by the API modules.

Inputs may be numpy-compatible host arrays (copied to the current CUDA
device) or torch CUDA tensors (used in place, zero-copy when float64 and
C-contiguous).  Outputs follow the input's residency, like the reference's
pure functions return fresh numpy arrays (dense.py:4-7).
"""

from __future__ import annotations

import numpy as np

from ._lib import DeviceUnavailable

UPLOAD_MIN_BYTES = 64 << 20  # numpy inputs above this go through corutv_upload


def torch_mod():
    import torch

    if not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device: the CoR-UTV B200 path has no CPU fallback")
    return torch


def is_device_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def shape_check(x, name):
    """The structural part of as_matrix (dense.py:41-47); finiteness is
    checked on the device."""
    if is_device_tensor(x) or is_host_tensor(x):
        shape = tuple(x.shape)
    else:
        x = np.asarray(x, dtype=float)
        shape = x.shape
    if len(shape) != 2:
        raise ValueError(f"{name} must be 2-D, got shape {shape}")
    if shape[0] < 1 or shape[1] < 1:
        raise ValueError(f"{name} must have positive dimensions, got {shape}")
    return x


def is_host_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and not x.is_cuda


def to_device(x, name="matrix", pin=False):
    """Return (device float64 tensor with unit inner stride, was_host).

    Host torch tensors (e.g. pinned buffers) are copied asynchronously on
    the current stream; results for them come back as host torch tensors."""
    torch = torch_mod()
    if is_host_tensor(x):
        if x.dim() != 2:
            raise ValueError(f"{name} must be 2-D, got shape {tuple(x.shape)}")
        if x.shape[0] < 1 or x.shape[1] < 1:
            raise ValueError(f"{name} must have positive dimensions, got {tuple(x.shape)}")
        t = x.to(torch.cuda.current_device(), dtype=torch.float64, non_blocking=True)
        if t.stride(1) != 1:
            t = t.contiguous()
        return t, "torch"
    x = shape_check(x, name)
    if is_device_tensor(x):
        t = x
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        if t.stride(1) != 1 or t.stride(0) < t.shape[1]:
            t = t.contiguous()
        return t, False
    host = np.ascontiguousarray(x, dtype=np.float64)
    if host.nbytes >= UPLOAD_MIN_BYTES and not pin:
        # large arrays: the library's chunked upload (pinned staging filled by
        # all host cores; the driver's pageable path moves ~11 GB/s)
        from . import _lib

        dev_t = torch.empty(host.shape, dtype=torch.float64, device=torch.cuda.current_device())
        h = _lib.handle(dev_t.device.index)
        h.call("corutv_upload", host.ctypes.data, host.shape[0], host.shape[1], host.shape[1], ptr(dev_t),
               host.shape[1])
        return dev_t, True
    src = torch.from_numpy(host)
    if pin:
        src = src.pin_memory()
    return src.to(torch.cuda.current_device(), non_blocking=pin), True


def to_output(t, was_host):
    if was_host == "torch":
        return t.cpu()
    if was_host:
        if (t.dim() == 2 and t.numel() * 8 >= UPLOAD_MIN_BYTES and t.stride(1) == 1
                and str(t.dtype) == "torch.float64"):
            # large results (L, S of the ALM solver): chunked pinned staging,
            # copied out by all host cores
            from . import _lib

            out = np.empty(tuple(t.shape), dtype=np.float64)
            h = _lib.handle(t.device.index)
            h.call("corutv_download", ptr(t), t.shape[0], t.shape[1], t.stride(0), out.ctypes.data, t.shape[1])
            return out
        return t.cpu().numpy()
    return t


def ptr(t) -> int:
    return t.data_ptr()


def raise_if_nonfinite(t, name):
    """as_matrix's finiteness check (dense.py:48-49) on the device
    (corutv_count_nonfinite): ValueError "<name> contains non-finite
    entries"."""
    import ctypes

    from . import _lib

    if t.dim() != 2 or t.numel() == 0:
        return
    if t.stride(1) != 1 or t.stride(0) < t.shape[1] or str(t.dtype) != "torch.float64":
        t = t.to(torch_mod().float64).contiguous()
    cnt = ctypes.c_int64(0)
    h = _lib.handle(t.device.index)
    h.call("corutv_count_nonfinite", ptr(t), t.shape[0], t.shape[1], t.stride(0), ctypes.byref(cnt))
    if cnt.value:
        raise ValueError(f"{name} contains non-finite entries")
