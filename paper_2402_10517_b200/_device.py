"""Device plumbing: torch supplies CUDA memory and streams (never compute here)."""

from __future__ import annotations

import numpy as np

from .errors import DeviceError


def torch():
    import torch as _t

    return _t


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    t = torch()
    if not _CUDA_OK:  # once a device was found it stays there: skip the per-call probe
        if not t.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 kernels have no CPU fallback")
        _CUDA_OK = True
    return t


def stream_ptr():
    """The current torch CUDA stream of the current device (raw handle)."""
    t = require_cuda()
    return t._C._cuda_getCurrentRawStream(t._C._cuda_getDevice())


def is_tensor(a) -> bool:
    t = torch()
    return isinstance(a, t.Tensor)


def to_device(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (no copy if already there)."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        out = a if a.is_cuda else a.cuda()
    else:
        arr = np.ascontiguousarray(a)
        out = t.from_numpy(arr).cuda()
    if dtype is not None and out.dtype != dtype:
        out = out.to(dtype)
    return out.contiguous()


def ptr(tensor) -> int:
    return int(tensor.data_ptr())
