"""Device plumbing: torch supplies CUDA memory and streams (never compute here)."""

from __future__ import annotations

import numpy as np

from .errors import DeviceError


def torch():
    import torch as _t

    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 kernels have no CPU fallback")
    return t


def stream_ptr():
    t = require_cuda()
    return t.cuda.current_stream().cuda_stream


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
