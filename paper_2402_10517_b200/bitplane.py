"""Bitplane representation on the GPU -- drop-in for anyprec.bitplane.

Same names, arguments, layout semantics and exceptions as the reference
(bitplane.py:1-152 of anyprec 0.1.0); the byte work runs in sm_100a kernels
through the C ABI (include/anyprec_b200.h).

Kind in = kind out: numpy inputs give numpy outputs (computed on the GPU and
copied back), CUDA tensors stay on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _device as dev
from ._lib import check, load
from .errors import CodeRangeError, LayoutError, ParameterError, ShapeError

TILE_WEIGHTS = 1024
TILE_BYTES = TILE_WEIGHTS // 8
LANES = 32
WORD_BYTES = 4

LAYOUT_LINEAR = "linear"
LAYOUT_PERMUTED = "permuted"

# out[4t + j] = in[32j + t]   (bitplane.py:31-36) -- host geometry only
_PERM = np.array([32 * (p & 3) + (p >> 2) for p in range(TILE_BYTES)], dtype=np.int64)


@dataclass
class BitplaneTensor:
    """n_max bit matrices; plane p holds code bit n_max-1-p (bitplane.py:40-69).

    ``planes`` is a uint8 (n_max, rows, padded_cols // 8) numpy array or CUDA
    tensor.
    """

    planes: object
    rows: int
    cols: int
    padded_cols: int
    layout: str

    def __post_init__(self):
        shape = tuple(self.planes.shape)
        if _dtype_name(self.planes) != "uint8" or len(shape) != 3:
            raise ShapeError("planes must be a 3-D uint8 array")
        if self.layout not in (LAYOUT_LINEAR, LAYOUT_PERMUTED):
            raise ParameterError(f"unknown layout {self.layout!r}")
        if self.padded_cols % TILE_WEIGHTS != 0:
            raise ShapeError(f"padded columns must be a multiple of {TILE_WEIGHTS}")
        expect = (shape[0], self.rows, self.padded_cols // 8)
        if shape != expect:
            raise ShapeError(f"planes shape {shape} != expected {expect}")
        if not 0 < self.cols <= self.padded_cols:
            raise ShapeError("column count out of range")

    @property
    def n_max(self) -> int:
        return int(self.planes.shape[0])

    @property
    def n_tiles(self) -> int:
        return self.padded_cols // TILE_WEIGHTS

    @property
    def on_device(self) -> bool:
        return dev.is_tensor(self.planes)

    def device_planes(self):
        """The planes as a contiguous CUDA uint8 tensor (uploads numpy once)."""
        return dev.to_device(self.planes)

    def to_device(self) -> "BitplaneTensor":
        return replace(self, planes=self.device_planes())

    def numpy(self) -> "BitplaneTensor":
        p = self.planes.cpu().numpy() if dev.is_tensor(self.planes) else self.planes
        return replace(self, planes=p)


def _dtype_name(a) -> str:
    if dev.is_tensor(a):
        return str(a.dtype).replace("torch.", "")
    return str(np.asarray(a).dtype) if not hasattr(a, "dtype") else str(a.dtype)


def pad_columns(cols: int) -> int:
    """bitplane.py:72-73"""
    return -(-cols // TILE_WEIGHTS) * TILE_WEIGHTS


def _validate_codes(codes, n_max: int):
    """bitplane.py:83-91 -- same checks, same exception classes, same order."""
    is_t = dev.is_tensor(codes)
    if not is_t:
        codes = np.asarray(codes)
    ndim = codes.dim() if is_t else codes.ndim
    size = codes.numel() if is_t else codes.size
    if ndim != 2 or size == 0:
        raise ShapeError("code matrix must be a non-empty 2-D array")
    if not 1 <= n_max <= 8:
        raise ParameterError(f"n_max {n_max} outside [1, 8]")
    if is_t:
        t = dev.torch()
        if codes.dtype.is_floating_point or codes.dtype == t.bool or codes.dtype.is_complex:
            raise CodeRangeError("codes must be integers")
        if codes.dtype != t.uint8:
            lo, hi = int(codes.min()), int(codes.max())
            if lo < 0 or hi >= (1 << n_max):
                raise CodeRangeError(f"codes exceed {n_max}-bit range")
            codes = codes.to(t.uint8)
        return codes, True
    if not np.issubdtype(codes.dtype, np.integer):
        raise CodeRangeError("codes must be integers")
    if codes.dtype != np.uint8:
        if codes.min() < 0 or codes.max() >= (1 << n_max):
            raise CodeRangeError(f"codes exceed {n_max}-bit range")
        codes = codes.astype(np.uint8)
    return codes, False


def _pack_device(codes_dev, n_max: int, permuted: bool):
    """Run the packer kernel; returns (planes tensor, padded).  Raises
    CodeRangeError when any code has bits at or above n_max."""
    t = dev.require_cuda()
    rows, cols = int(codes_dev.shape[0]), int(codes_dev.shape[1])
    padded = pad_columns(cols)
    planes = t.empty((n_max, rows, padded // 8), dtype=t.uint8, device=codes_dev.device)
    flag = t.zeros(1, dtype=t.int32, device=codes_dev.device)
    lib = load()
    check(
        lib.apb_pack(dev.ptr(codes_dev), rows, cols, int(codes_dev.stride(0)), n_max,
                     1 if permuted else 0, dev.ptr(planes), dev.ptr(flag), dev.stream_ptr()),
        "apb_pack",
    )
    code_or = int(flag.item())
    if code_or >> n_max:
        raise CodeRangeError(f"codes exceed {n_max}-bit range")
    return planes, padded


def pack_bitplanes(codes, n_max: int) -> BitplaneTensor:
    """Decompose a code matrix into MSB-first bitplanes, linear layout
    (bitplane.py:76-100).  The column tail packs as zero bits."""
    codes, is_t = _validate_codes(codes, n_max)
    codes_dev = dev.to_device(codes)
    planes, padded = _pack_device(codes_dev, n_max, permuted=False)
    rows, cols = int(codes_dev.shape[0]), int(codes_dev.shape[1])
    out = planes if is_t else planes.cpu().numpy()
    return BitplaneTensor(out, rows, cols, padded, LAYOUT_LINEAR)


def pack_permuted(codes, n_max: int) -> BitplaneTensor:
    """pack_bitplanes + permute_layout fused in one kernel pass (what
    engine.prepare uses, engine.py:151-152).  Always returns device planes."""
    codes, _ = _validate_codes(codes, n_max)
    codes_dev = dev.to_device(codes)
    planes, padded = _pack_device(codes_dev, n_max, permuted=True)
    return BitplaneTensor(planes, int(codes_dev.shape[0]), int(codes_dev.shape[1]), padded,
                          LAYOUT_PERMUTED)


def _permute(t: BitplaneTensor, inverse: bool) -> object:
    torch = dev.require_cuda()
    src = t.device_planes()
    out = torch.empty_like(src)
    check(
        load().apb_permute(dev.ptr(src), dev.ptr(out), t.n_max, t.rows, t.padded_cols,
                           1 if inverse else 0, dev.stream_ptr()),
        "apb_permute",
    )
    return out if t.on_device else out.cpu().numpy()


def permute_layout(t: BitplaneTensor) -> BitplaneTensor:
    """Rearrange each 128-byte tile for coalesced lane-major word reads
    (bitplane.py:126-130)."""
    if t.layout != LAYOUT_LINEAR:
        raise LayoutError("tensor is already permuted")
    return replace(t, planes=_permute(t, False), layout=LAYOUT_PERMUTED)


def inverse_permute_layout(t: BitplaneTensor) -> BitplaneTensor:
    """bitplane.py:133-136"""
    if t.layout != LAYOUT_PERMUTED:
        raise LayoutError("tensor is not permuted")
    return replace(t, planes=_permute(t, True), layout=LAYOUT_LINEAR)


def unpack_codes(t: BitplaneTensor, k: int):
    """Top-k-bit prefix codes from the first k planes only (bitplane.py:103-118)."""
    if not 1 <= k <= t.n_max:
        raise ParameterError(f"k={k} outside [1, {t.n_max}]")
    torch = dev.require_cuda()
    src = t.device_planes()
    out = torch.empty((t.rows, t.cols), dtype=torch.uint8, device=src.device)
    check(
        load().apb_unpack(dev.ptr(src), t.n_max, t.rows, t.cols, t.padded_cols,
                          1 if t.layout == LAYOUT_PERMUTED else 0, k, dev.ptr(out), t.cols,
                          dev.stream_ptr()),
        "apb_unpack",
    )
    return out if t.on_device else out.cpu().numpy()


def tile_permutation() -> np.ndarray:
    """The per-tile byte mapping (bitplane.py:139-141): output p reads input _PERM[p]."""
    return _PERM.copy()


def lane_weight_indices(lane: int) -> np.ndarray:
    """Weight indices covered by one lane's 4-byte word (bitplane.py:144-152)."""
    if not 0 <= lane < LANES:
        raise ParameterError(f"lane {lane} outside [0, {LANES})")
    return np.array(
        [256 * q + 8 * lane + i for q in range(WORD_BYTES) for i in range(8)], dtype=np.int64
    )
