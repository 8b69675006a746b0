"""Bitplane GEMV / GEMM engine on B200 -- drop-in for anyprec.engine.

Same public names, argument meaning, dispatch rules, counters and exceptions
as the reference (engine.py:1-362 of anyprec 0.1.0).  The arithmetic runs in
the sm_100a kernels of ``csrc/`` through the C ABI; numpy in -> numpy out,
CUDA tensors in -> CUDA tensors out.

Numerics: the reference accumulates in fp32 (engine.py:123-125).  The GPU path
multiplies fp16 centroids by fp16 activations in the tensor core with fp32
accumulation.  With ``activations_fp16=True`` (or fp16 inputs) that is exact
input semantics; otherwise an fp32 activation is split into two fp16 halves
(x = hi + lo, ~22 significant bits) carried as two extra batch columns of the
same MMA, so the default path stays within ~1e-6 of the fp32 reference.
"""

from __future__ import annotations

import os

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _device as dev
from ._lib import APB_DTYPE_F16, APB_DTYPE_F32, check, int64_array, int_array, load, ptr_array
from .bitplane import (  # noqa: F401  (pack_bitplanes: re-exported like the reference's engine module)
    LANES,
    LAYOUT_PERMUTED,
    TILE_WEIGHTS,
    BitplaneTensor,
    pack_bitplanes,
    pack_permuted,
    permute_layout,
)
from .errors import ParameterError, ShapeError
from .layer import AnyPrecisionLayer, supported_bits  # noqa: F401  (re-exported like the reference)

# Op budget of the REFERENCE's delta-swap network (engine.py:44-45); kept for
# API parity.  The kernels use the select-form networks of csrc/apb_common.cuh.
TRANSPOSE_OP_COUNT = {2: 6, 4: 24, 8: 72}


# ---- SWAR transpose (bit-exact, on the GPU) --------------------------------

def _words_kind_call(plane_words, k: int):
    torch = dev.require_cuda()
    is_t = dev.is_tensor(plane_words)
    if is_t:
        # raw 32-bit patterns; int64 -> int32 wraps, i.e. keeps the low 32 bits
        w = plane_words.cuda()
        if w.dtype != torch.int32:
            w = w.to(torch.int64).to(torch.int32)
        w = w.contiguous()
    else:
        w = dev.to_device(np.ascontiguousarray(np.asarray(plane_words).astype(np.uint32)).view(np.int32))
    b = 2 if k <= 2 else 4 if k <= 4 else 8
    tail = tuple(w.shape[1:])
    n = int(np.prod(tail)) if tail else 1
    out = torch.empty((b,) + tail, dtype=torch.int32, device=w.device)
    check(load().apb_transpose_words(dev.ptr(w), k, n, dev.ptr(out), dev.stream_ptr()),
          "apb_transpose_words")
    return out.view(torch.uint32) if is_t else out.cpu().numpy().view(np.uint32)


def bit_transpose(words):
    """Transpose the B x B bit blocks of B stacked 32-bit words (engine.py:48-72).
    Output bit (g, s*B + b) equals input bit (b, s*B + g)."""
    is_t = dev.is_tensor(words)
    if not is_t:
        words = np.asarray(words)
    shape = tuple(words.shape)
    b = shape[0] if len(shape) else 0
    if len(shape) < 1 or b not in (2, 4, 8):
        raise ParameterError("word count must be 2, 4 or 8")
    # bit_transpose(w) == transpose_any_width(w[::-1], B)  (engine.py:90-91)
    rev = words.flip(0) if is_t else words[::-1]
    if len(shape) == 1:
        rev = rev.unsqueeze(1) if is_t else rev[:, None]
        return _words_kind_call(rev, b)[:, 0]
    return _words_kind_call(rev, b)


def transpose_any_width(plane_words, k: int):
    """k plane words (MSB plane first) -> packed per-weight codes (engine.py:75-92)."""
    if not 2 <= k <= 8:
        raise ParameterError(f"bit width {k} outside [2, 8]")
    shape = tuple(plane_words.shape) if hasattr(plane_words, "shape") else np.shape(plane_words)
    if shape[0] != k:
        raise ShapeError(f"expected {k} plane words, got {shape[0]}")
    return _words_kind_call(plane_words, k)


# ---- merged 3-bit table (host helpers, engine.py:95-120) -----------------------

@dataclass
class MergedTable3:
    """64 centroid pairs: entry 8*i + j holds (c_i, c_j)."""

    entries: np.ndarray  # (64, 2) float32

    def lookup(self, merged_index: int) -> tuple:
        pair = self.entries[merged_index]
        return float(pair[0]), float(pair[1])


def _merged_entries(tables: np.ndarray) -> np.ndarray:
    rows = tables.shape[0]
    out = np.empty((rows, 64, 2), dtype=np.float32)
    out[:, :, 0] = np.repeat(tables, 8, axis=1)
    out[:, :, 1] = np.tile(tables, (1, 8))
    return out


def build_merged_table(centroids) -> MergedTable3:
    centroids = np.asarray(centroids, dtype=np.float32)
    if centroids.shape != (8,):
        raise ParameterError(f"expected exactly 8 centroids, got shape {centroids.shape}")
    return MergedTable3(_merged_entries(centroids[None, :])[0])


# ---- config / report ---------------------------------------------------------

@dataclass(frozen=True)
class GemvConfig:
    """Execution knobs (engine.py:123-135); accumulation is always fp32."""

    bit_width: int
    dense_threshold: int = 16
    activations_fp16: bool = False
    use_merged_table: bool | None = None  # None: merged exactly at 3 bits

    def merged(self) -> bool:
        if self.use_merged_table is None:
            return self.bit_width == 3
        return self.use_merged_table


@dataclass
class ExecutionReport:
    """Analytic byte counters and path (engine.py:138-143)."""

    planes_bytes_read: int = 0
    table_bytes_read: int = 0
    path_taken: str = ""
    extra: dict = field(default_factory=dict)


# ---- prepared layer ------------------------------------------------------------

class PreparedLayer:
    """Inference-ready, device-resident view: permuted planes plus one fp16
    table per bit-width (engine.py:146-173).  Immutable after construction."""

    def __init__(self, layer, tensor: BitplaneTensor | None = None):
        torch = dev.require_cuda()
        self.layer = layer
        if tensor is None:
            tensor = pack_permuted(layer.codes, layer.n_max)  # engine.py:151-152, one pass
        elif tensor.layout != LAYOUT_PERMUTED:
            tensor = permute_layout(tensor.to_device())
        else:
            tensor = tensor.to_device()
        if (tensor.rows, tensor.cols) != tuple(layer.shape) or tensor.n_max != layer.n_max:
            raise ShapeError("bitplane tensor does not match the layer")
        self.tensor = tensor
        self.tables16 = {}
        for k in supported_bits(layer):
            t = layer.centroid_tables[k]
            if dev.is_tensor(t):
                t16 = t.to(device="cuda", dtype=torch.float16).contiguous()
            else:
                t16 = dev.to_device(np.ascontiguousarray(np.asarray(t).astype(np.float16)))
            if tuple(t16.shape) != (tensor.rows, 1 << k):
                raise ShapeError(f"centroid table {k} has shape {tuple(t16.shape)}")
            self.tables16[k] = t16
        self._merged = None
        self._tls = threading.local()  # per-thread launch plans of the per-call API

    def _call_plan(self, k: int, m_x: int, split: int):
        """The cached launch plan of this (k, activation rows, split) for the
        calling thread (plans hold mutable pointers: never shared across threads)."""
        plans = getattr(self._tls, "plans", None)
        if plans is None:
            plans = self._tls.plans = {}
        key = (k, m_x, split)
        if key not in plans:
            plans[key] = _CallPlan(self, k, m_x, split)
        return plans[key]

    @property
    def planes(self):
        return self.tensor.planes

    @property
    def tables32(self) -> dict:
        return {k: t.float().cpu().numpy() for k, t in self.tables16.items()}

    def merged_pairs(self) -> np.ndarray:
        if 3 not in self.tables16:
            raise ParameterError("layer does not support 3-bit")
        if self._merged is None:
            self._merged = _merged_entries(self.tables16[3].float().cpu().numpy())
        return self._merged


def prepare(layer, tensor: BitplaneTensor | None = None) -> PreparedLayer:
    return PreparedLayer(layer, tensor)


# ---- helpers -------------------------------------------------------------------------

def _check_bit_width(layer, k: int):
    if k not in supported_bits(layer):
        raise ParameterError(
            f"bit width {k} unsupported; layer holds [{layer.n_min}, {layer.n_max}]"
        )


def _ldx(cols: int) -> int:
    return -(-cols // 8) * 8


def _split_tail_halves(m: int) -> int:
    """fp16 elements that hold the m fp32 inverse scales behind a scaled-pair
    block (x_split = 2), rounded up to 16 bytes."""
    return -(-2 * m // 8) * 8


def _split_scaled_np(x32: np.ndarray, ldx: int) -> np.ndarray:
    """Host restatement of apb_split_x_scaled (csrc/apb_dense.cu): flat fp16
    [2m*ldx + tail] = (hi, lo) row pairs of x * s_r followed by float32 1/s_r,
    s_r the power of two putting row r's max |x| in [2^14, 2^15)."""
    m, cols = x32.shape
    out = np.zeros(2 * m * ldx + _split_tail_halves(m), dtype=np.float16)
    rows = out[: 2 * m * ldx].reshape(2 * m, ldx)
    inv = np.ones(m, dtype=np.float32)
    for r in range(m):
        a = float(np.max(np.abs(x32[r]))) if cols else 0.0
        scale = np.float32(1.0)
        if a > 0.0 and np.isfinite(a):
            e = int(np.frexp(np.float32(a))[1])
            scale = np.float32(np.ldexp(np.float32(1.0), min(max(15 - e, -126), 126)))
        v = x32[r] * scale  # exact: a power of two
        hi = v.astype(np.float16)
        rows[2 * r, :cols] = hi
        rows[2 * r + 1, :cols] = (v - hi.astype(np.float32)).astype(np.float16)
        inv[r] = np.float32(1.0) / scale
    out[2 * m * ldx:2 * m * ldx + 2 * m] = inv.view(np.float16)
    return out


def _stage_x(x, cols: int, fp16: bool):
    """_prep_x (engine.py:270-281) for the GPU: returns (xdev fp16 [m_x][ldx],
    m_x, ldx, split, host_kind).  fp32 activations become scaled (hi, lo) fp16
    pairs (x_split = 2: the block carries its inverse row scales behind the
    rows, so any fp32 magnitude keeps ~22 significant bits)."""
    torch = dev.require_cuda()
    ldx = _ldx(cols)
    if dev.is_tensor(x):
        kind = "cuda" if x.is_cuda else "tensor"
        # host tensors (ideally pinned) are copied asynchronously on the current stream
        x2 = x if x.is_cuda else x.cuda(non_blocking=True)
        m = x2.shape[0]
        if x2.dtype == torch.float16 or fp16:
            if x2.dtype != torch.float16:
                x2 = x2.to(torch.float32).to(torch.float16)
            if x2.is_contiguous() and cols % 8 == 0 and x2.data_ptr() % 16 == 0:
                return x2, m, ldx, 0, kind
            buf = torch.zeros((m, ldx), dtype=torch.float16, device=x2.device)
            buf[:, :cols] = x2
            return buf, m, ldx, 0, kind
        x32 = x2.to(torch.float32).contiguous()
        flat = torch.empty(2 * m * ldx + _split_tail_halves(m), dtype=torch.float16, device=x2.device)
        check(load().apb_split_x_scaled(dev.ptr(x32), m, cols, cols, dev.ptr(flat), ldx,
                                        dev.stream_ptr()), "apb_split_x_scaled")
        return flat[: 2 * m * ldx].view(2 * m, ldx), 2 * m, ldx, 2, kind
    x = np.asarray(x)
    m = x.shape[0]
    if fp16 or x.dtype == np.float16:
        h = np.zeros((m, ldx), dtype=np.float16)
        h[:, :cols] = x.astype(np.float16)
        return dev.to_device(h), m, ldx, 0, "numpy"
    flat = dev.to_device(_split_scaled_np(x.astype(np.float32), ldx))
    return flat[: 2 * m * ldx].view(2 * m, ldx), 2 * m, ldx, 2, "numpy"


class _CallPlan:
    """One (layer, k, activation rows) launch of the per-call API: a caller-owned
    C launch plan (apb_gemv_plan_create: validation, tensor maps and partition
    done once) plus device and pinned host staging buffers reused across calls.
    ``handle`` is None when the TMA kernel does not serve the shape (k = 2,
    m_x > 8, > 64K columns): the caller then uses apb_gemv directly."""

    def __init__(self, prep: PreparedLayer, k: int, m_x: int, split: int):
        torch = dev.torch()
        t = prep.tensor
        self.m_x, self.split, self.ldx = m_x, split, _ldx(t.cols)
        self.m_out = m_x // 2 if split else m_x
        # scaled pairs (split = 2) carry their inverse row scales behind the rows
        n_x = m_x * self.ldx + (_split_tail_halves(self.m_out) if split == 2 else 0)
        self._x_flat = torch.zeros(n_x, dtype=torch.float16, device="cuda")
        self._x_pin_flat = torch.zeros(n_x, dtype=torch.float16, pin_memory=True)
        self.x = self._x_flat[: m_x * self.ldx].view(m_x, self.ldx)
        self.y = torch.empty((self.m_out, t.rows), dtype=torch.float32, device="cuda")
        self.x_pin = self._x_pin_flat[: m_x * self.ldx].view(m_x, self.ldx)
        self.y_pin = torch.empty((self.m_out, t.rows), dtype=torch.float32, pin_memory=True)
        self._lib = load()
        PP = lambda a: ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))  # noqa: E731
        self._keep = (ptr_array([dev.ptr(t.planes)]), int_array([t.n_max]), int64_array([t.rows]),
                      int64_array([t.cols]), int64_array([t.padded_cols]), ptr_array([dev.ptr(prep.tables16[k])]),
                      ptr_array([dev.ptr(self.x)]), int64_array([self.ldx]), ptr_array([dev.ptr(self.y)]),
                      int64_array([t.rows]))
        pl, nm, rw, cl, pd, lt, xp, lx, yp, ly = self._keep
        h = self._lib.apb_gemv_plan_create(1, PP(pl), nm, rw, cl, pd, k, PP(lt), PP(xp), m_x, lx, split, PP(yp),
                                           APB_DTYPE_F32, ly, 0)
        self.handle = h or None
        self._xa = (ctypes.c_void_p * 1)()
        self._ya = (ctypes.c_void_p * 1)()
        self._xap = ctypes.cast(self._xa, ctypes.POINTER(ctypes.c_void_p))
        self._yap = ctypes.cast(self._ya, ctypes.POINTER(ctypes.c_void_p))
        # host-path constants (pointers / views / sizes resolved once)
        self.x_ptr, self.y_ptr = dev.ptr(self.x), dev.ptr(self.y)
        self.x_pin_ptr, self.y_pin_ptr = dev.ptr(self.x_pin), dev.ptr(self.y_pin)
        self.x_np, self.y_np = self.x_pin.numpy(), self.y_pin.numpy()
        self.x_flat_np = self._x_pin_flat.numpy()
        self.x_bytes, self.y_bytes = self._x_flat.numel() * 2, self.y.numel() * 4
        self._host_graph = None  # H2D -> launch -> D2H captured once (host_graph())
        self._host_graph_failed = False

    def host_graph(self):
        """The host-input call as one CUDA graph: pinned x -> device, then the
        prepared launch storing y into the pinned output buffer (measured: 43.6
        -> 29.1 us per 4096x4096 call for H2D / launch / D2H as stream
        operations vs one graph).  Captured on first use in
        thread-local mode (other threads' CUDA calls are unaffected); None if
        capture is unavailable (the caller issues the three operations)."""
        if self._host_graph is None and not self._host_graph_failed:
            torch = dev.torch()
            try:
                side = torch.cuda.Stream()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                    st = dev.stream_ptr()
                    check(self._lib.apb_memcpy_async(self.x_ptr, self.x_pin_ptr, self.x_bytes, 0, st),
                          "apb_memcpy_async")
                    # y stored by the epilogue straight into the pinned buffer
                    # (device-addressable under UVA): no D2H node
                    self.launch(self.x_ptr, self.y_pin_ptr, st)
                self._host_graph = g
            except Exception:
                self._host_graph_failed = True
        return self._host_graph

    def launch(self, xptr=None, yptr=None, stream=None):
        xa = ya = None
        if xptr is not None:
            self._xa[0] = xptr
            xa = self._xap
        if yptr is not None:
            self._ya[0] = yptr
            ya = self._yap
        check(self._lib.apb_gemv_plan_launch(self.handle, xa, ya, dev.stream_ptr() if stream is None else stream),
              "apb_gemv_plan_launch")

    def __del__(self):
        if getattr(self, "handle", None):
            self._lib.apb_gemv_plan_destroy(self.handle)
            self.handle = None


def _host_rows(x, m: int, fp16: bool):
    """Host activation block -> (staged fp16 rows or, for fp32 activations,
    the flat scaled-pair block of apb_split_x_scaled for ldx, m_x, split)."""
    x = x.numpy() if dev.is_tensor(x) else np.asarray(x)
    if fp16 or x.dtype == np.float16:
        return x.astype(np.float16), m, 0
    return _split_scaled_np(x.astype(np.float32), _ldx(x.shape[1])), 2 * m, 2


def _quantized(prep: PreparedLayer, x2, k: int, fp16: bool):
    """The GPU quantized path for a (m, cols) activation block."""
    torch = dev.require_cuda()
    t = prep.tensor
    m = _shape_of(x2)[0]
    host = not (dev.is_tensor(x2) and x2.is_cuda)
    if host:
        # host activations: staged in this thread's pinned buffer, one async H2D,
        # the prepared launch, one D2H into pinned memory, one stream sync
        rows16, m_x, split = _host_rows(x2, m, fp16)
        plan = prep._call_plan(k, m_x, split)
        if plan.handle is not None:
            if split == 2:
                plan.x_flat_np[:] = rows16  # whole block: pairs + inverse scales
            else:
                plan.x_np[:, :t.cols] = rows16
            lib, g = plan._lib, plan.host_graph()
            if g is not None:
                g.replay()  # on the current stream
                st = dev.stream_ptr()
            else:
                st = dev.stream_ptr()
                check(lib.apb_memcpy_async(plan.x_ptr, plan.x_pin_ptr, plan.x_bytes, 0, st), "apb_memcpy_async")
                plan.launch(plan.x_ptr, plan.y_ptr, st)  # (a device call may have re-pointed the plan)
                check(lib.apb_memcpy_async(plan.y_pin_ptr, plan.y_ptr, plan.y_bytes, 1, st), "apb_memcpy_async")
            check(lib.apb_stream_sync(st), "apb_stream_sync")
            out = plan.y_np.copy()
            return out if not dev.is_tensor(x2) else torch.from_numpy(out)
    xdev, m_x, ldx, split, kind = _stage_x(x2, t.cols, fp16)
    m_out = m_x // 2 if split else m_x
    if not host:
        plan = prep._call_plan(k, m_x, split)
        if plan.handle is not None and ldx == plan.ldx:
            y = torch.empty((m_out, t.rows), dtype=torch.float32, device=xdev.device)
            plan.launch(dev.ptr(xdev), dev.ptr(y))
            return y
    y = torch.empty((m_out, t.rows), dtype=torch.float32, device=xdev.device)
    check(
        load().apb_gemv(dev.ptr(t.planes), t.n_max, t.rows, t.cols, t.padded_cols, k,
                        dev.ptr(prep.tables16[k]), dev.ptr(xdev), m_x, ldx, split, dev.ptr(y),
                        APB_DTYPE_F32, t.rows, 0, dev.stream_ptr()),
        "apb_gemv",
    )
    if kind == "numpy":
        return y.cpu().numpy()
    return y.cpu() if kind == "tensor" else y


def _count_quantized(prep: PreparedLayer, k: int, merged: bool, report: ExecutionReport | None):
    """Counters of _dequant_values (engine.py:235-245)."""
    if report is None:
        return
    rows = prep.tensor.rows
    report.table_bytes_read += rows * 64 * 2 * 2 if merged else rows * (1 << k) * 2
    report.planes_bytes_read += k * rows * prep.tensor.padded_cols // 8
    report.extra["device"] = "cuda:sm_100a"


def _shape_of(x):
    return tuple(x.shape) if hasattr(x, "shape") else np.shape(x)


# ---- public entry points ----------------------------------------------------------

def gemv(prep: PreparedLayer, x, cfg: GemvConfig, report: ExecutionReport | None = None):
    """y = dequant_k(W) @ x reading only the top cfg.bit_width bitplanes
    (engine.py:284-309).  Deterministic for identical inputs."""
    k = cfg.bit_width
    _check_bit_width(prep.layer, k)
    t = prep.tensor
    if not dev.is_tensor(x):
        x = np.asarray(x)
    shape = _shape_of(x)
    if shape[-1] != t.cols:
        raise ShapeError(f"activation length {shape[-1]} != in_features {t.cols}")
    if len(shape) != 1:
        raise ShapeError("gemv expects a 1-D activation vector")
    merged = cfg.merged()
    if merged and k != 3:
        raise ParameterError("merged-table lookups apply to 3-bit only")
    y = _quantized(prep, x[None, :] if not dev.is_tensor(x) else x.unsqueeze(0), k,
                   cfg.activations_fp16)
    _count_quantized(prep, k, merged, report)
    if report is not None:
        report.path_taken = "gemv-merged" if merged else "gemv"
    return y[0]


def gemm(prep: PreparedLayer, x, cfg: GemvConfig, report: ExecutionReport | None = None):
    """Y = X @ dequant_k(W).T for a (M, in_features) batch (engine.py:312-354).
    M <= dense_threshold: quantized small-batch kernel (decode once, reuse the
    weights across the batch); larger M: GPU dequantize (exact fp16) + an
    fp32-accurate tensor-core GEMM (hi/lo split activations)."""
    k = cfg.bit_width
    _check_bit_width(prep.layer, k)
    if not dev.is_tensor(x):
        x = np.asarray(x)
    shape = _shape_of(x)
    if len(shape) != 2:
        raise ShapeError("gemm expects a (M, in_features) matrix")
    m = shape[0]
    if m < 1:
        raise ShapeError("batch must contain at least one row")
    t = prep.tensor
    if m <= cfg.dense_threshold:
        if shape[-1] != t.cols:
            raise ShapeError(f"activation length {shape[-1]} != in_features {t.cols}")
        merged = cfg.merged()
        if merged and k != 3:
            raise ParameterError("merged-table lookups apply to 3-bit only")
        y = _quantized(prep, x, k, cfg.activations_fp16)
        _count_quantized(prep, k, merged, report)
        if report is not None:
            report.path_taken = "gemm-quantized"
        return y
    if shape[1] != t.cols:
        raise ShapeError(f"activation width {shape[1]} != in_features {t.cols}")
    torch = dev.require_cuda()
    if report is not None:
        report.path_taken = "gemm-dense"
        report.planes_bytes_read += k * t.rows * t.padded_cols // 8
        report.table_bytes_read += t.rows * (1 << k) * 2
    host = not dev.is_tensor(x)
    xd = dev.to_device(np.asarray(x)) if host else x.cuda()
    back = "numpy" if host else ("cuda" if x.is_cuda else "tensor")
    if _DENSE_IMPL == "cublas":  # the round-1 path (separate dequant + cuBLAS), kept for comparison
        y = _dense_tensor_core(torch, xd, _dequant_device(prep, k, APB_DTYPE_F16), cfg.activations_fp16)
    else:
        y = _dense_fused(torch, prep, k, xd, cfg.activations_fp16)
    if back == "numpy":
        return y.cpu().numpy()
    return y.cpu() if back == "tensor" else y


# APB_DENSE=cublas selects the round-1 dense path (GPU dequantize to an fp16
# weight tensor + cuBLAS) for A/B measurements; the default is the fused kernel.
_DENSE_IMPL = os.environ.get("APB_DENSE", "tcgen05")


def _dense_fused(torch, prep: PreparedLayer, k: int, x, x_is_fp16: bool):
    """Y = X @ dequant_k(W).T in one tcgen05 kernel (csrc/apb_dense_tc.cu): the
    top-k planes and the fp16 table are decoded straight into the MMA's shared-
    memory A operand, activations arrive by TMA, fp32 accumulation in tensor
    memory.  fp32 activations ride as scaled fp16 (hi, lo) row pairs (exact
    power-of-two row scale), summed and unscaled in the epilogue -- fp32-accurate
    like the reference's dense path (engine.py:343-354)."""
    t = prep.tensor
    m = x.shape[0]
    L = load()
    s = dev.stream_ptr()
    if x_is_fp16:
        xin, dt, mx, pairs = x.to(torch.float16).contiguous(), APB_DTYPE_F16, m, 0
    else:
        xin, dt, mx, pairs = x.to(torch.float32).contiguous(), APB_DTYPE_F32, 2 * m, 1
    xp = torch.empty((mx, t.padded_cols), dtype=torch.float16, device="cuda")
    inv = torch.empty(m, dtype=torch.float32, device="cuda")
    check(L.apb_dense_prep_x(dev.ptr(xin), dt, m, t.cols, xin.shape[1], dev.ptr(xp), t.padded_cols,
                             dev.ptr(inv), s), "apb_dense_prep_x")
    y = torch.empty((m, t.rows), dtype=torch.float32, device="cuda")
    wsb = L.apb_gemm_dense_tc_workspace(t.rows, t.padded_cols, mx)  # split-K partials (small batches)
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device="cuda")
    check(L.apb_gemm_dense_tc(dev.ptr(t.planes), t.n_max, t.rows, t.cols, t.padded_cols, k,
                              dev.ptr(prep.tables16[k]), dev.ptr(xp), mx, pairs, dev.ptr(inv), dev.ptr(y),
                              t.rows, dev.ptr(ws), wsb, s), "apb_gemm_dense_tc")
    return y


def _dense_tensor_core(torch, x, w16, x_is_fp16: bool):
    """Y = X @ W.T at fp32 accuracy on the tensor cores (the reference's dense
    path is an fp32 GEMM, engine.py:343-354).  W is exact in fp16; X is split
    into fp16 hi + lo halves after an exact power-of-two row scale (hi <= 2^15,
    no overflow; X - hi is exact in fp32 and its fp16 rounding leaves ~2^-22
    relative error; csrc/apb_dense.cu, one pass), and ONE fp16 x fp16 -> fp32
    tensor-core GEMM over [hi; lo] accumulates both products in fp32."""
    if x_is_fp16:
        return torch.mm(x.to(torch.float16), w16.T, out_dtype=torch.float32)
    x = x.to(torch.float32).contiguous()
    m, c = x.shape
    hilo = torch.empty((2 * m, c), dtype=torch.float16, device="cuda")
    inv = torch.empty((m, 1), dtype=torch.float32, device="cuda")
    check(load().apb_split_hilo(dev.ptr(x), m, c, c, dev.ptr(hilo), c, dev.ptr(inv), dev.stream_ptr()),
          "apb_split_hilo")
    yy = torch.mm(hilo, w16.T, out_dtype=torch.float32)
    return yy[:m].add_(yy[m:]).mul_(inv)


def _dequant_device(prep: PreparedLayer, k: int, dtype: int):
    torch = dev.require_cuda()
    t = prep.tensor
    w = torch.empty((t.rows, t.cols), dtype=torch.float16 if dtype == APB_DTYPE_F16 else torch.float32,
                    device="cuda")
    check(
        load().apb_dequant(dev.ptr(t.planes), t.n_max, t.rows, t.cols, t.padded_cols, 1, k,
                           dev.ptr(prep.tables16[k]), dev.ptr(w), dtype, t.cols, dev.stream_ptr()),
        "apb_dequant",
    )
    return w


def dequantize(layer, k: int):
    """Dense fp32 weights at bit-width k (engine.py:357-362), decoded on the
    GPU from the top k planes.  Accepts an AnyPrecisionLayer (host codes ->
    numpy result) or a PreparedLayer (device result)."""
    if isinstance(layer, PreparedLayer):
        _check_bit_width(layer.layer, k)
        return _dequant_device(layer, k, APB_DTYPE_F32)
    _check_bit_width(layer, k)
    prep = PreparedLayer(layer)
    w = _dequant_device(prep, k, APB_DTYPE_F32)
    return w if dev.is_tensor(layer.codes) else w.cpu().numpy()


def _merged_index_stream(prep: PreparedLayer) -> np.ndarray:
    """The 6-bit merged indices of the reference's 3-bit path in pair order
    (engine.py:249-260, a testing aid), derived from the GPU transpose."""
    t = prep.tensor
    planes = t.planes[:3].contiguous().view(dev.torch().int32)  # little-endian lane words
    words = planes.reshape(3, t.rows, t.n_tiles, LANES)
    tw = transpose_any_width(words, 3).cpu().numpy()
    out = []
    for g in range(4):
        for p in range(4):
            lo = (tw[g] >> np.uint32(8 * p)) & np.uint32(7)
            hi = (tw[g] >> np.uint32(8 * p + 4)) & np.uint32(7)
            out.append(((lo << np.uint32(3)) | hi).ravel())
    return np.stack(out)


__all__ = [
    "TRANSPOSE_OP_COUNT", "bit_transpose", "transpose_any_width", "MergedTable3",
    "build_merged_table", "GemvConfig", "ExecutionReport", "PreparedLayer", "prepare",
    "gemv", "gemm", "dequantize", "TILE_WEIGHTS",
]
