"""ctypes binding of the C ABI (include/anyprec_b200.h -> libanyprec_b200.so).

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``).
There is no fallback: if the library is missing or no CUDA device is present
the calls raise, they never route to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    CodeRangeError,
    DeviceError,
    LayoutError,
    ParameterError,
    ShapeError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
# APB_LIB_PATH overrides the library (tuning / instrumented builds only)
LIB_PATH = os.environ.get("APB_LIB_PATH") or os.path.join(_HERE, "libanyprec_b200.so")

APB_OK = 0
APB_ERR_SHAPE = 1
APB_ERR_PARAM = 2
APB_ERR_LAYOUT = 3
APB_ERR_CODE_RANGE = 4
APB_ERR_CUDA = 5
APB_ERR_NCCL = 6
APB_DTYPE_F32 = 0
APB_DTYPE_F16 = 1
APB_FLAG_PDL = 1
APB_FLAG_GLU = 2


class NormEpilogue(ctypes.Structure):
    """apb_norm_epilogue (include/anyprec_b200.h)."""

    _fields_ = [("mode", ctypes.c_int), ("resid", ctypes.c_void_p), ("norm_w", ctypes.c_void_p),
                ("partials", ctypes.c_void_p), ("n_partials", ctypes.c_int), ("norm_size", ctypes.c_int),
                ("eps", ctypes.c_float)]

# Every symbol declared in include/anyprec_b200.h, with its ctypes signature.
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_PP = ctypes.POINTER(ctypes.c_void_p)
_PI = ctypes.POINTER(ctypes.c_int)
_PI64 = ctypes.POINTER(ctypes.c_int64)
SIGNATURES = {
    "apb_version": ([], _I),
    "apb_status_string": ([_I], ctypes.c_char_p),
    "apb_pad_columns": ([_I64], _I64),
    "apb_pack": ([_P, _I64, _I64, _I64, _I, _I, _P, _P, _P], _I),
    "apb_permute": ([_P, _P, _I, _I64, _I64, _I, _P], _I),
    "apb_unpack": ([_P, _I, _I64, _I64, _I64, _I, _I, _P, _I64, _P], _I),
    "apb_transpose_words": ([_P, _I, _I64, _P, _P], _I),
    "apb_gemv": ([_P, _I, _I64, _I64, _I64, _I, _P, _P, _I, _I64, _I, _P, _I, _I64, _I, _P], _I),
    "apb_gemv_grouped": (
        [_I, _PP, _PI, _PI64, _PI64, _PI64, _I, _PP, _PP, _I, _PI64, _I, _PP, _I, _PI64, _I, _P],
        _I,
    ),
    "apb_dequant": ([_P, _I, _I64, _I64, _I64, _I, _I, _P, _P, _I, _I64, _P], _I),
    "apb_split_x": ([_P, _I, _I64, _I64, _P, _I64, _I, _P], _I),
    "apb_split_x_scaled": ([_P, _I, _I64, _I64, _P, _I64, _P], _I),
    "apb_rms_residual": ([_P, _P, _P, _P, _I64, ctypes.c_float, _P], _I),
    "apb_rope_cache": ([_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I64, _P], _I),
    "apb_silu_mul": ([_P, _P, _P, _I64, _P], _I),
    "apb_embed_rms": ([_P, _P, _I64, _P, _P, _P, ctypes.c_float, _P], _I),
    "apb_argmax_f16": ([_P, _I64, _P, _P], _I),
    "apb_memcpy_async": ([_P, _P, _I64, _I, _P], _I),
    "apb_stream_sync": ([_P], _I),
    "apb_gemm_small": ([_P, _I, _I64, _I64, _I64, _I, _P, _I, _P, _I64, _P, _I, _I64, _P], _I),
    "apb_gemv_allgather": (
        [_P, _I, _I64, _I64, _I64, _I, _P, _P, _I, _I64, _I, _I, _PP, _I64, _I, _I64, _PP, _I, _P], _I,
    ),
    "apb_gemv_plan_create": (
        [_I, _PP, _PI, _PI64, _PI64, _PI64, _I, _PP, _PP, _I, _PI64, _I, _PP, _I, _PI64, _I], _P,
    ),
    "apb_gemv_plan_launch": ([_P, _PP, _PP, _P], _I),
    "apb_gemv_plan_destroy": ([_P], None),
    "apb_gemv_grouped_norm": (
        [_I, _PP, _PI, _PI64, _PI64, _PI64, _I, _PP, _PP, _I, _PI64, _PP, _I, _PI64, _P, _I, _P],
        _I,
    ),
    "apb_gemv_grouped_peers": (
        [_I, _PP, _PI, _PI64, _PI64, _PI64, _I, _PP, _PP, _I, _PI64, _I, _PP, _I, _PI64, _I, _PP, _PP, _I, _P],
        _I,
    ),
    "apb_peer_wait": ([_P, _P, ctypes.c_uint32, _P, ctypes.c_longlong, _P], _I),
    "apb_peer_alloc": ([_I64, _P, _P], _I),
    "apb_peer_open": ([_P, _P], _I),
    "apb_peer_close": ([_P], _I),
    "apb_peer_free": ([_P], _I),
    "apb_peer_handle_bytes": ([], _I),
    "apb_split_hilo": ([_P, _I64, _I64, _I64, _P, _I64, _P, _P], _I),
    "apb_dense_prep_x": ([_P, _I, _I64, _I64, _I64, _P, _I64, _P, _P], _I),
    "apb_gemm_dense_tc": ([_P, _I, _I64, _I64, _I64, _I, _P, _P, _I64, _I, _P, _P, _I64, _P, _I64, _P], _I),
    "apb_gemm_dense_tc_workspace": ([_I64, _I64, _I64], _I64),
    "apb_quant_workspace": ([_I, _I, _I, _I], _I64),
    "apb_quant_build": ([_P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _I64, _P], _I),
    "apb_quant_continue": ([_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _I64, _P], _I),
    "apb_quant_upscale": ([_P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _I64, _P], _I),
    "apb_quant_upscale_general": ([_P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P], _I),
    "apb_quant_split": ([_P, _P, _P, _I, _I, _I, _P, _P, _P, _I64, _P], _I),
    "apb_quant_cluster_workspace": ([_I, _I, _I], _I64),
    "apb_quant_cluster": ([_P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _I64, _P], _I),
    "apb_quant_sse_levels": ([_P, _P, _P, _I, _P, _I, _I, _I, _P, _P], _I),
    "apb_attention_decode_workspace": ([_I, _I, _I64], _I64),
    "apb_attention_decode": ([_P, _P, _P, _P, _P, _P, _P, _I, _I, _I64, _I, ctypes.c_float, _P, _I64, _P, _P, _P,
                              _P], _I),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load the in-tree C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                    "there is no CPU fallback"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (argtypes, restype) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = restype
            _lib = lib
    return _lib


_STATUS_EXC = {
    APB_ERR_SHAPE: ShapeError,
    APB_ERR_PARAM: ParameterError,
    APB_ERR_LAYOUT: LayoutError,
    APB_ERR_CODE_RANGE: CodeRangeError,
    APB_ERR_CUDA: DeviceError,
    APB_ERR_NCCL: DeviceError,
}


def check(rc: int, what: str) -> None:
    if rc == APB_OK:
        return
    exc = _STATUS_EXC.get(rc, DeviceError)
    msg = load().apb_status_string(rc).decode()
    raise exc(f"{what}: {msg} (status {rc})")


def int64_array(vals):
    return (ctypes.c_int64 * len(vals))(*vals)


def int_array(vals):
    return (ctypes.c_int * len(vals))(*vals)


def ptr_array(vals):
    return (ctypes.c_void_p * len(vals))(*vals)
