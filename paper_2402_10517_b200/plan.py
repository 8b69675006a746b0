"""Pre-bound GEMV launch plans for decode-style loops.

A ``GemvPlan`` owns device activation/output buffers for a list of prepared
layers at one bit-width and pre-marshals the C-ABI arguments, so a call is a
single ``apb_gemv_grouped`` launch (all layers in one kernel) or one
``apb_gemv`` per layer, with no allocation and no per-call validation in
Python.  ``capture()`` records the launches into a CUDA graph so a decode step
replays without any host launch overhead.
"""

from __future__ import annotations

import ctypes

from . import _device as dev
from ._lib import (
    APB_DTYPE_F16,
    APB_DTYPE_F32,
    APB_FLAG_PDL,
    check,
    int64_array,
    int_array,
    load,
    ptr_array,
)
from .errors import ParameterError


def _ldx(cols: int) -> int:
    return -(-cols // 8) * 8


class GemvPlan:
    def __init__(self, preps, k: int, m: int = 1, grouped: bool = True, x_split: bool = False,
                 y_fp16: bool = False, pdl: bool = False, shared_x: bool = False):
        torch = dev.require_cuda()
        for p in preps:
            if k not in p.tables16:
                raise ParameterError(f"bit width {k} unsupported by a layer of the plan")
        self.preps = list(preps)
        self.k = k
        self.m = m
        self.grouped = grouped
        self.x_split = 1 if x_split else 0
        self.m_x = 2 * m if x_split else m
        self.y_dtype = APB_DTYPE_F16 if y_fp16 else APB_DTYPE_F32
        # programmatic dependent launch: safe here because the plan's weights
        # are never written by the kernels that precede it in a decode loop
        self.flags = APB_FLAG_PDL if pdl else 0
        ydt = torch.float16 if y_fp16 else torch.float32
        if shared_x:  # one activation for every layer (e.g. q/k/v, gate/up)
            cols = {p.tensor.cols for p in self.preps}
            if len(cols) != 1:
                raise ParameterError("shared_x needs layers with equal in_features")
            x0 = torch.zeros((self.m_x, _ldx(cols.pop())), dtype=torch.float16, device="cuda")
            self.x = [x0] * len(self.preps)
        else:
            self.x = [torch.zeros((self.m_x, _ldx(p.tensor.cols)), dtype=torch.float16, device="cuda")
                      for p in self.preps]
        self.y = [torch.zeros((m, p.tensor.rows), dtype=ydt, device="cuda") for p in self.preps]
        ts = [p.tensor for p in self.preps]
        n = len(ts)
        self._n = n
        self._planes = ptr_array([dev.ptr(t.planes) for t in ts])
        self._nmax = int_array([t.n_max for t in ts])
        self._rows = int64_array([t.rows for t in ts])
        self._cols = int64_array([t.cols for t in ts])
        self._padded = int64_array([t.padded_cols for t in ts])
        self._lut = ptr_array([dev.ptr(p.tables16[k]) for p in self.preps])
        self._xp = ptr_array([dev.ptr(x) for x in self.x])
        self._ldx = int64_array([x.shape[1] for x in self.x])
        self._yp = ptr_array([dev.ptr(y) for y in self.y])
        self._ldy = int64_array([t.rows for t in ts])
        self._lib = load()

    def algorithmic_bytes(self) -> int:
        """R*C*k/8 (unpadded top-k planes) + R*2^k*2 (fp16
        LUT) + M*C*2 (fp16 x) + M*R*2 (fp16 y), summed over the layers."""
        k, m = self.k, self.m
        tot = 0
        for p in self.preps:
            r, c = p.tensor.rows, p.tensor.cols
            tot += r * c * k // 8 + r * (1 << k) * 2 + m * c * 2 + m * r * 2
        return tot

    def run(self):
        s = dev.stream_ptr()
        L = self._lib
        if self.grouped:
            check(
                L.apb_gemv_grouped(self._n, ctypes.cast(self._planes, ctypes.POINTER(ctypes.c_void_p)),
                                   self._nmax, self._rows, self._cols, self._padded, self.k,
                                   ctypes.cast(self._lut, ctypes.POINTER(ctypes.c_void_p)),
                                   ctypes.cast(self._xp, ctypes.POINTER(ctypes.c_void_p)),
                                   self.m_x, self._ldx, self.x_split,
                                   ctypes.cast(self._yp, ctypes.POINTER(ctypes.c_void_p)),
                                   self.y_dtype, self._ldy, self.flags, s),
                "apb_gemv_grouped",
            )
            return
        for i in range(self._n):
            check(
                L.apb_gemv(self._planes[i], self._nmax[i], self._rows[i], self._cols[i],
                           self._padded[i], self.k, self._lut[i], self._xp[i], self.m_x,
                           self._ldx[i], self.x_split, self._yp[i], self.y_dtype, self._ldy[i],
                           self.flags, s),
                "apb_gemv",
            )

    def capture(self, repeats: int = 1):
        """Record ``repeats`` x run() into a CUDA graph (call run() once first)."""
        torch = dev.require_cuda()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(repeats):
                self.run()
        return g
