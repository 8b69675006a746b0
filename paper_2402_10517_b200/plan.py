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
    APB_FLAG_GLU,
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
                 y_fp16: bool = False, pdl: bool = False, shared_x: bool = False, glu: bool = False,
                 norm=None):
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
        # glu: every layer's rows are interleaved (gate_i, up_i); y = silu(gate) * up
        # with rows / 2 entries (the MLP's SiLU fused into the GEMV epilogue)
        if glu:
            if not grouped or any(p.tensor.rows % 2 for p in self.preps):
                raise ParameterError("glu needs a grouped plan over layers with an even row count")
            self.flags |= APB_FLAG_GLU
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
        # norm: None, or ("producer", resid f32, norm_w f16, partials f32) / ("consumer",
        # partials f32, norm_size, eps) -- RMSNorm folded into the epilogue
        # (apb_gemv_grouped_norm)
        self._norm = None
        if norm is not None:
            from ._lib import NormEpilogue

            # apb_gemv_grouped_norm has no hi/lo activation pairs: its m_x rows are
            # batch rows, so a split plan would write 2m output rows into y [m][R]
            if x_split:
                raise ParameterError("a norm epilogue cannot be combined with x_split activations")

            if norm[0] == "producer":
                _, resid, w, part = norm
                self._norm = NormEpilogue(1, dev.ptr(resid), dev.ptr(w), dev.ptr(part), part.numel(), 0, 0.0)
            elif norm[0] == "consumer":
                _, part, size, eps = norm
                self._norm = NormEpilogue(2, None, None, dev.ptr(part), part.numel(), int(size), float(eps))
            else:
                raise ParameterError(f"unknown norm epilogue {norm[0]!r}")
            self._norm_keep = norm  # the buffers must outlive the plan
        out_rows = [p.tensor.rows // 2 if glu else p.tensor.rows for p in self.preps]
        self.y = [torch.zeros((m, r), dtype=ydt, device="cuda") for r in out_rows]
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
        self._ldy = int64_array(out_rows)
        self._lib = load()

    def rebind(self, x_list, y_list):
        """Point the plan at caller-owned device activation / output buffers
        (same shapes and dtypes as the ones it allocated)."""
        if len(x_list) != len(self.x) or len(y_list) != len(self.y):
            raise ParameterError("rebind needs one x and one y per layer")
        for old, new in list(zip(self.x, x_list)) + list(zip(self.y, y_list)):
            if tuple(old.shape) != tuple(new.shape) or old.dtype != new.dtype:
                raise ParameterError("rebind buffers must match the plan's shapes and dtypes")
        # x on the device; y on the device or in pinned host memory (UVA: the
        # epilogue stores straight into it over PCIe, StepPlan zero_copy_y)
        if not all(x.is_cuda for x in x_list) or not all(y.is_cuda or y.is_pinned() for y in y_list):
            raise ParameterError("rebind: x must be device tensors, y device or pinned host tensors")
        self.x, self.y = list(x_list), list(y_list)
        self._xp = ptr_array([dev.ptr(x) for x in self.x])
        self._yp = ptr_array([dev.ptr(y) for y in self.y])

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
        if self._norm is not None:
            P = lambda a: ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))  # noqa: E731
            check(L.apb_gemv_grouped_norm(self._n, P(self._planes), self._nmax, self._rows, self._cols,
                                          self._padded, self.k, P(self._lut), P(self._xp), self.m_x, self._ldx,
                                          P(self._yp), self.y_dtype, self._ldy, ctypes.byref(self._norm),
                                          self.flags, s), "apb_gemv_grouped_norm")
            return
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


class StepPlan:
    """A decode step: a fixed sequence of ``GemvPlan`` launches (e.g. the
    q/k/v | o | gate/up | down groups of a decoder block at some bit-widths)
    driven end to end from HOST memory.

    All distinct activation buffers of the step live in one contiguous device
    block mirrored by one pinned host block, and all outputs likewise, so a
    step is: one H2D copy of every input, the launches (replayed from a CUDA
    graph after ``capture()``), one D2H copy of every output, one stream
    synchronisation.  ``x_host`` / ``y_host`` are the pinned views the caller
    fills / reads (one per distinct activation / per output, in plan order).

    zero_copy_y: the GEMV epilogues store the outputs straight into the pinned
    host block (a pinned allocation is device-addressable under UVA), so the
    D2H copy disappears from the end of the step; the same bytes cross PCIe
    as posted writes overlapped with the remaining launches.
    """

    def __init__(self, plans, zero_copy_y: bool = False):
        torch = dev.require_cuda()
        self.plans = list(plans)
        xs, seen = [], {}
        for p in self.plans:
            for x in p.x:
                if x.data_ptr() not in seen:
                    seen[x.data_ptr()] = len(xs)
                    xs.append(x)
        ys = [y for p in self.plans for y in p.y]
        n_x = sum(x.numel() for x in xs)
        self._xd = torch.empty(n_x, dtype=torch.float16, device="cuda")
        self._xh = torch.empty(n_x, dtype=torch.float16).pin_memory()
        ybytes = sum(y.numel() * y.element_size() for y in ys)
        self._yd = torch.empty(ybytes, dtype=torch.uint8, device="cuda")
        self._yh = torch.empty(ybytes, dtype=torch.uint8).pin_memory()
        # carve views, then rebind every plan onto them
        xviews, xhost, off = [], [], 0
        for x in xs:
            n = x.numel()
            xviews.append(self._xd[off:off + n].view(x.shape))
            xhost.append(self._xh[off:off + n].view(x.shape))
            off += n
        yviews, yhost, off = [], [], 0
        for y in ys:
            nb = y.numel() * y.element_size()
            yviews.append(self._yd[off:off + nb].view(y.dtype).view(y.shape))
            yhost.append(self._yh[off:off + nb].view(y.dtype).view(y.shape))
            off += nb
        self.zero_copy_y = zero_copy_y
        if zero_copy_y:
            yviews = yhost
        yi = 0
        for p in self.plans:
            p.rebind([xviews[seen[x.data_ptr()]] for x in p.x], yviews[yi:yi + len(p.y)])
            yi += len(p.y)
        self.x_host, self.y_host = xhost, yhost
        self.h2d_bytes = n_x * 2
        self.d2h_bytes = ybytes
        self._graph = None
        self._graph_copies = False

    def launch(self):
        for p in self.plans:
            p.run()

    def capture(self, host_copies: bool = True):
        """Record the step into a CUDA graph (run ``launch()`` once first).
        host_copies: the pinned H2D copy of the inputs and the D2H copy of the
        outputs are graph nodes too, so ``run_host()`` is one graph launch and
        one synchronisation (the copies still run every step)."""
        torch = dev.require_cuda()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            if host_copies:
                self._xd.copy_(self._xh, non_blocking=True)
            self.launch()
            if host_copies and not self.zero_copy_y:
                self._yh.copy_(self._yd, non_blocking=True)
        self._graph, self._graph_copies = g, host_copies
        return g

    def run_host(self):
        """x_host -> device, the step's launches, device -> y_host; returns y_host."""
        torch = dev.require_cuda()
        if self._graph is not None and self._graph_copies:
            self._graph.replay()
        else:
            self._xd.copy_(self._xh, non_blocking=True)
            if self._graph is not None:
                self._graph.replay()
            else:
                self.launch()
            if not self.zero_copy_y:
                self._yh.copy_(self._yd, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.y_host
