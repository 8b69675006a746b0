"""Any-precision quantizer on the GPU.

Same entry point, argument meaning, validation order and messages as the
reference's ``build_any_precision`` (quantizer.py:370-435, with
``_coerce_sensitivity`` :195-212): every output channel is clustered into
2^n_min groups by exact sensitivity-weighted 1-D k-means (dynamic programming,
clustering.py:89-197), then each bit up to n_max splits every cluster by exact
weighted 2-means (clustering.py:252-302).  The result is bit-identical to the
reference: same codes, same fp16 tables, same float64 per-channel SSE.

B200 path: the stable per-row argsort runs on the device (``torch.sort(...,
stable=True)`` -- a library primitive, like cuBLAS elsewhere), everything else
is csrc/apb_quant.cu through the C-ABI (``apb_quant_build``): one CTA per
channel for the DP and for every bit level.  There is no CPU fallback.
"""

from __future__ import annotations

import logging

import numpy as np

from . import _device as dev
from .errors import ParameterError, ShapeError
from .layer import MAX_BITS, MIN_BITS, AnyPrecisionLayer

log = logging.getLogger(__name__)

# workspace budget per launch block (the DP keeps (2^n_min - 2) x n argmin rows
# plus ~7 float64 rows per channel)
_WORKSPACE_BUDGET = 4 << 30


def _to_device_f64(torch, a):
    if dev.is_tensor(a):
        return a.to(device="cuda", dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


def _coerce_sensitivity(torch, w, sens):
    """quantizer.py:195-212 on the device: finite weights, sensitivity shape,
    finite and non-negative values, zero-sum rows -> uniform (logged)."""
    if not bool(torch.isfinite(w).all()):
        raise ParameterError("weights must be finite")
    if sens is None:
        return torch.ones_like(w)
    values = sens if dev.is_tensor(sens) or isinstance(sens, np.ndarray) else getattr(sens, "values", sens)
    s = _to_device_f64(torch, values)
    if tuple(s.shape) != tuple(w.shape):
        raise ShapeError(f"sensitivity shape {tuple(s.shape)} != weights shape {tuple(w.shape)}")
    if not bool(torch.isfinite(s).all()):
        raise ParameterError("sensitivities must be finite")
    if bool((s < 0).any()):
        raise ParameterError("sensitivity values must be non-negative")
    dead = s.sum(dim=1) <= 0
    if bool(dead.any()):
        idx = torch.nonzero(dead).view(-1)
        log.warning("zero-sensitivity channel(s) %s: falling back to uniform weights", idx[:8].tolist())
        s = s.clone()
        s[dead] = 1.0
    return s.contiguous()


def build_any_precision(weights, sens, n_min: int, n_max: int, *, record_levels: bool = False,
                        row_block: int | None = None, threads: int = 1, as_numpy: bool = True):
    """Seed at n_min, upscale one bit at a time to n_max (quantizer.py:370-435).

    ``weights`` / ``sens``: (out_channels, in_features) numpy arrays or torch
    tensors (any float dtype; computed in float64 like the reference).  ``sens``
    may be None (uniform), an array or a SensitivityMap-like object with
    ``.values``.  ``row_block`` bounds the channels per device pass (default:
    as many as a 4 GB workspace holds); ``threads`` is accepted for signature
    compatibility.  Returns an ``AnyPrecisionLayer`` with host numpy fields
    (``as_numpy=False``: device tensors), including ``channel_sse`` and, with
    ``record_levels``, ``level_codes``.
    """
    torch = dev.require_cuda()
    from ._lib import check, load

    w = _to_device_f64(torch, weights)
    if w.dim() != 2 or w.numel() == 0:
        raise ShapeError("weight matrix must be a non-empty 2-D array")
    if not MIN_BITS <= n_min <= n_max <= MAX_BITS:
        raise ParameterError(f"bit range [{n_min}, {n_max}] outside [{MIN_BITS}, {MAX_BITS}]")
    s = _coerce_sensitivity(torch, w.contiguous(), sens)
    w = w.contiguous()
    rows, n = w.shape
    if n >= 1 << 31:
        raise ShapeError("in_features too large")

    lib = load()
    per_row = lib.apb_quant_workspace(1, n, n_min, n_max)
    block = max(1, min(rows, _WORKSPACE_BUDGET // max(per_row, 1)))
    if row_block is not None:
        block = max(1, min(block, int(row_block)))
    levels = n_max - n_min + 1
    codes = torch.empty(rows, n, dtype=torch.uint8, device="cuda")
    tables = {k: torch.empty(rows, 1 << k, dtype=torch.float16, device="cuda") for k in range(n_min, n_max + 1)}
    sse = torch.empty(levels, rows, dtype=torch.float64, device="cuda")
    lvl = torch.empty(levels, rows, n, dtype=torch.uint8, device="cuda") if record_levels else None
    ws = torch.empty(lib.apb_quant_workspace(block, n, n_min, n_max), dtype=torch.uint8, device="cuda")
    st, P = dev.stream_ptr(), dev.ptr
    for lo in range(0, rows, block):
        hi = min(rows, lo + block)
        nb = hi - lo
        wb, sb = w[lo:hi], s[lo:hi]
        # stable ascending argsort; -0.0 and +0.0 compare equal as in numpy
        order = torch.sort(wb + 0.0, dim=1, stable=True).indices.contiguous()
        tb = torch.empty(sum(nb << k for k in range(n_min, n_max + 1)), dtype=torch.float16, device="cuda")
        sseb = torch.empty(levels, nb, dtype=torch.float64, device="cuda")
        lvlb = torch.empty(levels, nb, n, dtype=torch.uint8, device="cuda") if record_levels else None
        check(lib.apb_quant_build(P(wb), P(sb), P(order), nb, n, n_min, n_max, P(codes[lo:hi]), P(tb), P(sseb),
                                  P(lvlb) if lvlb is not None else None, P(ws), ws.numel(), st),
              "apb_quant_build")
        off = 0
        for k in range(n_min, n_max + 1):
            tables[k][lo:hi] = tb[off:off + (nb << k)].view(nb, 1 << k)
            off += nb << k
        sse[:, lo:hi] = sseb
        if record_levels:
            lvl[:, lo:hi] = lvlb
    conv = (lambda t: t.cpu().numpy()) if as_numpy else (lambda t: t)
    layer = AnyPrecisionLayer(
        n_min=n_min, n_max=n_max, codes=conv(codes),
        centroid_tables={k: conv(t) for k, t in tables.items()},
        shape=(rows, n),
        channel_sse={k: conv(sse[k - n_min]) for k in range(n_min, n_max + 1)},
    )
    if record_levels:
        layer.level_codes = {k: conv(lvl[k - n_min]) for k in range(n_min, n_max + 1)}
    return layer


def continue_upscale(weights, sens, layer, new_n_max: int, *, row_block: int | None = None,
                     as_numpy: bool = True):
    """Extend an existing layer to a higher parent bit-width (quantizer.py:438-512):
    the stored n_max-bit codes define the clusters that keep splitting (codes
    must be value-contiguous in each row's sorted order, else ParameterError),
    the fp16 table of the old n_max is the parent of the first split, and the
    error record of the existing levels is recomputed against the new codes."""
    torch = dev.require_cuda()
    from ._lib import check, load

    w = _to_device_f64(torch, weights).contiguous()
    if tuple(w.shape) != tuple(layer.shape):
        raise ShapeError(f"weights shape {tuple(w.shape)} != layer shape {tuple(layer.shape)}")
    if not layer.n_max < new_n_max <= MAX_BITS:
        raise ParameterError(f"new parent bit-width {new_n_max} must be in ({layer.n_max}, {MAX_BITS}]")
    s = _coerce_sensitivity(torch, w, sens)
    rows, n = w.shape
    k0 = layer.n_max
    codes_in = layer.codes if dev.is_tensor(layer.codes) else torch.from_numpy(np.ascontiguousarray(layer.codes))
    codes_in = codes_in.to(device="cuda", dtype=torch.uint8).contiguous()
    t0 = layer.centroid_tables[k0]
    t0 = (t0 if dev.is_tensor(t0) else torch.from_numpy(np.ascontiguousarray(t0, dtype=np.float16)))
    t0 = t0.to(device="cuda", dtype=torch.float16).contiguous()

    lib = load()
    per_row = lib.apb_quant_workspace(1, n, 2, new_n_max)
    block = max(1, min(rows, _WORKSPACE_BUDGET // max(per_row, 1)))
    if row_block is not None:
        block = max(1, min(block, int(row_block)))
    new_levels = new_n_max - k0
    codes = torch.empty(rows, n, dtype=torch.uint8, device="cuda")
    tables = {k: torch.empty(rows, 1 << k, dtype=torch.float16, device="cuda") for k in range(k0 + 1, new_n_max + 1)}
    sse = torch.empty(new_levels, rows, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.apb_quant_workspace(block, n, 2, new_n_max), dtype=torch.uint8, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    st, P = dev.stream_ptr(), dev.ptr
    for lo in range(0, rows, block):
        hi = min(rows, lo + block)
        nb = hi - lo
        order = torch.sort(w[lo:hi] + 0.0, dim=1, stable=True).indices.contiguous()
        tb = torch.empty(sum(nb << k for k in range(k0 + 1, new_n_max + 1)), dtype=torch.float16, device="cuda")
        sseb = torch.empty(new_levels, nb, dtype=torch.float64, device="cuda")
        check(lib.apb_quant_continue(P(w[lo:hi]), P(s[lo:hi]), P(order), P(codes_in[lo:hi]), P(t0[lo:hi]), nb, n,
                                     k0, new_n_max, P(codes[lo:hi]), P(tb), P(sseb), P(bad), P(ws), ws.numel(),
                                     st), "apb_quant_continue")
        if int(bad.item()):
            raise ParameterError("stored codes are not value-contiguous; re-quantize from weights instead")
        off = 0
        for k in range(k0 + 1, new_n_max + 1):
            tables[k][lo:hi] = tb[off:off + (nb << k)].view(nb, 1 << k)
            off += nb << k
        sse[:, lo:hi] = sseb
    # the existing levels: old tables, error recomputed against the new codes
    all_tables, all_sse = {}, {}
    for k in range(layer.n_min, k0 + 1):
        tk = layer.centroid_tables[k]
        tk = (tk if dev.is_tensor(tk) else torch.from_numpy(np.ascontiguousarray(tk, dtype=np.float16)))
        tk = tk.to(device="cuda", dtype=torch.float16).contiguous()
        out = torch.empty(rows, dtype=torch.float64, device="cuda")
        check(lib.apb_quant_sse_levels(P(w), P(s), P(codes), new_n_max - k, P(tk), k, rows, n, P(out), st),
              "apb_quant_sse_levels")
        all_tables[k], all_sse[k] = tk, out
    for k in range(k0 + 1, new_n_max + 1):
        all_tables[k], all_sse[k] = tables[k], sse[k - k0 - 1]
    conv = (lambda t: t.cpu().numpy()) if as_numpy else (lambda t: t)
    return AnyPrecisionLayer(n_min=layer.n_min, n_max=new_n_max, codes=conv(codes),
                             centroid_tables={k: conv(t) for k, t in all_tables.items()}, shape=(rows, n),
                             channel_sse={k: conv(t) for k, t in all_sse.items()})


# ---- the rest of the reference quantizer module (quantizer.py:31-72, 122-307) ----

class SensitivityMap:
    """Importance of every weight (float64, the weight matrix's shape, >= 0),
    as the reference's quantizer.py:31-47 defines it; ``fallback`` marks maps
    that were synthesised from degenerate calibration data."""

    def __init__(self, values, fallback: bool = False):
        v = np.asarray(values, dtype=np.float64)
        _require(v.ndim == 2, ShapeError, "sensitivity map must be 2-D")
        _require(not np.any(v < 0), ParameterError, "sensitivity values must be non-negative")
        self.values, self.fallback = v, fallback

    @classmethod
    def uniform(cls, shape, fallback: bool = False) -> "SensitivityMap":
        return cls(np.full(shape, 1.0), fallback=fallback)


def _require(ok: bool, exc, msg: str) -> None:
    """Raise the reference's exception class / message when a check fails."""
    if not ok:
        raise exc(msg)


class ChannelQuantization:
    """A channel quantized at one bit-width: integer codes and its 2^k sorted
    float64 centroids (data contract of quantizer.py:50-72)."""

    def __init__(self, bit_width: int, codes, centroids):
        k = bit_width
        c = np.asarray(codes)
        cent = np.asarray(centroids, dtype=np.float64)
        _require(MIN_BITS <= k <= MAX_BITS, ParameterError, f"bit width {k} outside [{MIN_BITS}, {MAX_BITS}]")
        _require(cent.shape == (1 << k,), ShapeError,
                 f"expected {1 << k} centroids for {k}-bit channel, got {cent.shape}")
        _require(c.size == 0 or (c.min() >= 0 and c.max() < (1 << k)), ParameterError,
                 "codes out of range for bit width")
        self.bit_width, self.codes, self.centroids = k, c, cent

    def dequantized(self) -> np.ndarray:
        return np.take(self.centroids, self.codes)


class KMeans1DResult(tuple):
    """(centroids (k,) float64, assignments (n,) int64, padded bool) -- the
    reference's NamedTuple (clustering.py:25-28)."""

    def __new__(cls, centroids, assignments, padded):
        return super().__new__(cls, (centroids, assignments, padded))

    centroids = property(lambda self: self[0])
    assignments = property(lambda self: self[1])
    padded = property(lambda self: self[2])


def estimate_sensitivity_diag(gradient_samples, shape=None) -> SensitivityMap:
    """Diagonal-Fisher importance: per weight, the mean over the calibration
    samples of the squared gradient (behaviour of quantizer.py:160-187).  The
    squares are accumulated sample after sample in float64 and divided once,
    the reference's order, so the map matches it bit for bit.  With no samples
    the map is uniform over ``shape``; rows whose mean is zero everywhere
    become uniform rows; either case sets ``fallback``."""
    grads = [np.asarray(g, dtype=np.float64) for g in gradient_samples]
    if len(grads) == 0:
        _require(shape is not None, ParameterError, "empty sample list needs an explicit shape for the fallback")
        log.warning("estimate_sensitivity_diag: no gradient samples, uniform importance")
        return SensitivityMap.uniform(shape, fallback=True)
    first = grads[0].shape
    _require(all(g.shape == first for g in grads), ShapeError, "gradient samples must share one shape")
    fisher = np.zeros(first, dtype=np.float64)
    for g in grads:
        np.add(fisher, np.square(g), out=fisher)
    fisher /= len(grads)
    zero_rows = np.flatnonzero(~(fisher > 0).any(axis=1))
    if zero_rows.size == 0:
        return SensitivityMap(fisher)
    log.warning("estimate_sensitivity_diag: %d channel(s) without gradient signal -> uniform", zero_rows.size)
    fisher[zero_rows] = 1.0
    return SensitivityMap(fisher, fallback=True)


def _cluster_device(torch, w, s, k: int):
    """apb_quant_cluster over the rows of (w, s): bounds, float64 means, codes."""
    from ._lib import check, load

    lib = load()
    rows, n = w.shape
    if k > 4096:
        raise ParameterError(f"cluster count {k} above the device limit 4096")
    order = torch.sort(w + 0.0, dim=1, stable=True).indices.contiguous()
    bounds = torch.empty(rows, k + 1, dtype=torch.int32, device="cuda")
    means = torch.empty(rows, k, dtype=torch.float64, device="cuda")
    codes = torch.empty(rows, n, dtype=torch.int32, device="cuda")
    ws = torch.empty(lib.apb_quant_cluster_workspace(rows, n, k), dtype=torch.uint8, device="cuda")
    P = dev.ptr
    check(lib.apb_quant_cluster(P(w), P(s), P(order), rows, n, k, P(bounds), P(means), P(codes), P(ws),
                                ws.numel(), dev.stream_ptr()), "apb_quant_cluster")
    return bounds, means, codes


def kmeans_1d_weighted(values, weights, k: int) -> KMeans1DResult:
    """Globally optimal weighted k-means of a 1-D array (quantizer.py:122-157) on
    the GPU: same validation, same partition (smallest leading cluster on ties),
    empty clusters duplicate the largest real centroid."""
    values = np.asarray(values, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    if values.ndim != 1 or values.size == 0:
        raise ShapeError("values must be a non-empty 1-D array")
    if weights.shape != values.shape:
        raise ShapeError(f"weights shape {weights.shape} != values shape {values.shape}")
    if k < 1:
        raise ParameterError(f"k must be >= 1, got {k}")
    if np.any(weights < 0):
        raise ParameterError("weights must be non-negative")
    if weights.sum() <= 0:
        raise ParameterError("total weight must be positive")
    torch = dev.require_cuda()
    w = torch.from_numpy(values[None, :].copy()).cuda()
    s = torch.from_numpy(weights[None, :].copy()).cuda()
    _, means, codes = _cluster_device(torch, w, s, k)
    distinct = int(np.count_nonzero(np.diff(np.sort(values)) > 0)) + 1
    return KMeans1DResult(means[0].cpu().numpy(), codes[0].cpu().numpy().astype(np.int64), bool(distinct < k))


def quantize_seed(weights, sens, n1: int, *, row_block: int = 64) -> list:
    """Every output channel quantized to n1 bits independently by exact weighted
    k-means with k = 2^n1 (quantizer.py:281-307), on the GPU."""
    weights = np.asarray(weights, dtype=np.float64) if not dev.is_tensor(weights) else weights
    if len(weights.shape) != 2:
        raise ShapeError("weight matrix must be 2-D")
    if not MIN_BITS <= n1 <= MAX_BITS:
        raise ParameterError(f"seed bit-width {n1} outside [{MIN_BITS}, {MAX_BITS}]")
    torch = dev.require_cuda()
    w = _to_device_f64(torch, weights).contiguous()
    s = _coerce_sensitivity(torch, w, sens)
    _, means, codes = _cluster_device(torch, w, s, 1 << n1)
    means, codes = means.cpu().numpy(), codes.cpu().numpy().astype(np.int64)
    return [ChannelQuantization(n1, codes[r], means[r]) for r in range(w.shape[0])]


def upscale(cq: ChannelQuantization, row, sens) -> ChannelQuantization:
    """Split every cluster of one channel into two (quantizer.py:310-367) on the
    GPU: value-contiguous codes go through the split kernels with the channel's
    float64 centroids as parents; any other code assignment through the
    per-cluster 2-means kernel (the reference's _upscale_general semantics:
    zero-weight clusters weighted uniformly, single-valued clusters kept whole,
    empty clusters duplicating the parent)."""
    from ._lib import check, load

    row = np.asarray(row, dtype=np.float64)
    sens = np.asarray(sens, dtype=np.float64)
    if row.shape != cq.codes.shape or sens.shape != row.shape:
        raise ShapeError("row/sensitivity length does not match the channel codes")
    if cq.bit_width >= MAX_BITS:
        raise ParameterError(f"cannot upscale past {MAX_BITS} bits")
    if not np.all(np.isfinite(row)):
        raise ParameterError("weights must be finite")
    if not np.all(np.isfinite(sens)):
        raise ParameterError("sensitivities must be finite")
    if np.any(sens < 0):
        raise ParameterError("sensitivity values must be non-negative")
    torch = dev.require_cuda()
    lib, P, st = load(), dev.ptr, dev.stream_ptr()
    n, k0 = row.size, cq.bit_width
    w = torch.from_numpy(row[None, :].copy()).cuda()
    s = torch.from_numpy(sens[None, :].copy()).cuda()
    codes_in = torch.from_numpy(np.asarray(cq.codes).astype(np.uint8)[None, :].copy()).cuda()
    parents = torch.from_numpy(np.ascontiguousarray(cq.centroids, dtype=np.float64)[None, :]).cuda()
    codes = torch.empty(1, n, dtype=torch.uint8, device="cuda")
    means = torch.empty(1, 2 << k0, dtype=torch.float64, device="cuda")
    order = torch.sort(w + 0.0, dim=1, stable=True).indices.contiguous()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.empty(lib.apb_quant_workspace(1, n, 2, k0 + 1), dtype=torch.uint8, device="cuda")
    check(lib.apb_quant_upscale(P(w), P(s), P(order), P(codes_in), P(parents), 1, n, k0, P(codes), P(means),
                                P(bad), P(ws), ws.numel(), st), "apb_quant_upscale")
    if int(bad.item()):  # codes are not value-contiguous: per-cluster 2-means
        by_code = torch.sort(codes_in.gather(1, order).to(torch.int32), dim=1, stable=True).indices
        gorder = order.gather(1, by_code).contiguous()
        scratch = torch.empty(2 * n + 3 * (n + (1 << k0) + 1), dtype=torch.float64, device="cuda")
        check(lib.apb_quant_upscale_general(P(w), P(s), P(gorder), P(codes_in), P(parents), 1, n, k0, P(codes),
                                            P(means), P(scratch), st), "apb_quant_upscale_general")
    return ChannelQuantization(k0 + 1, codes[0].cpu().numpy().astype(np.asarray(cq.codes).dtype),
                               means[0].cpu().numpy())
