"""Mirror of the reference's batched exact 1-D k-means helpers
(clustering.py:204-302) on the GPU kernels of csrc/apb_quant.cu.

``cluster_rows(values, weights, k)`` -> (bounds, order, sorted values, sorted
weights, padded) exactly like the reference (DP bounds with empty trailing
intervals for low-distinct rows, smallest leading cluster on ties), and
``split_boundaries(sv, sw, pw, pwv, pwv2, bounds)`` -> the optimal weighted
2-means split of every interval.  The prefix arrays are recomputed on the
device from (sv, sw) the way ``_prefix_sums`` builds them (sequential float64
cumsums), so they equal the caller's when the caller built them that way; the
interval count of ``bounds`` must be a power of two <= 256 here.
"""

from __future__ import annotations

import numpy as np

from . import _device as dev
from .errors import ParameterError
from .quantizer import KMeans1DResult  # noqa: F401  (defined in clustering.py in the reference)


def cluster_rows(values, weights, k: int):
    """Exact weighted k-means over each row of a (R, n) batch (clustering.py:204-227)."""
    from .quantizer import _cluster_device

    values = np.asarray(values, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    if values.ndim != 2 or weights.shape != values.shape:
        raise ParameterError("values and weights must be (R, n) arrays of one shape")
    if k < 1:
        raise ParameterError(f"cluster count {k} must be >= 1")
    torch = dev.require_cuda()
    w = torch.from_numpy(np.ascontiguousarray(values)).cuda()
    s = torch.from_numpy(np.ascontiguousarray(weights)).cuda()
    bounds, _, _ = _cluster_device(torch, w, s, k)
    order = np.argsort(values, axis=1, kind="stable")
    sv = np.take_along_axis(values, order, axis=1)
    sw = np.take_along_axis(weights, order, axis=1)
    distinct = 1 + np.count_nonzero(np.diff(sv, axis=1) > 0, axis=1)
    return bounds.cpu().numpy().astype(np.int64), order, sv, sw, distinct < k


def split_boundaries(sv, sw, pw, pwv, pwv2, bounds):
    """Optimal weighted 2-means split of every interval (clustering.py:252-302)."""
    from ._lib import check, load

    sv = np.ascontiguousarray(sv, dtype=np.float64)
    sw = np.ascontiguousarray(sw, dtype=np.float64)
    bounds = np.asarray(bounds)
    rows, n = sv.shape
    m = bounds.shape[1] - 1
    if m < 1 or m & (m - 1) or m > 256:
        raise ParameterError(f"{m} intervals: the device split handles powers of two up to 256")
    torch = dev.require_cuda()
    lib = load()
    P = dev.ptr
    d_sv, d_sw = torch.from_numpy(sv).cuda(), torch.from_numpy(sw).cuda()
    ident = torch.arange(n, device="cuda", dtype=torch.int64).repeat(rows, 1).contiguous()
    b = torch.from_numpy(np.ascontiguousarray(bounds, dtype=np.int32)).cuda()
    out = torch.empty(rows, 2 * m + 1, dtype=torch.int32, device="cuda")
    log2m = m.bit_length() - 1
    ws = torch.empty(lib.apb_quant_workspace(rows, n, 2, log2m + 1), dtype=torch.uint8, device="cuda")
    check(lib.apb_quant_split(P(d_sv), P(d_sw), P(ident), rows, n, log2m, P(b), P(out), P(ws), ws.numel(),
                              dev.stream_ptr()), "apb_quant_split")
    return out.cpu().numpy().astype(np.int64)
