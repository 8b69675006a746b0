"""Row-sharded any-precision linears across the GPUs of one node.

SURVEY.md section 8(e): every y[r] depends only on row r's planes and centroid
row plus the full activation, and the reference explicitly allows row-range
partitioning (row-sharded reference outputs concatenate to the
unsharded result).  Rank i of P holds rows [i*R/P, (i+1)*R/P) of every plane and
of every centroid table -- P contiguous slabs per plane, no re-layout -- computes
its slice with the local GEMV kernel and all-gathers the fp32 (or fp16) y slices
over NVLink (NCCL).  x is replicated.

The only exchange step is the all-gather; uneven shards are padded to the
largest shard and trimmed after the collective.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _device as dev
from .engine import PreparedLayer


def shard_bounds(rows: int, world: int, rank: int) -> tuple:
    """Contiguous row range of ``rank`` (same rule as the bench / tests)."""
    return rows * rank // world, rows * (rank + 1) // world


def max_shard(rows: int, world: int) -> int:
    return max(shard_bounds(rows, world, r)[1] - shard_bounds(rows, world, r)[0]
               for r in range(world))


@dataclass
class _ShardLayer:
    """AnyPrecisionLayer-shaped view of a row slice (codes/tables sliced)."""

    n_min: int
    n_max: int
    codes: object
    centroid_tables: dict
    shape: tuple


def shard_layer(layer, world: int, rank: int):
    """Row slice of a reference-style layer (codes + per-k tables)."""
    r0, r1 = shard_bounds(layer.shape[0], world, rank)
    tables = {k: layer.centroid_tables[k][r0:r1] for k in range(layer.n_min, layer.n_max + 1)}
    return _ShardLayer(layer.n_min, layer.n_max, layer.codes[r0:r1], tables,
                       (r1 - r0, layer.shape[1]))


def gather_rows(local_y, rows: int, group=None):
    """All-gather row slices ``local_y`` [..., shard_rows] of a row-sharded
    output into [..., rows] on every rank (uneven shards padded/trimmed)."""
    import torch.distributed as dist

    torch = dev.torch()
    world = dist.get_world_size(group)
    width = max_shard(rows, world)
    lead = tuple(local_y.shape[:-1])
    pad = torch.zeros(lead + (width,), dtype=local_y.dtype, device=local_y.device)
    pad[..., : local_y.shape[-1]] = local_y
    flat = torch.empty(world * pad.numel(), dtype=local_y.dtype, device=local_y.device)
    dist.all_gather_into_tensor(flat, pad.reshape(-1), group=group)
    out = flat.view((world,) + lead + (width,))
    parts = []
    for r in range(world):
        r0, r1 = shard_bounds(rows, world, r)
        parts.append(out[r][..., : r1 - r0])
    return torch.cat(parts, dim=-1)


class RowShardedLayer:
    """One rank's shard of a large linear + the all-gather of its output.

    ``layer`` is the full (host or device) layer; only the local row slab is
    packed and uploaded.  ``gemv``/``gemm`` take the replicated activation and
    return the full output on every rank."""

    def __init__(self, layer, group=None, prep_fn=PreparedLayer):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.rows = layer.shape[0]
        self.local = prep_fn(shard_layer(layer, self.world, self.rank))

    def gemv(self, x, cfg, report=None):
        from .engine import gemv

        torch = dev.torch()
        y = gemv(self.local, x if dev.is_tensor(x) else torch.as_tensor(x).cuda(), cfg, report)
        return gather_rows(y, self.rows, self.group)

    def gemm(self, x, cfg, report=None):
        from .engine import gemm

        torch = dev.torch()
        y = gemm(self.local, x if dev.is_tensor(x) else torch.as_tensor(x).cuda(), cfg, report)
        return gather_rows(y, self.rows, self.group)
