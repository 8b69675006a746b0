"""Row-sharded any-precision linears across the GPUs of one node.

SURVEY.md section 8(e): every y[r] depends only on row r's planes and centroid
row plus the full activation, and the reference explicitly allows row-range
partitioning (row-sharded reference outputs concatenate to the
unsharded result).  Rank i of P holds rows [i*R/P, (i+1)*R/P) of every plane and
of every centroid table -- P contiguous slabs per plane, no re-layout -- computes
its slice with the local GEMV kernel and all-gathers the fp32 (or fp16) y slices
over NVLink (NCCL).  x is replicated.

The only exchange step is the all-gather; uneven shards are padded to the
largest shard and trimmed after the collective (``gather_rows``, NCCL), or --
the B200 path -- fused into the GEMV itself: ``ShardedGemvPlan`` stores every
output value straight into every rank's output block over NVLink and counts
the arrivals (``PeerGather`` holds the IPC-mapped blocks).
"""

from __future__ import annotations

import ctypes
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


# ---------------------------------------------------------------------------
# Fused all-gather: the GEMV epilogue stores every output value into every
# rank's output block over NVLink (apb_gemv_grouped_peers), then a one-thread
# wait kernel (apb_peer_wait) completes the step.  No NCCL on the data path.

_CTRL_BYTES = 64  # arrivals u32 | expected u32 | status i32 | pad


def _align(n: int, a: int = 256) -> int:
    return -(-n // a) * a


def output_layout(rows_list, m: int, esz: int):
    """Byte offsets of the full outputs [m][rows] inside a rank's block, and the
    block size (outputs + control words).  Identical on every rank."""
    offs, o = [], 0
    for r in rows_list:
        offs.append(o)
        o += _align(m * r * esz)
    return offs, o + _CTRL_BYTES


def slab_pointers(bases, rank: int, offs, full_rows, m: int, esz: int, ctrl_off: int):
    """Addresses the fused launch of ``rank`` needs, from every rank's block base
    as mapped in this process: its own slab of each output, the same slab in
    each peer's block (``[problem][peer]``, peers in rank order without
    ``rank``), and the arrival counters (peers, then own)."""
    world = len(bases)
    peers = [r for r in range(world) if r != rank]
    r0s = [shard_bounds(R, world, rank)[0] for R in full_rows]
    own = [bases[rank] + o + r0 * esz for o, r0 in zip(offs, r0s)]
    y_peers = [bases[p] + o + r0 * esz for o, r0 in zip(offs, r0s) for p in peers]
    flags = [bases[p] + ctrl_off for p in peers] + [bases[rank] + ctrl_off]
    return own, y_peers, flags


class PeerGather:
    """One symmetric block per rank (cudaMalloc + CUDA IPC handle), every peer's
    block opened in this process; ``bases[r]`` is rank r's block as addressed
    from here.  Control words at ``ctrl_off``: arrivals, expected, status."""

    def __init__(self, nbytes: int, group=None):
        """Collective-safe: every rank takes part in the same handle exchange and
        barrier whatever fails locally; ``ok`` says whether THIS rank mapped every
        peer (callers agree on it across ranks before using the block)."""
        import torch.distributed as dist

        from ._lib import load

        lib = load()
        self._lib = lib
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nbytes = nbytes
        self.ctrl_off = nbytes - _CTRL_BYTES
        self._own, self._opened, self.bases, self.ok = None, [], [], True
        hb = lib.apb_peer_handle_bytes()
        handle = ctypes.create_string_buffer(hb)
        ptr = ctypes.c_void_p()
        mine = None
        if lib.apb_peer_alloc(nbytes, ctypes.byref(ptr), handle) == 0:
            self._own = ptr.value
            mine = bytes(handle.raw)
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=group)
        if any(h is None for h in handles):
            self.ok = False
        else:
            for r, h in enumerate(handles):
                if r == self.rank:
                    self.bases.append(self._own)
                    continue
                p = ctypes.c_void_p()
                if lib.apb_peer_open(ctypes.create_string_buffer(h, hb), ctypes.byref(p)) != 0:
                    self.ok = False
                    break
                self.bases.append(p.value)
                self._opened.append(p.value)
        dist.barrier(group)

    @classmethod
    def simulated(cls, nbytes: int, world: int):
        """``world`` blocks in ONE process on one GPU, each "rank" addressing the
        others directly -- the single-GPU test bed for the fused gather."""
        torch = dev.require_cuda()
        blocks = [torch.zeros(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world)]
        out = []
        for r in range(world):
            g = cls.__new__(cls)
            g._lib, g.world, g.rank, g.nbytes, g.ok = None, world, r, nbytes, True
            g.ctrl_off = nbytes - _CTRL_BYTES
            g.bases = [dev.ptr(b) for b in blocks]
            g._own, g._opened, g._blocks = g.bases[r], [], blocks
            out.append(g)
        return out

    def arrivals(self, rank=None) -> int:
        return self.bases[self.rank if rank is None else rank] + self.ctrl_off

    def view(self, offset: int, shape, dtype):
        """The own block's bytes [offset, ...) as a torch tensor (no copy)."""
        torch = dev.torch()
        if hasattr(self, "_blocks"):
            blk = self._blocks[self.rank]
        else:
            blk = _wrap_device_bytes(torch, self._own, self.nbytes)
        n = 1
        for d in shape:
            n *= d
        esz = torch.tensor([], dtype=dtype).element_size()
        return blk[offset: offset + n * esz].view(dtype).view(*shape)

    def status(self) -> int:
        torch = dev.torch()
        return int(self.view(self.ctrl_off + 8, (1,), torch.int32).item())

    def close(self):
        if self._lib is None:
            return
        for p in self._opened:
            self._lib.apb_peer_close(p)
        if self._own:
            self._lib.apb_peer_free(self._own)
        self._opened, self._own, self._lib = [], None, None


def _wrap_device_bytes(torch, address: int, nbytes: int):
    """A uint8 CUDA tensor over memory this package allocated (no ownership)."""
    class _Cuda:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (address, False), "version": 3}

    return torch.as_tensor(_Cuda(), device="cuda")


class ShardedGemvPlan:
    """This rank's row slab of a grouped GEMV whose outputs are all-gathered by
    the kernel itself: ``launch_gemv()`` writes every rank's block,
    ``launch_wait()`` blocks the stream until all ranks' slabs have landed in
    this rank's block; ``run()`` does both.  ``y[i]`` is the full [m][rows_i]
    output of problem i in this rank's block."""

    def __init__(self, local_preps, full_rows, k: int, gather: PeerGather, m: int = 1, y_fp16: bool = True,
                 pdl: bool = True, shared_x: bool = False, spin_limit: int = 1 << 26):
        from ._lib import APB_DTYPE_F16, APB_DTYPE_F32, APB_FLAG_PDL, int64_array, int_array, load, ptr_array
        from .plan import _ldx

        torch = dev.require_cuda()
        self._lib = load()
        self.k, self.m, self.gather = k, m, gather
        world, rank = gather.world, gather.rank
        esz = 2 if y_fp16 else 4
        self.y_dtype = APB_DTYPE_F16 if y_fp16 else APB_DTYPE_F32
        self.flags = APB_FLAG_PDL if pdl else 0
        offs, need = output_layout(full_rows, m, esz)
        if need > gather.nbytes:
            raise ValueError("PeerGather block too small for these outputs")
        ts = [p.tensor for p in local_preps]
        for t, R in zip(ts, full_rows):
            if t.rows != shard_bounds(R, world, rank)[1] - shard_bounds(R, world, rank)[0]:
                raise ValueError("local layer rows do not match this rank's shard")
        if shared_x:
            x0 = torch.zeros((m, _ldx(ts[0].cols)), dtype=torch.float16, device="cuda")
            self.x = [x0] * len(ts)
        else:
            self.x = [torch.zeros((m, _ldx(t.cols)), dtype=torch.float16, device="cuda") for t in ts]
        ydt = torch.float16 if y_fp16 else torch.float32
        self.y = [gather.view(o, (m, R), ydt) for o, R in zip(offs, full_rows)]
        self.per_step = sum(m * R for R in full_rows)
        own, y_peers, flagp = slab_pointers(gather.bases, rank, offs, full_rows, m, esz, gather.ctrl_off)
        self._n = len(ts)
        self._n_peers = world - 1
        self._planes = ptr_array([dev.ptr(t.planes) for t in ts])
        self._nmax = int_array([t.n_max for t in ts])
        self._rows = int64_array([t.rows for t in ts])
        self._cols = int64_array([t.cols for t in ts])
        self._padded = int64_array([t.padded_cols for t in ts])
        self._lut = ptr_array([dev.ptr(p.tables16[k]) for p in local_preps])
        self._xp = ptr_array([dev.ptr(x) for x in self.x])
        self._ldx = int64_array([x.shape[1] for x in self.x])
        self._yp = ptr_array(own)
        self._ldy = int64_array(list(full_rows))
        self._ypeers = ptr_array(y_peers or [0])
        self._flagp = ptr_array(flagp)
        ctrl = gather.bases[rank] + gather.ctrl_off
        self._arr, self._exp, self._status = ctrl, ctrl + 4, ctrl + 8
        self._spin = spin_limit

    def launch_gemv(self):
        from ._lib import check

        P = lambda a: ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))  # noqa: E731
        check(self._lib.apb_gemv_grouped_peers(
            self._n, P(self._planes), self._nmax, self._rows, self._cols, self._padded, self.k, P(self._lut),
            P(self._xp), self.m, self._ldx, 0, P(self._yp), self.y_dtype, self._ldy, self._n_peers,
            P(self._ypeers), P(self._flagp), self.flags, dev.stream_ptr()), "apb_gemv_grouped_peers")

    def launch_wait(self):
        from ._lib import check

        check(self._lib.apb_peer_wait(self._arr, self._exp, self.per_step, self._status, self._spin,
                                      dev.stream_ptr()), "apb_peer_wait")

    def run(self):
        self.launch_gemv()
        self.launch_wait()
