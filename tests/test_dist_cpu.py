"""World-size-2 gloo test of the row-sharded path on CPU.

Each rank computes its row slab with the CPU oracle (test-side compute; the
product path uses the GPU kernel) and the product's gather_rows/shard logic
reassembles the full output; it must equal the unsharded oracle result
bit for bit (row partitioning does not change any row's arithmetic)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, rows, cols, k, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle as ora
    from paper_2402_10517_b200 import dist as pdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        codes, tables = ora.random_layer_arrays(np.random.default_rng(7), rows, cols, 3, 8)

        class L:
            n_min, n_max, shape = 3, 8, (rows, cols)

        L.codes, L.centroid_tables = codes, tables
        sh = pdist.shard_layer(L, world, rank)
        r0, r1 = pdist.shard_bounds(rows, world, rank)
        assert sh.shape == (r1 - r0, cols)
        x = np.random.default_rng(1).standard_normal((2, cols)).astype(np.float32)
        planes = ora.permute(ora.pack_bitplanes(sh.codes, 8))
        y_local = ora.gemm(planes, cols, k, sh.centroid_tables[k], x)  # (2, shard)
        y = pdist.gather_rows(torch.from_numpy(y_local), rows).numpy()
        full = ora.gemm(ora.permute(ora.pack_bitplanes(codes, 8)), cols, k, tables[k], x)
        q.put((rank, bool(np.array_equal(y, full)), y.shape))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows", [64, 67])  # even and ragged shards
def test_row_sharded_gather_world2(rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, 1500, 4, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, ok, shape in res:
        assert ok, (rank, shape)
        assert shape == (2, rows)


def test_shard_bounds_cover_rows():
    from paper_2402_10517_b200.dist import max_shard, shard_bounds

    for rows in (1, 7, 4096, 28672, 11008):
        for world in (1, 2, 4, 8):
            spans = [shard_bounds(rows, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max_shard(rows, world) == max(b - a for a, b in spans)


def _fused_worker(rank, world, port, shapes, m, q):
    """The fused gather's addressing protocol (dist.output_layout /
    slab_pointers) end to end on CPU: every rank owns a host "block", the block
    bases are exchanged like the IPC handles, each rank stores its oracle-computed
    slab at the addresses the kernel would use (routed to the owning rank), and
    every block must then hold the unsharded result with the full arrival count."""
    import torch.distributed as dist

    from oracle import oracle as ora
    from paper_2402_10517_b200 import dist as pdist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        esz = 4
        full_rows = [r for r, _ in shapes]
        offs, nbytes = pdist.output_layout(full_rows, m, esz)
        ctrl_off = nbytes - 64
        block = np.zeros(nbytes, dtype=np.uint8)
        base = (rank + 1) << 40  # a distinct fake device address per rank
        bases = [None] * world
        dist.all_gather_object(bases, base)
        own, y_peers, flags = pdist.slab_pointers(bases, rank, offs, full_rows, m, esz, ctrl_off)
        assert len(y_peers) == len(shapes) * (world - 1) and len(flags) == world
        x = np.random.default_rng(1).standard_normal((m, shapes[0][1])).astype(np.float32)
        writes, fulls = [], []
        for i, (rows, cols) in enumerate(shapes):
            codes, tables = ora.random_layer_arrays(np.random.default_rng(20 + i), rows, cols, 3, 8)
            full = ora.gemm(ora.permute(ora.pack_bitplanes(codes, 8)), cols, 5, tables[5], x)  # (m, rows)
            fulls.append(full)
            r0, r1 = pdist.shard_bounds(rows, world, rank)
            mine = ora.gemm(ora.permute(ora.pack_bitplanes(codes[r0:r1], 8)), cols, 5,
                            tables[5][r0:r1], x)
            dsts = [own[i]] + y_peers[i * (world - 1):(i + 1) * (world - 1)]
            for addr in dsts:  # y[m][row] at addr + (m * ldy + row) * esz, ldy = full rows
                for mm in range(m):
                    writes.append((addr + mm * rows * esz, mine[mm].astype("<f4").tobytes()))
        count = sum(m * (pdist.shard_bounds(R, world, rank)[1] - pdist.shard_bounds(R, world, rank)[0])
                    for R in full_rows)
        signals = [(f, count) for f in flags]
        everything = [None] * world
        dist.all_gather_object(everything, (writes, signals))
        arrivals = 0
        for ws, sig in everything:
            for addr, data in ws:
                if base <= addr < base + nbytes:  # a store into this rank's block
                    o = addr - base
                    block[o:o + len(data)] = np.frombuffer(data, dtype=np.uint8)
            for f, c in sig:
                if f == base + ctrl_off:
                    arrivals += c
        ok = arrivals == sum(m * R for R in full_rows)
        for i, R in enumerate(full_rows):
            got = block[offs[i]:offs[i] + m * R * esz].view("<f4").reshape(m, R)
            ok = ok and np.array_equal(got, fulls[i])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_fused_gather_addressing_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    shapes = [(67, 1100), (40, 1100)]
    procs = [ctx.Process(target=_fused_worker, args=(r, 2, port, shapes, 2, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(ok for _, ok in res), res
