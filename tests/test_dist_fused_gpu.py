"""Fused GEMV + all-gather (dist.ShardedGemvPlan over apb_gemv_grouped_peers /
apb_peer_wait) on ONE GPU: P simulated ranks, each with its own output block,
address each other's blocks directly -- the same stores and arrival counters
the IPC-mapped multi-GPU path uses.  Every rank must end each step holding the
complete output, bit-identical to the concatenation of the per-shard outputs of
the plain launch, and the bounded wait must time out (not hang) when a peer's
arrivals are missing."""

import numpy as np
import pytest

from oracle import oracle as ora

pytestmark = pytest.mark.gpu


def _layer(seed, rows, cols):
    from paper_2402_10517_b200 import AnyPrecisionLayer

    codes, tables = ora.random_layer_arrays(np.random.default_rng(seed), rows, cols, 3, 8)
    return AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols))


@pytest.mark.parametrize("world,k,m,fp16", [(2, 3, 1, True), (3, 5, 1, False), (4, 8, 4, True), (2, 4, 2, False)])
def test_fused_allgather_simulated_ranks(world, k, m, fp16):
    import torch

    from paper_2402_10517_b200 import dist, engine, plan

    shapes = [(1000, 3000), (777, 3000)]
    layers = [_layer(10 + i, r, c) for i, (r, c) in enumerate(shapes)]
    full_rows = [r for r, _ in shapes]
    esz = 2 if fp16 else 4
    _, nbytes = dist.output_layout(full_rows, m, esz)
    gathers = dist.PeerGather.simulated(nbytes, world)
    shard_preps = [[engine.prepare(dist.shard_layer(L, world, r)) for L in layers] for r in range(world)]
    plans = [dist.ShardedGemvPlan(shard_preps[r], full_rows, k, gathers[r], m=m, y_fp16=fp16, shared_x=True,
                                  spin_limit=1 << 22) for r in range(world)]
    refs = [plan.GemvPlan(shard_preps[r], k, m=m, grouped=True, shared_x=True, y_fp16=fp16) for r in range(world)]
    g = torch.Generator(device="cuda").manual_seed(world * 10 + k)
    for step in range(3):  # the arrival targets advance per step
        x = torch.randn(m, 3000, device="cuda", generator=g).half()
        for p in plans + refs:
            p.x[0][:, :3000].copy_(x)
        for p in plans:
            p.launch_gemv()
        for p in plans:
            p.launch_wait()
        for p in refs:
            p.run()
        torch.cuda.synchronize()
        for r in range(world):
            assert gathers[r].status() == 0, (step, r)
        for i, R in enumerate(full_rows):
            want = torch.cat([refs[r].y[i] for r in range(world)], dim=1)
            for r in range(world):
                assert torch.equal(plans[r].y[i], want.to(plans[r].y[i].dtype)), (step, r, i)
        # and the numbers are the layer's: vs the unsharded API
        y_full = engine.gemv(engine.prepare(layers[0]), x[0], engine.GemvConfig(bit_width=k, activations_fp16=True))
        err = float((plans[0].y[0][0].float() - y_full.float()).norm() / y_full.float().norm())
        assert err < (2e-3 if fp16 else 1e-5), err


def test_fused_allgather_wait_times_out_instead_of_hanging():
    import torch

    from paper_2402_10517_b200 import dist, engine

    L = _layer(3, 512, 1024)
    _, nbytes = dist.output_layout([512], 1, 2)
    gathers = dist.PeerGather.simulated(nbytes, 2)
    p0 = dist.ShardedGemvPlan([engine.prepare(dist.shard_layer(L, 2, 0))], [512], 3, gathers[0], spin_limit=20000)
    p0.run()  # rank 1 never contributes
    torch.cuda.synchronize()
    assert gathers[0].status() == 1


def _ipc_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as tdist

    from paper_2402_10517_b200 import dist, engine, plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # both "ranks" on the one GPU: same-device IPC
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shapes = [(1000, 2048), (300, 2048)]
        layers = [_layer(40 + i, r, c) for i, (r, c) in enumerate(shapes)]
        full_rows = [r for r, _ in shapes]
        _, nbytes = dist.output_layout(full_rows, 1, 2)
        g = dist.PeerGather(nbytes)  # cudaMalloc + IPC handle, exchanged over gloo
        preps = [engine.prepare(dist.shard_layer(L, world, rank)) for L in layers]
        sp = dist.ShardedGemvPlan(preps, full_rows, 4, g, shared_x=True, spin_limit=1 << 26)
        ref = plan.GemvPlan(preps, 4, grouped=True, shared_x=True, y_fp16=True)
        ok = True
        for step in range(3):
            x = torch.randn(1, 2048, generator=torch.Generator().manual_seed(step)).half().cuda()
            sp.x[0][:, :2048].copy_(x)
            ref.x[0][:, :2048].copy_(x)
            sp.run()
            ref.run()
            torch.cuda.synchronize()
            ok = ok and g.status() == 0
            slabs = [None] * world
            tdist.all_gather_object(slabs, [y.cpu() for y in ref.y])
            for i in range(len(shapes)):
                want = torch.cat([slabs[r][i] for r in range(world)], dim=1)
                ok = ok and torch.equal(sp.y[i].cpu(), want)
            tdist.barrier()
        g.close()
        q.put((rank, bool(ok)))
    finally:
        tdist.destroy_process_group()


def test_fused_allgather_two_processes_ipc():
    """The real multi-process path (IPC-mapped blocks, cross-process stores and
    system-scope arrival counters), both ranks on the one GPU of the box."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert all(ok for _, ok in res), res


def test_survey_named_entry_points_allgather_and_gemm_small():
    """apb_gemv_allgather (2 simulated ranks, each rank's slab into both outputs,
    then apb_peer_wait) and apb_gemm_small give the plain kernel's numbers."""
    import ctypes

    import torch

    from paper_2402_10517_b200 import _device as dev
    from paper_2402_10517_b200 import dist, engine, plan
    from paper_2402_10517_b200._lib import APB_DTYPE_F32, check, load, ptr_array

    lib, P, st = load(), dev.ptr, dev.stream_ptr()
    L = _layer(8, 900, 2048)
    full = engine.prepare(L)
    x = torch.randn(1, 2048, device="cuda").half()
    ref = plan.GemvPlan([full], 5, grouped=True)
    ref.x[0].copy_(x)
    ref.run()
    # gemm_small: M = 3 rows through the SURVEY-named entry point
    X = torch.randn(3, 2048, device="cuda").half()
    Y = torch.empty(3, 900, device="cuda")
    t = full.tensor
    check(lib.apb_gemm_small(P(t.planes), t.n_max, t.rows, t.cols, t.padded_cols, 5, P(full.tables16[5]), 3, P(X),
                             2048, P(Y), APB_DTYPE_F32, 900, st), "apb_gemm_small")
    Yr = engine.gemm(full, X, engine.GemvConfig(bit_width=5, activations_fp16=True))
    assert torch.equal(Y, Yr)
    # allgather, world 2 on one GPU
    outs = [torch.zeros(1, 900, device="cuda") for _ in range(2)]
    ctrl = [torch.zeros(4, dtype=torch.int32, device="cuda") for _ in range(2)]  # arrivals, expected, status
    yr = ptr_array([P(o) for o in outs])
    fr = ptr_array([P(c) for c in ctrl])
    PP = lambda a: ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))  # noqa: E731
    for r in range(2):
        shard = engine.prepare(dist.shard_layer(L, 2, r))
        r0, _ = dist.shard_bounds(900, 2, r)
        s_ = shard.tensor
        check(lib.apb_gemv_allgather(P(s_.planes), s_.n_max, s_.rows, s_.cols, s_.padded_cols, 5,
                                     P(shard.tables16[5]), P(x), 1, 2048, r, 2, PP(yr), r0, APB_DTYPE_F32, 900,
                                     PP(fr), 0, st), "apb_gemv_allgather")
    for r in range(2):
        c = ctrl[r]
        check(lib.apb_peer_wait(P(c), P(c) + 4, 900, P(c) + 8, 1 << 20, st), "apb_peer_wait")
    torch.cuda.synchronize()
    for r in range(2):
        assert int(ctrl[r][2]) == 0
        assert torch.allclose(outs[r], ref.y[0], rtol=1e-5, atol=1e-5)
    assert torch.equal(outs[0], outs[1])


@pytest.fixture(scope="module")
def layers70b():
    """BASELINE configs[3]: Llama-2-70B layer shapes (q/o 8192x8192, gate/up
    28672x8192 sharing x; down 8192x28672), random codes / sorted tables."""
    return {"qg": [_layer(70, 8192, 8192), _layer(71, 28672, 8192)], "down": [_layer(72, 8192, 28672)]}


@pytest.mark.parametrize("world,k", [(2, 3), (4, 8), (8, 3), (8, 6)])
def test_fused_allgather_llama70b_shapes(layers70b, world, k):
    """configs[3] as a parity case: every 70B shape row-sharded over `world`
    simulated ranks with the fused all-gather; every rank ends the step holding
    the full output, bit-identical to the per-shard plain launches, and the
    gathered numbers match the unsharded layer."""
    import torch

    from paper_2402_10517_b200 import dist, engine, plan

    g = torch.Generator(device="cuda").manual_seed(700 + world * 10 + k)
    for name, layers in layers70b.items():
        cols = layers[0].shape[1]
        full_rows = [L.shape[0] for L in layers]
        _, nbytes = dist.output_layout(full_rows, 1, 2)
        gathers = dist.PeerGather.simulated(nbytes, world)
        shard_preps = [[engine.prepare(dist.shard_layer(L, world, r)) for L in layers] for r in range(world)]
        plans = [dist.ShardedGemvPlan(shard_preps[r], full_rows, k, gathers[r], m=1, y_fp16=True,
                                      shared_x=len(layers) > 1, spin_limit=1 << 22) for r in range(world)]
        refs = [plan.GemvPlan(shard_preps[r], k, m=1, grouped=True, shared_x=len(layers) > 1, y_fp16=True)
                for r in range(world)]
        x = torch.randn(1, cols, device="cuda", generator=g).half()
        for p in plans + refs:
            for xb in {id(t): t for t in p.x}.values():
                xb[:, :cols].copy_(x)
        for p in plans:
            p.launch_gemv()
        for p in plans:
            p.launch_wait()
        for p in refs:
            p.run()
        torch.cuda.synchronize()
        assert all(gathers[r].status() == 0 for r in range(world))
        for i in range(len(layers)):
            want = torch.cat([refs[r].y[i] for r in range(world)], dim=1)
            for r in range(world):
                assert torch.equal(plans[r].y[i], want), (name, r, i)
        # the gathered fp16 outputs against the C oracle on the UNSHARDED layer:
        # within fp16 output rounding (the payload of the all-gather is fp16)
        xh = x[0].float().cpu().numpy()
        for i, L in enumerate(layers):
            planes = ora.permute(ora.pack_bitplanes(L.codes, 8))
            want = ora.gemm(planes, cols, k, L.centroid_tables[k], ora.prep_x(xh, cols, True), nthreads=8)
            want16 = want.astype(np.float16).astype(np.float32)
            for r in range(world):
                got = plans[r].y[i][0].float().cpu().numpy()
                err = ora.rel_err(got, want16)
                assert err < 1e-3, (name, i, r, err)
        for gt in gathers:
            gt.close()
        del plans, refs, shard_preps
        torch.cuda.empty_cache()
