"""GPU parity of the B200 kernels against the reference (golden vectors) and the
CPU oracle, called through the drop-in API / C ABI.

Bars (see DESIGN.md section "Parity"):
  * packing, permutation, prefix unpack, SWAR transpose, merged index stream:
    bit-exact;
  * gemv / gemm: rel_err (helpers.py:131-137 normwise) < 1e-5 against the
    reference's fp32 output -- the reference's own oracle tolerance
    (test_engine.py:149-156); north_star allows 1e-2;
  * plane isolation, determinism, thread-safety: bit-exact.
Mirrors test_bitplane.py, test_engine.py and test_acceptance.py #5-#9.
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import oracle as ora

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-5


@pytest.fixture(scope="module")
def api():
    from paper_2402_10517_b200 import AnyPrecisionLayer, bitplane, engine, errors

    return AnyPrecisionLayer, bitplane, engine, errors


@pytest.fixture(scope="module")
def bp():
    return np.load(os.path.join(GOLD, "bitplane_golden.npz"))


@pytest.fixture(scope="module")
def tr():
    return np.load(os.path.join(GOLD, "transpose_golden.npz"))


@pytest.fixture(scope="module")
def eg():
    return np.load(os.path.join(GOLD, "engine_golden.npz"))


def _names(npz, suffix):
    return sorted({k.split("/")[0] for k in npz.files if k.endswith(suffix)})


def _layer_from_golden(api, eg, name):
    AnyPrecisionLayer = api[0]
    rows, cols, n_min, n_max = (int(v) for v in eg[f"{name}/meta"])
    tables = {k: eg[f"{name}/table{k}"] for k in range(n_min, n_max + 1)}
    return AnyPrecisionLayer(n_min=n_min, n_max=n_max, codes=eg[f"{name}/codes"],
                             centroid_tables=tables, shape=(rows, cols))


def _random_layer(api, seed, rows, cols, n_min=3, n_max=8):
    AnyPrecisionLayer = api[0]
    codes, tables = ora.random_layer_arrays(np.random.default_rng(seed), rows, cols, n_min, n_max)
    return AnyPrecisionLayer(n_min=n_min, n_max=n_max, codes=codes, centroid_tables=tables,
                             shape=(rows, cols))


# ---- bitplane codec (bitplane.py:76-152) ------------------------------------------

def test_pack_permute_unpack_golden(api, bp):
    _, bitplane, _, _ = api
    for name in _names(bp, "/linear"):
        codes = bp[f"{name}/codes"]
        n_max = int(bp[f"{name}/n_max"])
        lin = bitplane.pack_bitplanes(codes, n_max)
        assert lin.layout == "linear" and lin.padded_cols == int(bp[f"{name}/padded"])
        assert np.array_equal(lin.planes, bp[f"{name}/linear"]), name
        per = bitplane.permute_layout(lin)
        assert np.array_equal(per.planes, bp[f"{name}/permuted"]), name
        fused = bitplane.pack_permuted(codes, n_max)
        assert np.array_equal(fused.planes.cpu().numpy(), bp[f"{name}/permuted"]), name
        back = bitplane.inverse_permute_layout(per)
        assert np.array_equal(back.planes, lin.planes)
        for k in range(1, n_max + 1):
            want = bp[f"{name}/unpack{k}"]
            assert np.array_equal(bitplane.unpack_codes(per, k), want), (name, k)
            assert np.array_equal(bitplane.unpack_codes(lin, k), want), (name, k)


def test_pack_large_matches_oracle(api):
    _, bitplane, _, _ = api
    rng = np.random.default_rng(123)
    for rows, cols, n_max in ((4096, 4096, 8), (37, 11008, 8), (300, 1500, 5)):
        codes = rng.integers(0, 1 << n_max, size=(rows, cols), dtype=np.uint8)
        want_lin = ora.pack_bitplanes(codes, n_max)
        got = bitplane.pack_permuted(codes, n_max).planes.cpu().numpy()
        assert np.array_equal(got, ora.permute(want_lin)), (rows, cols)
        assert np.array_equal(bitplane.pack_bitplanes(codes, n_max).planes, want_lin)


def test_pack_errors(api):
    _, bitplane, _, errors = api
    with pytest.raises(errors.CodeRangeError):
        bitplane.pack_bitplanes(np.array([[8]]), 3)
    with pytest.raises(errors.CodeRangeError):  # only the device OR-flag can see this one
        bitplane.pack_bitplanes(np.array([[1, 2, 200]], dtype=np.uint8), 7)
    # a single out-of-range code deep in a large matrix: the kernel skips the
    # shared atomic once a bit is recorded, so a NEW bit must still get through
    big = np.random.default_rng(3).integers(0, 1 << 7, size=(3000, 5000), dtype=np.uint8)
    big[2999, 4999] = 200
    with pytest.raises(errors.CodeRangeError):
        bitplane.pack_permuted(big, 7)
    big[2999, 4999] = 100
    bitplane.pack_permuted(big, 7)  # in range: no error
    with pytest.raises(errors.ShapeError):
        bitplane.pack_bitplanes(np.zeros((0, 4), dtype=np.uint8), 3)
    with pytest.raises(errors.ParameterError):
        bitplane.pack_bitplanes(np.zeros((2, 4), dtype=np.uint8), 9)
    t = bitplane.pack_bitplanes(np.array([[1]], dtype=np.uint8), 2)
    with pytest.raises(errors.ParameterError):
        bitplane.unpack_codes(t, 0)
    with pytest.raises(errors.LayoutError):
        bitplane.inverse_permute_layout(t)
    with pytest.raises(errors.LayoutError):
        bitplane.permute_layout(bitplane.permute_layout(t))


def test_plane_isolation_unpack(api):
    # test_bitplane.py:69-79 on the device
    _, bitplane, _, _ = api
    rng = np.random.default_rng(4)
    codes = rng.integers(0, 256, size=(33, 3000), dtype=np.uint8)
    t = bitplane.pack_permuted(codes, 8)
    import torch

    for k in range(1, 8):
        want = bitplane.unpack_codes(t, k).clone()
        noisy = bitplane.BitplaneTensor(t.planes.clone(), t.rows, t.cols, t.padded_cols, t.layout)
        noisy.planes[k:] = torch.randint(0, 256, noisy.planes[k:].shape, dtype=torch.uint8,
                                         device="cuda")
        assert torch.equal(bitplane.unpack_codes(noisy, k), want), k
        assert np.array_equal(want.cpu().numpy(), codes >> (8 - k))


# ---- SWAR transpose (engine.py:48-92), acceptance #7 --------------------------------

def test_transpose_golden(api, tr):
    _, _, engine, _ = api
    for b in (2, 4, 8):
        assert np.array_equal(engine.bit_transpose(tr[f"bt{b}/in"]), tr[f"bt{b}/out"]), b
    for k in range(2, 9):
        assert np.array_equal(engine.transpose_any_width(tr[f"taw{k}/in"], k), tr[f"taw{k}/out"])


def test_transpose_million_groups_vs_naive(api):
    _, _, engine, _ = api
    rng = np.random.default_rng(555)
    groups = 1_000_000
    for k in (2, 3, 4, 5, 6, 7, 8):
        words = rng.integers(0, 2**32, size=(k, groups), dtype=np.uint32)
        tw = engine.transpose_any_width(words, k)
        b = tw.shape[0]
        mask = np.uint32((1 << b) - 1)
        # naive per-bit oracle (helpers.py:91-105), vectorised over groups
        for j in range(32):
            want = np.zeros(groups, dtype=np.int64)
            for p in range(k):
                want |= ((words[p] >> np.uint32(j)) & np.uint32(1)).astype(np.int64) << (k - 1 - p)
            got = (tw[j % b] >> np.uint32(b * (j // b))) & mask
            assert np.array_equal(got.astype(np.int64), want), (k, j)


def test_transpose_errors(api):
    _, _, engine, errors = api
    with pytest.raises(errors.ParameterError):
        engine.bit_transpose(np.zeros((3, 2), dtype=np.uint32))
    with pytest.raises(errors.ParameterError):
        engine.transpose_any_width(np.zeros((1, 4), dtype=np.uint32), 1)
    with pytest.raises(errors.ShapeError):
        engine.transpose_any_width(np.zeros((4, 4), dtype=np.uint32), 3)


def test_merged_index_stream_golden(api, eg):
    _, _, engine, _ = api
    n = 0
    for name in _names(eg, "/merged_stream"):
        prep = engine.prepare(_layer_from_golden(api, eg, name))
        assert np.array_equal(engine._merged_index_stream(prep), eg[f"{name}/merged_stream"]), name
        n += 1
    assert n >= 3


# ---- GEMV / GEMM (engine.py:284-362), acceptance #5 ------------------------------

def test_gemv_golden_every_k(api, eg):
    _, _, engine, _ = api
    for name in _names(eg, "/meta"):
        layer = _layer_from_golden(api, eg, name)
        prep = engine.prepare(layer)
        assert np.array_equal(prep.planes.cpu().numpy(), eg[f"{name}/permuted"]), name
        x = eg[f"{name}/x"].astype(np.float64)
        for k in layer.supported_bits():
            rep = engine.ExecutionReport()
            y = engine.gemv(prep, x, engine.GemvConfig(bit_width=k), report=rep)
            assert y.dtype == np.float32 and y.shape == (layer.shape[0],)
            assert ora.rel_err(y, eg[f"{name}/gemv{k}"]) < TOL, (name, k, ora.rel_err(y, eg[f"{name}/gemv{k}"]))
            assert [rep.planes_bytes_read, rep.table_bytes_read] == list(eg[f"{name}/gemv{k}/counters"])
            assert rep.path_taken == str(eg[f"{name}/gemv{k}/path"])
            y16 = engine.gemv(prep, x, engine.GemvConfig(bit_width=k, activations_fp16=True))
            assert ora.rel_err(y16, eg[f"{name}/gemv16_{k}"]) < TOL, (name, k)


def test_gemm_golden_quantized_and_dense(api, eg):
    _, _, engine, _ = api
    for name in _names(eg, "/meta"):
        layer = _layer_from_golden(api, eg, name)
        prep = engine.prepare(layer)
        X = eg[f"{name}/X"]
        for k in layer.supported_bits():
            for m in (1, 2, 8, 16, 17):
                rep = engine.ExecutionReport()
                y = engine.gemm(prep, X[:m], engine.GemvConfig(bit_width=k), report=rep)
                want = eg[f"{name}/gemm{k}_m{m}"]
                assert y.shape == want.shape
                assert ora.rel_err(y, want) < TOL, (name, k, m, ora.rel_err(y, want))
                assert rep.path_taken == str(eg[f"{name}/gemm{k}_m{m}/path"]), (name, m)
                assert [rep.planes_bytes_read, rep.table_bytes_read] == list(
                    eg[f"{name}/gemm{k}_m{m}/counters"])


def test_dequantize_golden(api, eg):
    _, _, engine, _ = api
    n = 0
    for name in _names(eg, "/meta"):
        layer = _layer_from_golden(api, eg, name)
        for k in layer.supported_bits():
            key = f"{name}/dequant{k}"
            if key in eg.files:
                assert np.array_equal(engine.dequantize(layer, k), eg[key]), (name, k)
                n += 1
    assert n > 10


@pytest.mark.parametrize("shape", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_gemv_llama7b_shapes_vs_oracle(api, shape):
    _, _, engine, _ = api
    rows, cols = shape
    layer = _random_layer(api, 7 + rows + cols, rows, cols)
    prep = engine.prepare(layer)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(cols)
    per = prep.planes.cpu().numpy()
    for k in range(3, 9):
        t = layer.centroid_tables[k]
        want = ora.gemm(per, cols, k, t, ora.prep_x(x, cols, False), nthreads=8)
        y = engine.gemv(prep, x, engine.GemvConfig(bit_width=k))
        assert ora.rel_err(y, want) < TOL, (shape, k, ora.rel_err(y, want))
        want16 = ora.gemm(per, cols, k, t, ora.prep_x(x, cols, True), nthreads=8)
        y16 = engine.gemv(prep, x, engine.GemvConfig(bit_width=k, activations_fp16=True))
        assert ora.rel_err(y16, want16) < TOL, (shape, k)


@pytest.mark.parametrize("shape", [(8192, 8192), (28672, 8192), (8192, 28672)])
def test_gemv_llama70b_shapes_vs_oracle(api, shape):
    # BASELINE configs[3] shapes, unsharded, against the C oracle on 8 host
    # threads (test_engine.py:149-156's bar): the GPU packer bit-exact against the
    # oracle's CPU packing at 235 MB, then gemv at k = 3 / 6 / 8 with fp32
    # (scaled hi/lo pairs) and fp16 activations
    _, _, engine, _ = api
    rows, cols = shape
    layer = _random_layer(api, 700 + rows + cols, rows, cols)
    prep = engine.prepare(layer)
    planes = prep.planes.cpu().numpy()
    assert np.array_equal(planes, ora.permute(ora.pack_bitplanes(layer.codes, 8))), shape
    x = np.random.default_rng(rows).standard_normal(cols)
    for k in (3, 6, 8):
        t = layer.centroid_tables[k]
        for fp16 in (False, True):
            want = ora.gemm(planes, cols, k, t, ora.prep_x(x, cols, fp16), nthreads=8)
            y = engine.gemv(prep, x, engine.GemvConfig(bit_width=k, activations_fp16=fp16))
            assert ora.rel_err(y, want) < TOL, (shape, k, fp16, ora.rel_err(y, want))


@pytest.mark.parametrize("scale", [1e-30, 1e-6, 1.0, 3e4, 1e5, 1e30])
def test_fp32_activation_magnitudes(api, scale):
    # fp32 activations of any magnitude (engine.py:270-281 keeps them fp32): the
    # hi/lo pairs are taken after a power-of-two row scale (x_split = 2), so
    # |x| >= 65520 does not overflow fp16 and tiny rows keep ~22 bits; rows of
    # one batch may differ by 60 orders of magnitude, an all-zero row stays zero
    _, _, engine, _ = api
    rows, cols = 700, 3000
    layer = _random_layer(api, 123, rows, cols)
    prep = engine.prepare(layer)
    planes = prep.planes.cpu().numpy()
    rng = np.random.default_rng(int(abs(np.log10(scale))) + 5)
    x = (rng.standard_normal((4, cols)) * scale).astype(np.float32)
    x[1] *= 1e-20 if scale > 1 else 1e20
    x[2] = 0.0
    for k in (3, 5, 8):
        want = ora.gemm(planes, cols, k, layer.centroid_tables[k], ora.prep_x(x, cols, False))
        for m in (1, 2, 4):  # row-copy and batch-in-N mappings
            y = engine.gemm(prep, x[:m], engine.GemvConfig(bit_width=k))
            assert np.all(np.isfinite(y)), (scale, k, m)
            for r in range(m):
                if r == 2:
                    assert not np.any(y[r]), (scale, k)
                    continue
                assert ora.rel_err(y[r], want[r]) < TOL, (scale, k, m, r, ora.rel_err(y[r], want[r]))
        yv = engine.gemv(prep, x[0], engine.GemvConfig(bit_width=k))  # per-call host path
        assert ora.rel_err(yv, want[0]) < TOL, (scale, k)
    import torch

    xd = torch.from_numpy(x).cuda()  # device path: apb_split_x_scaled
    yd = engine.gemm(prep, xd, engine.GemvConfig(bit_width=4))
    want = ora.gemm(planes, cols, 4, layer.centroid_tables[4], ora.prep_x(x, cols, False))
    for r in (0, 1, 3):
        assert ora.rel_err(yd[r].cpu().numpy(), want[r]) < TOL, (scale, r)
    assert not torch.any(yd[2])


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16, 40])
def test_small_batch_gemm_vs_oracle(api, m):
    _, _, engine, _ = api
    rows, cols = 333, 2500  # ragged rows and columns
    layer = _random_layer(api, 50 + m, rows, cols, 2, 8)
    prep = engine.prepare(layer)
    X = np.random.default_rng(m).standard_normal((m, cols))
    per = prep.planes.cpu().numpy()
    for k in (2, 3, 4, 5, 8):
        t = layer.centroid_tables[k]
        cfg = engine.GemvConfig(bit_width=k, dense_threshold=64)
        rep = engine.ExecutionReport()
        y = engine.gemm(prep, X, cfg, report=rep)
        assert rep.path_taken == "gemm-quantized"
        want = ora.gemm(per, cols, k, t, ora.prep_x(X, cols, False), nthreads=8)
        assert ora.rel_err(y, want) < TOL, (m, k, ora.rel_err(y, want))
        y16 = engine.gemm(prep, X, engine.GemvConfig(bit_width=k, dense_threshold=64,
                                                     activations_fp16=True))
        want16 = ora.gemm(per, cols, k, t, ora.prep_x(X, cols, True), nthreads=8)
        assert ora.rel_err(y16, want16) < TOL, (m, k)


def test_acceptance_corpus_vs_dense_oracle(api):
    # test_acceptance.py:136-174 corpus: 50 layers up to 4096x4096, gemv vs the
    # fp64 dense oracle at every supported k.
    _, _, engine, _ = api
    rng = np.random.default_rng(4242)
    sizes = [(4096, 4096), (2048, 2048)]
    for _ in range(12):
        sizes.append((int(rng.integers(64, 257)), int(rng.integers(512, 2049))))
    while len(sizes) < 50:
        sizes.append((int(rng.integers(2, 64)), int(rng.integers(8, 513))))
    for rows, cols in sizes:
        n_min = int(rng.integers(2, 5))
        n_max = int(rng.integers(n_min, 9))
        AnyPrecisionLayer = api[0]
        codes, tables = ora.random_layer_arrays(rng, rows, cols, n_min, n_max)
        layer = AnyPrecisionLayer(n_min=n_min, n_max=n_max, codes=codes, centroid_tables=tables,
                                  shape=(rows, cols))
        prep = engine.prepare(layer)
        x = rng.normal(size=cols)
        for k in layer.supported_bits():
            y = engine.gemv(prep, x, engine.GemvConfig(bit_width=k))
            ref = ora.dense_reference_gemv(codes, n_max, tables[k], x, k)
            assert ora.rel_err(y, ref) < TOL, (rows, cols, k, ora.rel_err(y, ref))


def test_plane_isolation_gemv_bit_exact(api):
    # test_engine.py:165-176 / acceptance #6: corrupting planes >= k leaves y identical
    import torch

    _, _, engine, _ = api
    layer = _random_layer(api, 6, 100, 3100, 2, 8)
    prep = engine.prepare(layer)
    x = torch.randn(3100, device="cuda")
    for k in range(2, 9):
        want = engine.gemv(prep, x, engine.GemvConfig(bit_width=k)).clone()
        noisy = engine.prepare(layer)
        if k < 8:
            noisy.planes[k:] = torch.randint(0, 256, noisy.planes[k:].shape, dtype=torch.uint8,
                                             device="cuda")
        got = engine.gemv(noisy, x, engine.GemvConfig(bit_width=k))
        assert torch.equal(got, want), k


def test_merged_and_plain_bit_identical(api):
    _, _, engine, _ = api
    layer = _random_layer(api, 7, 64, 2048, 3, 5)
    prep = engine.prepare(layer)
    x = np.random.default_rng(7).normal(size=2048)
    a = engine.gemv(prep, x, engine.GemvConfig(bit_width=3, use_merged_table=True))
    b = engine.gemv(prep, x, engine.GemvConfig(bit_width=3, use_merged_table=False))
    assert np.array_equal(a, b)


def test_deterministic_and_thread_safe(api):
    # test_engine.py:311-323
    _, _, engine, _ = api
    layer = _random_layer(api, 23, 1200, 2048, 2, 6)
    prep = engine.prepare(layer)
    rng = np.random.default_rng(23)
    xs = [rng.normal(size=2048) for _ in range(16)]
    cfg = engine.GemvConfig(bit_width=4)
    serial = [engine.gemv(prep, x, cfg) for x in xs]
    with ThreadPoolExecutor(max_workers=8) as pool:
        parallel = list(pool.map(lambda x: engine.gemv(prep, x, cfg), xs))
    for a, b in zip(serial, parallel):
        assert np.array_equal(a, b)
    again = [engine.gemv(prep, x, cfg) for x in xs]
    for a, b in zip(serial, again):
        assert np.array_equal(a, b)


def test_bandwidth_counters_proportional(api):
    # acceptance #9: planes bytes read scale exactly as k/8
    _, _, engine, _ = api
    layer = _random_layer(api, 999, 32, 3000, 2, 8)
    prep = engine.prepare(layer)
    x = np.random.default_rng(9).normal(size=3000)
    reads = {}
    for k in range(2, 9):
        rep = engine.ExecutionReport()
        engine.gemv(prep, x, engine.GemvConfig(bit_width=k), report=rep)
        reads[k] = rep.planes_bytes_read
    for k in range(2, 9):
        assert reads[k] * 8 == reads[8] * k


def test_gemv_errors(api):
    _, _, engine, errors = api
    layer = _random_layer(api, 11, 2, 1024, 3, 5)
    prep = engine.prepare(layer)
    with pytest.raises(errors.ShapeError):
        engine.gemv(prep, np.zeros(1000), engine.GemvConfig(bit_width=3))
    with pytest.raises(errors.ParameterError):
        engine.gemv(prep, np.zeros(1024), engine.GemvConfig(bit_width=2))
    with pytest.raises(errors.ShapeError):
        engine.gemv(prep, np.zeros((2, 1024)), engine.GemvConfig(bit_width=3))
    with pytest.raises(errors.ParameterError):
        engine.gemv(prep, np.zeros(1024), engine.GemvConfig(bit_width=4, use_merged_table=True))
    with pytest.raises(errors.ShapeError):
        engine.gemm(prep, np.zeros((0, 1024)), engine.GemvConfig(bit_width=3))
    with pytest.raises(errors.ShapeError):
        engine.gemm(prep, np.zeros(1024), engine.GemvConfig(bit_width=3))
    with pytest.raises(errors.ShapeError):
        engine.gemm(prep, np.zeros((64, 1000)), engine.GemvConfig(bit_width=3))
    with pytest.raises(errors.ParameterError):
        engine.dequantize(layer, 2)


def test_device_tensors_stay_on_device(api):
    import torch

    _, _, engine, _ = api
    layer = _random_layer(api, 12, 256, 4096)
    prep = engine.prepare(layer)
    x = torch.randn(4096, device="cuda")
    y = engine.gemv(prep, x, engine.GemvConfig(bit_width=4))
    assert y.is_cuda and y.dtype == torch.float32
    yh = engine.gemv(prep, x.cpu().numpy(), engine.GemvConfig(bit_width=4))
    assert np.array_equal(y.cpu().numpy(), yh)
    x16 = x.half()
    y16 = engine.gemv(prep, x16, engine.GemvConfig(bit_width=4))
    y16b = engine.gemv(prep, x16.float(), engine.GemvConfig(bit_width=4, activations_fp16=True))
    assert torch.equal(y16, y16b)


def test_plan_relaunch_with_new_activation_pattern(api):
    # apb_gemv_plan_launch may re-point a plan created with ONE x shared by both
    # layers at two distinct x buffers (and back): the shared-activation staging
    # follows the pointers of each launch, so layer 1 never reuses layer 0's x
    import ctypes

    import torch

    from paper_2402_10517_b200 import _device as dev
    from paper_2402_10517_b200._lib import APB_DTYPE_F32, check, int64_array, int_array, load, ptr_array

    _, _, engine, _ = api
    preps = [engine.prepare(_random_layer(api, 40 + i, 512, 2048)) for i in range(2)]
    lib, k = load(), 4
    PP = lambda a: ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))  # noqa: E731
    xs = torch.randn(1, 2048, device="cuda").half()
    xa, xb = torch.randn(1, 2048, device="cuda").half(), torch.randn(1, 2048, device="cuda").half()
    ys = [torch.zeros(1, 512, device="cuda") for _ in range(2)]
    keep = [ptr_array([dev.ptr(p.planes) for p in preps]), int_array([8, 8]), int64_array([512, 512]),
            int64_array([2048, 2048]), int64_array([2048, 2048]), ptr_array([dev.ptr(p.tables16[k]) for p in preps]),
            ptr_array([dev.ptr(xs), dev.ptr(xs)]), int64_array([2048, 2048]), ptr_array([dev.ptr(y) for y in ys])]
    pl, nm, rw, cl, pd, lt, xp, lx, yp = keep
    h = lib.apb_gemv_plan_create(2, PP(pl), nm, rw, cl, pd, k, PP(lt), PP(xp), 1, lx, 0, PP(yp), APB_DTYPE_F32,
                                 int64_array([512, 512]), 0)
    assert h
    try:
        for pair in ((xa, xb), (xs, xs), (xb, xa)):
            check(lib.apb_gemv_plan_launch(h, PP(ptr_array([dev.ptr(t) for t in pair])), None, dev.stream_ptr()),
                  "apb_gemv_plan_launch")
            torch.cuda.synchronize()
            for p, xx, y in zip(preps, pair, ys):
                want = engine.gemv(p, xx[0], engine.GemvConfig(bit_width=k))
                assert torch.equal(y[0], want)
    finally:
        lib.apb_gemv_plan_destroy(h)


def test_norm_plan_rejects_split_activations(api):
    import torch

    from paper_2402_10517_b200 import plan

    _, _, engine, errors = api
    prep = engine.prepare(_random_layer(api, 9, 64, 1024))
    part = torch.zeros(320, device="cuda")
    with pytest.raises(errors.ParameterError):
        plan.GemvPlan([prep], 4, x_split=True, norm=("consumer", part, 1024, 1e-5))


def test_grouped_equals_single(api):
    # the grouped launch (one kernel for several layers) gives each layer's own
    # result (random activations; the round-1 version compared all-zero outputs)
    import torch

    from paper_2402_10517_b200 import plan

    _, _, engine, _ = api
    shapes = [(4096, 4096), (1100, 4096), (4096, 11008), (17, 300)]
    preps = [engine.prepare(_random_layer(api, 100 + i, r, c)) for i, (r, c) in enumerate(shapes)]
    g = torch.Generator(device="cuda").manual_seed(11)
    for k in (3, 4, 6, 8):
        p = plan.GemvPlan(preps, k, m=1, grouped=True)
        q = plan.GemvPlan(preps, k, m=1, grouped=False)
        for (r, c), xa, xb in zip(shapes, p.x, q.x):
            xa[:, :c].copy_(torch.randn(1, c, device="cuda", generator=g).half())
            xb.copy_(xa)
        p.run()
        q.run()
        torch.cuda.synchronize()
        for (r, c), ya, yb in zip(shapes, p.y, q.y):
            # the same products; the fp32 sums are split by warp group along each CTA's
            # item sequence, which the partition of the grouped launch shifts: equal
            # within fp32 reassociation (each launch shape itself is bit-reproducible)
            assert ya.abs().max() > 0
            assert float((ya - yb).norm() / yb.norm()) < 1e-6, (k, r)


def test_large_shape_properties(api):
    # size-independent properties at 70B shapes: (1) GPU unpack == codes >> (8-k)
    # bit-exact; (2) linearity y(a+b) = y(a) + y(b); (3) checksum of checksums:
    # sum_r y_r == x . colsum(dequant_k(W)) using the (independent) dequant kernel.
    import torch

    _, bitplane, engine, _ = api
    AnyPrecisionLayer = api[0]
    rows, cols = 28672, 8192
    g = torch.Generator(device="cuda").manual_seed(0)
    codes = torch.randint(0, 256, (rows, cols), dtype=torch.uint8, device="cuda", generator=g)
    tables = {k: torch.sort(torch.randn(rows, 1 << k, device="cuda", generator=g), dim=1).values.half()
              for k in range(3, 9)}
    layer = AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables,
                              shape=(rows, cols))
    prep = engine.prepare(layer)
    for k in (3, 5, 8):
        assert torch.equal(bitplane.unpack_codes(prep.tensor, k), codes >> (8 - k)), k
    a = torch.randn(cols, device="cuda", generator=g).half()
    b = torch.randn(cols, device="cuda", generator=g).half()
    for k in (3, 4, 8):
        cfg = engine.GemvConfig(bit_width=k)
        ya, yb = engine.gemv(prep, a, cfg), engine.gemv(prep, b, cfg)
        yab = engine.gemv(prep, (a.float() + b.float()), cfg)
        assert ora.rel_err((ya + yb).cpu().numpy(), yab.cpu().numpy()) < TOL, k
        w = engine.dequantize(prep, k).double()
        colsum = w.sum(0)
        lhs = float(ya.double().sum())
        rhs = float((a.double() * colsum).sum())
        scale = float((a.double().abs() * w.abs().sum(0)).sum())
        assert abs(lhs - rhs) <= 1e-5 * scale, (k, lhs, rhs)


def test_step_plan_host_roundtrip(api):
    # plan.StepPlan (one H2D of every activation, the launches from a graph, one
    # D2H of every output) gives exactly the outputs of the single-layer API
    import torch

    from paper_2402_10517_b200 import plan

    _, _, engine, _ = api
    shapes = [(4096, 4096), (1100, 4096), (333, 3000)]
    preps = [engine.prepare(_random_layer(api, 200 + i, r, c)) for i, (r, c) in enumerate(shapes)]
    plans = [plan.GemvPlan(preps[:2], 3, grouped=True, pdl=True, shared_x=True),
             plan.GemvPlan([preps[2]], 8, grouped=False, pdl=True)]
    sp = plan.StepPlan(plans)
    g = torch.Generator().manual_seed(5)
    for x in sp.x_host:
        x.copy_(torch.randn(x.shape, generator=g).half())
    sp.launch()
    torch.cuda.synchronize()
    sp.capture()
    y = [t.clone() for t in sp.run_host()]
    assert not y[0].is_cuda and len(y) == 3
    x0 = sp.x_host[0][0, :4096].clone()
    x1 = sp.x_host[1][0, :3000].clone()
    cfg3 = engine.GemvConfig(bit_width=3, activations_fp16=True)
    cfg8 = engine.GemvConfig(bit_width=8, activations_fp16=True)
    # grouped launch vs each layer alone: the same products, fp32 sums split by warp
    # group along a different CTA partition -- equal within fp32 reassociation
    for j in (0, 1):
        yj = engine.gemv(preps[j], x0, cfg3)
        assert float((y[j][0] - yj).norm() / yj.norm()) < 1e-6, j
    assert torch.equal(y[2][0], engine.gemv(preps[2], x1, cfg8))
    # the copies are graph nodes: new host inputs are read on every replay, and
    # the copy-less graph (host copies issued around it) gives the same bits
    for x in sp.x_host:
        x.copy_(torch.randn(x.shape, generator=g).half())
    y2 = [t.clone() for t in sp.run_host()]
    x0 = sp.x_host[0][0, :4096].clone()
    x1 = sp.x_host[1][0, :3000].clone()
    y20 = engine.gemv(preps[0], x0, cfg3)
    assert float((y2[0][0] - y20).norm() / y20.norm()) < 1e-6
    assert torch.equal(y2[2][0], engine.gemv(preps[2], x1, cfg8))
    sp.capture(host_copies=False)
    y3 = [t.clone() for t in sp.run_host()]
    assert all(torch.equal(a, b) for a, b in zip(y2, y3))
    # zero-copy outputs: the epilogues store into the pinned host block itself
    zp = [plan.GemvPlan(preps[:2], 3, grouped=True, pdl=True, shared_x=True),
          plan.GemvPlan([preps[2]], 8, grouped=False, pdl=True)]
    sz = plan.StepPlan(zp, zero_copy_y=True)
    for a, b in zip(sz.x_host, sp.x_host):
        a.copy_(b)
    sz.launch()
    torch.cuda.synchronize()
    sz.capture()
    for _ in range(3):
        y4 = [t.clone() for t in sz.run_host()]
    assert all(torch.equal(a, b) for a, b in zip(y2, y4))


@pytest.mark.parametrize("shape", [(333, 1500), (17, 300), (1000, 11008), (4096, 3000)])
def test_tma_kernel_paths_vs_oracle(api, shape):
    # every dispatch path of the TMA-fed kernel (csrc/apb_gemv7.cu) against the C
    # oracle: row-copy mapping (1-2 activation rows; fp32 x = hi/lo pair), batch-in-N
    # mapping (3..8 rows), one or two CTAs per SM (small / large launches), ragged
    # rows (rows % 16 != 0), tail tiles (cols % 1024 != 0, odd column counts)
    _, _, engine, _ = api
    rows, cols = shape
    layer = _random_layer(api, 7 + rows, rows, cols)
    prep = engine.prepare(layer)
    planes = prep.planes.cpu().numpy()
    rng = np.random.default_rng(rows * 31 + cols)
    for k in (3, 4, 5, 8):
        for m, fp16 in ((1, True), (1, False), (2, True), (3, True), (4, False), (5, True), (8, True)):
            x = rng.standard_normal((m, cols))
            cfg = engine.GemvConfig(bit_width=k, activations_fp16=fp16, dense_threshold=16)
            y = engine.gemm(prep, x, cfg)
            want = ora.gemm(planes, cols, k, layer.centroid_tables[k], ora.prep_x(x, cols, fp16))
            err = ora.rel_err(y, want)
            assert err < TOL, (shape, k, m, fp16, err)


@pytest.mark.parametrize("shape", [(11008, 4096), (4096, 11008)])
def test_small_batch_llama7b_mlp_shapes_vs_oracle(api, shape):
    # BASELINE configs[2]: the small-batch any-precision GEMM (M = 1, 2, 4, 8) on
    # the Llama-2-7B MLP shapes at k = 3, 4, 8 (engine.py:312-341), vs the oracle
    _, _, engine, _ = api
    rows, cols = shape
    layer = _random_layer(api, 11 + rows, rows, cols)
    prep = engine.prepare(layer)
    planes = prep.planes.cpu().numpy()
    rng = np.random.default_rng(rows + 7 * cols)
    for k in (3, 4, 8):
        for m in (1, 2, 4, 8):
            x = rng.standard_normal((m, cols))
            y = engine.gemm(prep, x, engine.GemvConfig(bit_width=k, activations_fp16=True))
            want = ora.gemm(planes, cols, k, layer.centroid_tables[k], ora.prep_x(x, cols, True), nthreads=8)
            err = ora.rel_err(y, want)
            assert err < TOL, (shape, k, m, err)


@pytest.mark.parametrize("m,fp16", [(1, False), (1, True), (4, False)])
def test_glu_epilogue_matches_silu_of_plain_outputs(api, m, fp16):
    """APB_FLAG_GLU: interleaved (gate, up) rows -> silu(gate . x) * (up . x) from
    the same fp32 row sums the plain launch produces (fp32: 1e-6; fp16 output:
    one rounding of that value)."""
    import torch

    from paper_2402_10517_b200 import plan

    _, _, engine, _ = api
    prep = engine.prepare(_random_layer(api, 77, 2 * 1100, 2900))
    for k in (3, 6):
        glu = plan.GemvPlan([prep], k, m=m, grouped=True, y_fp16=fp16, glu=True)
        ref = plan.GemvPlan([prep], k, m=m, grouped=True, y_fp16=False)
        x = torch.randn(m, 2900, device="cuda", generator=torch.Generator(device="cuda").manual_seed(k)).half()
        glu.x[0][:, :2900].copy_(x)
        ref.x[0][:, :2900].copy_(x)
        glu.run()
        ref.run()
        torch.cuda.synchronize()
        y = ref.y[0]
        want = torch.nn.functional.silu(y[:, 0::2]) * y[:, 1::2]
        got = glu.y[0].float()
        assert got.shape == (m, 1100)
        if fp16:
            assert torch.allclose(got, want.half().float(), rtol=2e-3, atol=1e-3), k
        else:
            assert torch.allclose(got, want, rtol=1e-5, atol=1e-5), k


def test_norm_epilogues_producer_and_consumer(api):
    """apb_gemv_grouped_norm: the producer adds W.x to the fp32 residual,
    writes fp16(resid * w) and per-CTA sums of squares (their total = sum
    resid^2); the consumer scales every row sum by rsqrt(total / n + eps) -- also
    before the GLU epilogue."""
    import torch

    from paper_2402_10517_b200 import plan

    _, _, engine, _ = api
    H = 2048
    prod = engine.prepare(_random_layer(api, 91, H, 1500))
    cons = engine.prepare(_random_layer(api, 92, 2 * 700, H))
    g = torch.Generator(device="cuda").manual_seed(3)
    resid0 = torch.randn(H, device="cuda", generator=g)
    w = (torch.rand(H, device="cuda", generator=g) + 0.5).half()
    part = torch.zeros(320, device="cuda")
    for k in (3, 7):
        resid = resid0.clone()
        p = plan.GemvPlan([prod], k, grouped=True, y_fp16=True, norm=("producer", resid, w, part))
        ref = plan.GemvPlan([prod], k, grouped=True, y_fp16=False)
        x = torch.randn(1, 1500, device="cuda", generator=g).half()
        p.x[0][:, :1500].copy_(x)
        ref.x[0][:, :1500].copy_(x)
        p.run()
        ref.run()
        torch.cuda.synchronize()
        want_r = resid0 + ref.y[0][0]
        assert torch.allclose(resid, want_r, rtol=0, atol=1e-5)
        assert torch.equal(p.y[0][0], (resid * w.float()).half())
        assert abs(float(part.sum()) - float((resid * resid).sum())) <= 1e-4 * float((resid * resid).sum())
        s = float(torch.rsqrt((resid * resid).sum() / H + 1e-5))
        # consumer (plain and GLU) fed the producer's output
        c = plan.GemvPlan([cons], k, grouped=True, y_fp16=False, norm=("consumer", part, H, 1e-5))
        cg = plan.GemvPlan([cons], k, grouped=True, y_fp16=False, glu=True, norm=("consumer", part, H, 1e-5))
        cr = plan.GemvPlan([cons], k, grouped=True, y_fp16=False)
        for q in (c, cg, cr):
            q.x[0][:, :H].copy_(p.y[0])
            q.run()
        torch.cuda.synchronize()
        plain = cr.y[0][0]
        assert torch.allclose(c.y[0][0], s * plain, rtol=1e-5, atol=1e-5)
        gl = torch.nn.functional.silu(s * plain[0::2]) * (s * plain[1::2])
        assert torch.allclose(cg.y[0][0], gl, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("m", [64, 300])
def test_dense_path_tensor_core_fp32_accuracy(api, m):
    """gemm-dense (M > dense_threshold): exact fp16 dequantisation + hi/lo split
    activations on the tensor cores must meet the reference's fp32 bar (1e-5
    vs fp64), per row, including rows scaled by 1e4 / 1e-4 and an all-zero row."""
    import torch

    _, _, engine, _ = api
    layer = _random_layer(api, 55, 1100, 4096)
    prep = engine.prepare(layer)
    rng = np.random.default_rng(m)
    X = rng.standard_normal((m, 4096)).astype(np.float32)
    X[1] *= 1e4
    X[2] *= 1e-4
    X[3] = 0.0
    X[4, ::7] *= 300.0  # wide range inside one row
    for k in (3, 6, 8):
        rep = engine.ExecutionReport()
        y = engine.gemm(prep, X, engine.GemvConfig(bit_width=k), report=rep)
        assert rep.path_taken == "gemm-dense"
        W = engine.dequantize(layer, k).astype(np.float64)
        want = X.astype(np.float64) @ W.T
        err = np.abs(y.astype(np.float64) - want).max(axis=1)
        scale = np.maximum(np.abs(want).max(axis=1), 1e-30)
        assert np.all(y[3] == 0.0)
        rows = np.arange(m) != 3
        assert (err[rows] / scale[rows]).max() < 1e-5, (k, (err[rows] / scale[rows]).max())
        assert ora.rel_err(y, want) < TOL


@pytest.mark.parametrize("m,rows,cols", [(17, 300, 2500), (128, 256, 1024), (257, 129, 3000), (64, 4096, 4096)])
def test_dense_tcgen05_vs_dense_oracle(api, m, rows, cols):
    """The fused tcgen05 dense kernel (csrc/apb_dense_tc.cu: planes + table
    decoded into the UMMA A operand, TMA activations, TMEM accumulator) against
    the fp64 product of the reference dequantisation (engine.py:343-362), every
    k = 2..8, ragged rows / columns / batch (partial 128-row tiles on both MMA
    operands), fp32 activations (hi/lo pairs) and activations_fp16."""
    _, _, engine, _ = api
    layer = _random_layer(api, 900 + m, rows, cols, 2, 8)
    prep = engine.prepare(layer)
    X = np.random.default_rng(m).standard_normal((m, cols)).astype(np.float32)
    X16 = X.astype(np.float16).astype(np.float64)
    for k in range(2, 9):
        W = engine.dequantize(layer, k).astype(np.float64)
        rep = engine.ExecutionReport()
        y = engine.gemm(prep, X, engine.GemvConfig(bit_width=k, dense_threshold=16), report=rep)
        assert rep.path_taken == "gemm-dense"
        assert ora.rel_err(y, X.astype(np.float64) @ W.T) < TOL, (k, ora.rel_err(y, X.astype(np.float64) @ W.T))
        y16 = engine.gemm(prep, X, engine.GemvConfig(bit_width=k, dense_threshold=16, activations_fp16=True))
        assert ora.rel_err(y16, X16 @ W.T) < TOL, k


def test_dense_tcgen05_split_k_deterministic(api):
    """Small-batch dense launches split K across CTAs (apb_gemm_dense_tc_workspace
    > 0 for a 4096-row layer at M = 24); the fixed-order partial sum keeps the
    result bit-identical across calls and equal to the single-pass kernel (no
    workspace) within fp32 reassociation, and within 1e-5 of the fp64 product."""
    import torch

    from paper_2402_10517_b200 import _lib

    _, _, engine, _ = api
    L = _lib.load()
    layer = _random_layer(api, 4242, 4096, 4096, 3, 8)
    prep = engine.prepare(layer)
    t = prep.tensor
    assert L.apb_gemm_dense_tc_workspace(t.rows, t.padded_cols, 48) > 0
    X = np.random.default_rng(7).standard_normal((24, 4096)).astype(np.float32)
    cfg = engine.GemvConfig(bit_width=5, dense_threshold=16)
    y1 = engine.gemm(prep, X, cfg)
    y2 = engine.gemm(prep, X, cfg)
    assert np.array_equal(y1, y2)
    W = engine.dequantize(layer, 5).astype(np.float64)
    assert ora.rel_err(y1, X.astype(np.float64) @ W.T) < TOL
    # the same call without a workspace runs single-pass
    xd = torch.from_numpy(X).cuda()
    xp = torch.empty((48, t.padded_cols), dtype=torch.float16, device="cuda")
    inv = torch.empty(24, dtype=torch.float32, device="cuda")
    from paper_2402_10517_b200 import _device as dev

    _lib.check(L.apb_dense_prep_x(dev.ptr(xd), 0, 24, 4096, 4096, dev.ptr(xp), t.padded_cols, dev.ptr(inv),
                                  dev.stream_ptr()), "prep")
    y0 = torch.empty((24, t.rows), dtype=torch.float32, device="cuda")
    _lib.check(L.apb_gemm_dense_tc(dev.ptr(t.planes), t.n_max, t.rows, t.cols, t.padded_cols, 5,
                                   dev.ptr(prep.tables16[5]), dev.ptr(xp), 48, 1, dev.ptr(inv), dev.ptr(y0), t.rows,
                                   None, 0, dev.stream_ptr()), "dense")
    torch.cuda.synchronize()
    # single pass vs split K: fp32 reassociation of the (scaled) hi/lo products only
    assert ora.rel_err(y0.cpu().numpy(), X.astype(np.float64) @ W.T) < TOL
    assert ora.rel_err(y0.cpu().numpy(), y1) < 2e-5


def test_dense_tcgen05_small_parent_and_rows(api):
    """Dense tcgen05 path with an n_max = 5 parent (the plane-chunk TMA map has 5
    planes) and a 33-row layer (one partial 128-row tile), k = 2..5, against the
    fp64 product of the reference dequantisation."""
    _, _, engine, _ = api
    layer = _random_layer(api, 4343, 33, 1500, 2, 5)
    prep = engine.prepare(layer)
    X = np.random.default_rng(11).standard_normal((40, 1500)).astype(np.float32)
    for k in range(2, 6):
        W = engine.dequantize(layer, k).astype(np.float64)
        y = engine.gemm(prep, X, engine.GemvConfig(bit_width=k, dense_threshold=16))
        assert ora.rel_err(y, X.astype(np.float64) @ W.T) < TOL, k


_REPRO_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import oracle as ora
from paper_2402_10517_b200 import AnyPrecisionLayer, engine, plan
out = {{}}
rng = np.random.default_rng(5)
preps = []
for i, (r, c) in enumerate([(2000, 3000), (1000, 3000), (3500, 3000)]):
    codes, tables = ora.random_layer_arrays(np.random.default_rng(50 + i), r, c, 3, 8)
    preps.append(engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(r, c))))
x = torch.from_numpy(rng.standard_normal((1, 3000))).half().cuda()
for k in (3, 5, 8):
    p = plan.GemvPlan(preps, k, m=1, grouped=True, shared_x=True, y_fp16=False, pdl=True)
    for xb in {{id(t): t for t in p.x}}.values():
        xb[:, :3000].copy_(x)
    for rep in range(3):
        p.run()
        torch.cuda.synchronize()
        for j, y in enumerate(p.y):
            out[f"k{{k}}_l{{j}}_r{{rep}}"] = y.cpu().numpy()
np.savez({path!r}, **out)
"""


def test_gemv_grouped_bits_reproducible_across_processes(tmp_path):
    # a grouped PDL launch (3 layers sharing x, more items than CTAs) gives the
    # same bits run after run and in a second process (fixed partition and
    # fixed fp32 reduction order, apb_gemv7.cu header)
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for run in ("a", "b"):
        path = str(tmp_path / f"run_{run}.npz")
        subprocess.run([sys.executable, "-c", _REPRO_SCRIPT.format(root=root, path=path)], check=True,
                       cwd=root, timeout=600)
        res[run] = np.load(path)
    names = res["a"].files
    assert len(names) == 27
    for n in names:
        assert np.array_equal(res["a"][n], res["b"][n]), n
        base = n.rsplit("_r", 1)[0] + "_r0"
        assert np.array_equal(res["b"][n], res["b"][base]), n


_PAIR_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from oracle import oracle as ora
from paper_2402_10517_b200 import AnyPrecisionLayer, engine
out = {{}}
for rows, cols, m, k in ((300, 3000, 300, 4), (4096, 4096, 512, 3), (1000, 2048, 257, 8)):
    codes, tables = ora.random_layer_arrays(np.random.default_rng(rows + m), rows, cols, 3, 8)
    layer = AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols))
    prep = engine.prepare(layer)
    x = np.random.default_rng(m).standard_normal((m, cols)).astype(np.float32)
    out[f"{{rows}}_{{m}}_{{k}}"] = engine.gemm(prep, x, engine.GemvConfig(bit_width=k))
    W = engine.dequantize(layer, k).astype(np.float64)
    out[f"{{rows}}_{{m}}_{{k}}_ref"] = x.astype(np.float64) @ W.T
np.savez({path!r}, **out)
"""


def test_dense_cta_pair_path_vs_oracle(tmp_path):
    # the opt-in CTA-pair (cta_group::2) dense kernel (APB_DENSE_PAIR=1) against
    # the fp64 product of the reference dequantisation at the 1e-5 bar, M > 128
    # (the 256-wide pair tile), an odd number of 128-row tiles (an all-padding CTA)
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = str(tmp_path / "pair.npz")
    subprocess.run([sys.executable, "-c", _PAIR_SCRIPT.format(root=root, path=path)],
                   env=dict(os.environ, APB_DENSE_PAIR="1"), check=True, cwd=root, timeout=600)
    r = np.load(path)
    names = [n for n in r.files if not n.endswith("_ref")]
    assert len(names) == 3
    for n in names:
        assert ora.rel_err(r[n], r[n + "_ref"]) < TOL, (n, ora.rel_err(r[n], r[n + "_ref"]))


# ---- reference edge cases (test_engine.py:141-163, 247-253) ----------------------------

@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_zero_activations_give_exact_zero(api, k):
    # test_engine.py:141-145: zero x -> y exactly 0 on every path (quantized GEMV,
    # small batch, tcgen05 dense), fp32 and fp16 activations
    _, _, engine, _ = api
    prep = engine.prepare(_random_layer(api, 4, 8, 1024, 2, 5))
    for fp16 in (False, True):
        assert not engine.gemv(prep, np.zeros(1024), engine.GemvConfig(bit_width=k, activations_fp16=fp16)).any()
        for m in (3, 40):
            y = engine.gemm(prep, np.zeros((m, 1024)), engine.GemvConfig(bit_width=k, activations_fp16=fp16))
            assert y.shape == (m, 8) and not y.any(), (m, fp16)


@pytest.mark.parametrize("rows,cols,n_max", [(4, 1024, 4), (1, 1, 8), (3, 5, 3), (17, 1025, 8)])
def test_tiny_and_ragged_layers_vs_oracle(api, rows, cols, n_max):
    # test_engine.py:157-163 (4 x 1024 full-width tiny layer) plus a 1 x 1 layer, a
    # sub-tile ragged one and one a row / column past a tile: gemv and gemm
    # (quantized and dense paths) against the C oracle at the 1e-5 bar
    _, _, engine, _ = api
    layer = _random_layer(api, rows * 7 + cols, rows, cols, 2, n_max)
    prep = engine.prepare(layer)
    planes = prep.planes.cpu().numpy()
    rng = np.random.default_rng(cols)
    for k in range(2, n_max + 1):
        t = layer.centroid_tables[k]
        x = rng.standard_normal(cols)
        want = ora.gemm(planes, cols, k, t, ora.prep_x(x, cols, False), nthreads=4)
        assert ora.rel_err(engine.gemv(prep, x, engine.GemvConfig(bit_width=k)), want) < TOL, k
        X = rng.standard_normal((20, cols))
        W = engine.dequantize(layer, k).astype(np.float64)
        y = engine.gemm(prep, X, engine.GemvConfig(bit_width=k))  # M = 20 > 16: dense path
        assert ora.rel_err(y, X @ W.T) < TOL, k
        y4 = engine.gemm(prep, X[:4], engine.GemvConfig(bit_width=k))  # quantized small batch
        assert ora.rel_err(y4, X[:4] @ W.T) < TOL, k


def test_gemm_m1_equals_gemv(api):
    # test_engine.py:247-253: a one-row GEMM is the GEMV (here bit-identical)
    _, _, engine, _ = api
    prep = engine.prepare(_random_layer(api, 13, 6, 1024, 2, 5))
    x = np.random.default_rng(13).standard_normal((1, 1024))
    for k in (2, 3, 4, 5):
        y = engine.gemm(prep, x, engine.GemvConfig(bit_width=k))
        yv = engine.gemv(prep, x[0], engine.GemvConfig(bit_width=k))
        assert np.array_equal(y[0], yv), k
