"""Pin the CPU oracle (oracle/anyprec_oracle.c) to the reference's own outputs.

The golden vectors were produced by importing the reference anyprec 0.1.0
(tests/golden/make_golden.py).  Integer work (packing, permutation, prefix
reads, SWAR transpose, merged index stream) must match bit for bit; float
work (gemv/gemm) must match within the reference's own oracle tolerance
(test_engine.py:149-156 uses rel_err < 1e-5 against an fp64 dense product).
"""

import os

import numpy as np
import pytest

from oracle import oracle as ora

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def bp():
    return np.load(os.path.join(GOLD, "bitplane_golden.npz"))


@pytest.fixture(scope="module")
def tr():
    return np.load(os.path.join(GOLD, "transpose_golden.npz"))


@pytest.fixture(scope="module")
def eg():
    return np.load(os.path.join(GOLD, "engine_golden.npz"))


def _cases(npz, suffix):
    return sorted({k.split("/")[0] for k in npz.files if k.endswith(suffix)})


def test_pack_and_permute_bit_exact(bp):
    names = _cases(bp, "/linear")
    assert len(names) >= 8
    for name in names:
        codes = bp[f"{name}/codes"]
        n_max = int(bp[f"{name}/n_max"])
        lin = ora.pack_bitplanes(codes, n_max)
        assert np.array_equal(lin, bp[f"{name}/linear"]), name
        per = ora.permute(lin)
        assert np.array_equal(per, bp[f"{name}/permuted"]), name
        assert np.array_equal(ora.permute(per, inverse=True), lin), name


def test_unpack_prefix_bit_exact(bp):
    for name in _cases(bp, "/linear"):
        codes = bp[f"{name}/codes"]
        n_max = int(bp[f"{name}/n_max"])
        per = bp[f"{name}/permuted"]
        lin = bp[f"{name}/linear"]
        for k in range(1, n_max + 1):
            want = bp[f"{name}/unpack{k}"]
            assert np.array_equal(ora.unpack_codes(per, codes.shape[1], k, True), want), (name, k)
            assert np.array_equal(ora.unpack_codes(lin, codes.shape[1], k, False), want), (name, k)
            assert np.array_equal(want, codes >> (n_max - k))


def test_pad_columns():
    # test_bitplane.py:90-93
    assert ora.pad_columns(1) == 1024
    assert ora.pad_columns(1024) == 1024
    assert ora.pad_columns(1025) == 2048


def test_code_range_rejected():
    with pytest.raises(ora.OracleError):
        ora.pack_bitplanes(np.array([[8]], dtype=np.uint8), 3)


def test_bit_transpose_and_any_width(tr):
    for b in (2, 4, 8):
        assert np.array_equal(ora.bit_transpose(tr[f"bt{b}/in"]), tr[f"bt{b}/out"]), b
    for k in range(2, 9):
        got = ora.transpose_any_width(tr[f"taw{k}/in"], k)
        assert np.array_equal(got, tr[f"taw{k}/out"]), k
        # and against the naive per-bit oracle (helpers.py:91-105)
        bw = got.shape[0]
        want = ora.naive_field_extract(tr[f"taw{k}/in"], k)
        mask = np.uint32((1 << bw) - 1)
        for j in range(32):
            field = (got[j % bw] >> np.uint32(bw * (j // bw))) & mask
            assert np.array_equal(field.astype(np.int64), want[j]), (k, j)


def _engine_names(eg):
    return _cases(eg, "/meta")


def test_gemv_matches_reference(eg):
    for name in _engine_names(eg):
        rows, cols, n_min, n_max = (int(v) for v in eg[f"{name}/meta"])
        per = eg[f"{name}/permuted"]
        x = eg[f"{name}/x"]
        for k in range(n_min, n_max + 1):
            table = eg[f"{name}/table{k}"]
            y = ora.gemm(per, cols, k, table, ora.prep_x(x, cols, False), merged=(k == 3))
            ref = eg[f"{name}/gemv{k}"]
            assert ora.rel_err(y, ref) < 1e-5, (name, k, ora.rel_err(y, ref))
            y16 = ora.gemm(per, cols, k, table, ora.prep_x(x, cols, True))
            assert ora.rel_err(y16, eg[f"{name}/gemv16_{k}"]) < 1e-5, (name, k)
            # and the restated fp64 dense oracle (helpers.py:123-128)
            dense = ora.dense_reference_gemv(eg[f"{name}/codes"], n_max, table, x, k)
            assert ora.rel_err(y, dense) < 1e-5, (name, k)


def test_merged_equals_plain_bit_exact(eg):
    for name in _engine_names(eg):
        rows, cols, n_min, n_max = (int(v) for v in eg[f"{name}/meta"])
        if not n_min <= 3 <= n_max:
            continue
        per = eg[f"{name}/permuted"]
        x32 = ora.prep_x(eg[f"{name}/x"], cols, False)
        t3 = eg[f"{name}/table3"]
        a = ora.gemm(per, cols, 3, t3, x32, merged=True)
        b = ora.gemm(per, cols, 3, t3, x32, merged=False)
        assert np.array_equal(a, b), name


def test_gemm_quantized_matches_reference(eg):
    for name in _engine_names(eg):
        rows, cols, n_min, n_max = (int(v) for v in eg[f"{name}/meta"])
        per = eg[f"{name}/permuted"]
        X = eg[f"{name}/X"]
        for k in range(n_min, n_max + 1):
            table = eg[f"{name}/table{k}"]
            for m in (1, 2, 8, 16, 17):
                want = eg[f"{name}/gemm{k}_m{m}"]
                got = ora.gemm(per, cols, k, table, ora.prep_x(X[:m], cols, False))
                # m == 17 took the reference's dense path (fp32 matmul); same tolerance
                assert ora.rel_err(got, want) < 1e-5, (name, k, m)


def test_threaded_bit_identical_to_serial(eg):
    name = "L33x3000"
    rows, cols, n_min, n_max = (int(v) for v in eg[f"{name}/meta"])
    per = eg[f"{name}/permuted"]
    x32 = ora.prep_x(eg[f"{name}/x"], cols, False)
    for k in (3, 4, 8):
        t = eg[f"{name}/table{k}"]
        serial = ora.gemm(per, cols, k, t, x32, nthreads=1)
        par = ora.gemm(per, cols, k, t, x32, nthreads=7)
        assert np.array_equal(serial, par), k


def test_dequantize_matches_reference(eg):
    n = 0
    for name in _engine_names(eg):
        rows, cols, n_min, n_max = (int(v) for v in eg[f"{name}/meta"])
        for k in range(n_min, n_max + 1):
            key = f"{name}/dequant{k}"
            if key not in eg.files:
                continue
            got = ora.dequantize(eg[f"{name}/codes"], n_max, k, eg[f"{name}/table{k}"])
            assert np.array_equal(got, eg[key]), (name, k)
            n += 1
    assert n > 10


def test_random_layer_generator_reproduces_reference(eg):
    # helpers.random_layer restated in oracle.random_layer_arrays must follow the
    # same RNG call order, so seeded fixtures can be regenerated without the reference.
    rng = np.random.default_rng(40)
    codes, tables = ora.random_layer_arrays(rng, 16, 2000, 2, 8)
    assert np.array_equal(codes, eg["L16x2000/codes"])
    for k in range(2, 9):
        assert np.array_equal(tables[k], eg[f"L16x2000/table{k}"])


def test_quant_golden_fixture_is_consistent():
    """The reference-made quantizer fixture: level codes are bit prefixes of
    the parent codes and every table row is ascending (quantizer.py:4-7)."""
    import os

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "quant_golden.npz"))
    for name in z["cases"]:
        name = str(name)
        n_min, n_max = (int(v) for v in z[f"{name}/bits"])
        codes = z[f"{name}/codes"]
        for k in range(n_min, n_max + 1):
            np.testing.assert_array_equal(z[f"{name}/level{k}"], codes >> (n_max - k))
            t = z[f"{name}/table{k}"].astype(np.float64)
            assert (np.diff(t, axis=1) >= 0).all()
