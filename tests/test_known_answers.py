"""The reference's known-answer tests for this path,
restated against the B200 package: host-only geometry / table facts run in the
CPU suite, the ones that need the device are marked gpu.

  test_bitplane.py:21-33   all-zero codes -> zero planes; 0b101 plane placement
  test_bitplane.py:97-113  permutation definition, fixed point, bijection, lane-0 weights
  test_engine.py:36-70     transpose: all-ones, formal bit definition, involution,
                           unsupported width, op budget {2:6, 4:24, 8:72}
  test_engine.py:114-130   merged 3-bit table entry layout, pairwise lookups
  test_engine.py:218-245   exact bandwidth counters and path strings; shape / k rejection
  test_engine.py:266-272   gemm dispatch boundary: M = 16 quantized, M = 17 dense
"""

import numpy as np
import pytest


# ---- host-only -----------------------------------------------------------------------

def test_permutation_definition_fixed_point_bijection():
    from paper_2402_10517_b200.bitplane import tile_permutation

    perm = tile_permutation()
    assert all(perm[4 * t + j] == 32 * j + t for t in range(32) for j in range(4))
    assert perm[0] == 0
    assert sorted(perm.tolist()) == list(range(128))


def test_lane_zero_weight_coverage():
    from paper_2402_10517_b200.bitplane import lane_weight_indices

    want = [*range(0, 8), *range(256, 264), *range(512, 520), *range(768, 776)]
    assert lane_weight_indices(0).tolist() == want
    covered = sorted(i for t in range(32) for i in lane_weight_indices(t).tolist())
    assert covered == list(range(1024))


def test_transpose_operation_budget():
    from paper_2402_10517_b200.engine import TRANSPOSE_OP_COUNT

    assert TRANSPOSE_OP_COUNT[4] <= 40
    assert TRANSPOSE_OP_COUNT == {2: 6, 4: 24, 8: 72}


def test_merged_table_entry_layout_and_pairs():
    from paper_2402_10517_b200.engine import build_merged_table
    from paper_2402_10517_b200.errors import ParameterError

    c = np.arange(8, dtype=np.float32) * 0.5
    table = build_merged_table(c)
    assert table.lookup(0) == (0.0, 0.0)
    assert table.lookup(0b000001) == (0.0, 0.5)
    for i in range(8):
        for j in range(8):
            assert table.entries[8 * i + j, 0] == c[i] and table.entries[8 * i + j, 1] == c[j]
    r = np.random.default_rng(3).normal(size=8).astype(np.float32)
    t2 = build_merged_table(r)
    assert all(t2.lookup(8 * i + j) == (float(r[i]), float(r[j])) for i in range(8) for j in range(8))
    with pytest.raises(ParameterError):
        build_merged_table(np.zeros(7))


# ---- device ------------------------------------------------------------------------------

@pytest.mark.gpu
def test_zero_codes_and_single_code_bit_placement():
    from paper_2402_10517_b200.bitplane import pack_bitplanes

    t = pack_bitplanes(np.zeros((3, 10), dtype=np.uint8), 4).numpy()
    assert not np.asarray(t.planes).any() and t.padded_cols == 1024
    t = pack_bitplanes(np.array([[0b101]], dtype=np.uint8), 3).numpy()
    planes = np.asarray(t.planes)
    assert (planes[0, 0, 0], planes[1, 0, 0], planes[2, 0, 0]) == (1, 0, 1)


@pytest.mark.gpu
def test_transpose_known_answers():
    from paper_2402_10517_b200.engine import bit_transpose
    from paper_2402_10517_b200.errors import ParameterError

    for b in (2, 4, 8):
        assert np.all(np.asarray(bit_transpose(np.full((b, 3), 0xFFFFFFFF, dtype=np.uint32))) == 0xFFFFFFFF)
    rng = np.random.default_rng(0)
    for b in (2, 4, 8):
        w = rng.integers(0, 2 ** 32, size=(b,), dtype=np.uint32)
        out = np.asarray(bit_transpose(w))
        for g in range(b):
            for s in range(32 // b):
                for bit in range(b):
                    assert (int(out[g]) >> (s * b + bit)) & 1 == (int(w[bit]) >> (s * b + g)) & 1
        w = rng.integers(0, 2 ** 32, size=(b, 100), dtype=np.uint32)
        assert np.array_equal(np.asarray(bit_transpose(np.asarray(bit_transpose(w)))), w)
    with pytest.raises(ParameterError):
        bit_transpose(np.zeros((3, 2), dtype=np.uint32))


def _mk(seed, rows, cols, n_min, n_max):
    from oracle import oracle as ora
    from paper_2402_10517_b200 import AnyPrecisionLayer, engine

    codes, tables = ora.random_layer_arrays(np.random.default_rng(seed), rows, cols, n_min, n_max)
    layer = AnyPrecisionLayer(n_min=n_min, n_max=n_max, codes=codes, centroid_tables=tables, shape=(rows, cols))
    return layer, engine.prepare(layer)


@pytest.mark.gpu
def test_report_counters_paths_and_rejections():
    from paper_2402_10517_b200.engine import ExecutionReport, GemvConfig, gemm, gemv
    from paper_2402_10517_b200.errors import ParameterError, ShapeError

    _, prep = _mk(10, 8, 2048, 2, 8)
    x = np.random.default_rng(10).normal(size=2048)
    for k in (2, 4, 8):
        rep = ExecutionReport()
        gemv(prep, x, GemvConfig(bit_width=k), report=rep)
        assert rep.planes_bytes_read == k * 8 * 2048 // 8
        assert rep.table_bytes_read == 8 * (1 << k) * 2
        assert rep.path_taken == "gemv"
    rep = ExecutionReport()
    gemv(prep, x, GemvConfig(bit_width=3), report=rep)
    assert rep.path_taken == "gemv-merged" and rep.table_bytes_read == 8 * 64 * 2 * 2
    _, p2 = _mk(11, 2, 1024, 2, 3)
    with pytest.raises(ShapeError):
        gemv(p2, np.zeros(1000), GemvConfig(bit_width=2))
    _, p3 = _mk(12, 2, 1024, 3, 5)
    with pytest.raises(ParameterError):
        gemv(p3, np.zeros(1024), GemvConfig(bit_width=2))
    _, p4 = _mk(24, 3, 1024, 2, 3)
    rng = np.random.default_rng(24)
    for m, want in ((16, "gemm-quantized"), (17, "gemm-dense")):
        rep = ExecutionReport()
        gemm(p4, rng.normal(size=(m, 1024)), GemvConfig(bit_width=2), report=rep)
        assert rep.path_taken == want
