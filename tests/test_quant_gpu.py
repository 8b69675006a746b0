"""GPU quantizer (csrc/apb_quant.cu) against the REFERENCE's build_any_precision
outputs (tests/golden/quant_golden.npz, made by make_quant_golden.py): codes,
fp16 tables and float64 channel SSE must be bit-identical."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "quant_golden.npz")


def _cases():
    with np.load(GOLDEN) as z:
        return [str(c) for c in z["cases"]]


@pytest.mark.parametrize("name", _cases())
def test_quantizer_bit_exact_vs_reference(name):
    from paper_2402_10517_b200.quantizer import build_any_precision

    z = np.load(GOLDEN)
    w = z[f"{name}/weights"]
    s = z[f"{name}/sens"] if f"{name}/sens" in z else None
    n_min, n_max = (int(v) for v in z[f"{name}/bits"])
    layer = build_any_precision(w, s, n_min, n_max, record_levels=True)
    assert layer.codes.dtype == np.uint8
    np.testing.assert_array_equal(layer.codes, z[f"{name}/codes"])
    for k in range(n_min, n_max + 1):
        np.testing.assert_array_equal(layer.level_codes[k], z[f"{name}/level{k}"], err_msg=f"level codes k={k}")
        np.testing.assert_array_equal(layer.centroid_tables[k].view(np.uint16),
                                      z[f"{name}/table{k}"].view(np.uint16), err_msg=f"table k={k}")
        np.testing.assert_array_equal(layer.channel_sse[k].view(np.uint64), z[f"{name}/sse{k}"].view(np.uint64),
                                      err_msg=f"sse k={k}")


def test_quantizer_row_blocks_and_torch_inputs_agree():
    """Splitting the channels over several device passes (row_block) and
    passing torch tensors give the same bits as one pass over numpy."""
    import torch

    from paper_2402_10517_b200.quantizer import build_any_precision

    rng = np.random.default_rng(5)
    w = rng.standard_normal((37, 2048))
    s = rng.random((37, 2048))
    a = build_any_precision(w, s, 3, 6)
    b = build_any_precision(torch.from_numpy(w).cuda(), torch.from_numpy(s).cuda(), 3, 6, row_block=8)
    np.testing.assert_array_equal(a.codes, b.codes)
    for k in range(3, 7):
        np.testing.assert_array_equal(a.centroid_tables[k].view(np.uint16), b.centroid_tables[k].view(np.uint16))
        np.testing.assert_array_equal(a.channel_sse[k], b.channel_sse[k])


def test_quantizer_full_layer_properties():
    """Llama-2-7B q_proj-sized layer (4096 x 4096): prefix property of the codes
    (the k-bit code is the top k bits of the parent code), ascending tables,
    SSE never larger after a split (before fp16 rounding effects), and the
    layer serves through the GEMV."""
    import torch

    from paper_2402_10517_b200 import engine
    from paper_2402_10517_b200.quantizer import build_any_precision

    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randn(4096, 4096, device="cuda", dtype=torch.float64, generator=g) * 0.02
    s = torch.rand(4096, 4096, device="cuda", dtype=torch.float64, generator=g)
    layer = build_any_precision(w, s, 3, 8, record_levels=True, as_numpy=False)
    for k in range(3, 9):
        assert torch.equal(layer.level_codes[k], layer.codes >> (8 - k)), k
        t = layer.centroid_tables[k].float()
        assert bool((t[:, 1:] >= t[:, :-1]).all()), k
    sse = torch.stack([layer.channel_sse[k] for k in range(3, 9)])
    assert bool((sse[1:] <= sse[:-1] * (1 + 1e-3) + 1e-9).all())
    prep = engine.prepare(layer)
    x = torch.randn(4096, device="cuda", generator=g).half()
    for k in (3, 8):
        y = engine.gemv(prep, x, engine.GemvConfig(bit_width=k))
        ref = engine.dequantize(prep, k).float() @ x.float()
        err = float((y.float() - ref).norm() / ref.norm())
        assert err < 1e-2, (k, err)


def test_quantizer_validation_matches_reference():
    from paper_2402_10517_b200.errors import ParameterError, ShapeError
    from paper_2402_10517_b200.quantizer import build_any_precision

    w = np.ones((4, 16))
    with pytest.raises(ShapeError):
        build_any_precision(np.ones(16), None, 3, 4)
    with pytest.raises(ParameterError):
        build_any_precision(w, None, 1, 4)
    with pytest.raises(ParameterError):
        build_any_precision(w, None, 5, 4)
    bad = w.copy()
    bad[0, 0] = np.nan
    with pytest.raises(ParameterError, match="weights must be finite"):
        build_any_precision(bad, None, 3, 4)
    with pytest.raises(ShapeError):
        build_any_precision(w, np.ones((4, 15)), 3, 4)
    with pytest.raises(ParameterError, match="non-negative"):
        build_any_precision(w, -np.ones((4, 16)), 3, 4)


def test_continue_upscale_bit_exact_vs_reference():
    """continue_upscale (quantizer.py:438-512): 3..5-bit layer (the reference's
    own) extended to 8 bits -- codes, every table and every level's SSE (the
    existing levels recomputed in original column order) bit-identical; codes
    that are not value-contiguous raise the reference's ParameterError."""
    from paper_2402_10517_b200 import AnyPrecisionLayer
    from paper_2402_10517_b200.errors import ParameterError
    from paper_2402_10517_b200.quantizer import continue_upscale

    z = np.load(GOLDEN)
    w, s = z["cont/weights"], z["cont/sens"]
    base = AnyPrecisionLayer(n_min=3, n_max=5, codes=z["cont/base_codes"],
                             centroid_tables={k: z[f"cont/base_table{k}"] for k in range(3, 6)}, shape=w.shape)
    ext = continue_upscale(w, s, base, 8)
    np.testing.assert_array_equal(ext.codes, z["cont/codes"])
    for k in range(3, 9):
        np.testing.assert_array_equal(ext.centroid_tables[k].view(np.uint16), z[f"cont/table{k}"].view(np.uint16),
                                      err_msg=f"table k={k}")
        np.testing.assert_array_equal(ext.channel_sse[k].view(np.uint64), z[f"cont/sse{k}"].view(np.uint64),
                                      err_msg=f"sse k={k}")
    bad = AnyPrecisionLayer(n_min=3, n_max=5, codes=z["cont/bad_codes"], centroid_tables=base.centroid_tables,
                            shape=w.shape)
    with pytest.raises(ParameterError, match=str(z["cont/bad_msg"])):
        continue_upscale(w, s, bad, 8)
    with pytest.raises(ParameterError):
        continue_upscale(w, s, base, 5)


def test_quantize_seed_and_kmeans_bit_exact_vs_reference():
    """quantize_seed (quantizer.py:281-307: sign pattern, 8 distinct values,
    SensitivityMap weights, a dead channel, fewer values than clusters) and
    kmeans_1d_weighted (quantizer.py:122-157 at k = 1, 3, 5, 7, 12 and a padded
    case): codes / assignments and float64 centroids bit-identical."""
    from paper_2402_10517_b200.errors import ParameterError, ShapeError
    from paper_2402_10517_b200.quantizer import SensitivityMap, kmeans_1d_weighted, quantize_seed

    z = np.load(GOLDEN)
    for name in z["seed_cases"]:
        name = str(name)
        w = z[f"seed/{name}/weights"]
        s = SensitivityMap(z[f"seed/{name}/sens"]) if f"seed/{name}/sens" in z else None
        cqs = quantize_seed(w, s, int(z[f"seed/{name}/n1"]))
        np.testing.assert_array_equal(np.stack([c.codes for c in cqs]), z[f"seed/{name}/codes"], err_msg=name)
        np.testing.assert_array_equal(np.stack([c.centroids for c in cqs]).view(np.uint64),
                                      z[f"seed/{name}/centroids"].view(np.uint64), err_msg=name)
    for name in z["km_cases"]:
        name = str(name)
        res = kmeans_1d_weighted(z[f"km/{name}/values"], z[f"km/{name}/weights"], int(z[f"km/{name}/k"]))
        np.testing.assert_array_equal(res.assignments, z[f"km/{name}/assignments"], err_msg=name)
        np.testing.assert_array_equal(res.centroids.view(np.uint64), z[f"km/{name}/centroids"].view(np.uint64),
                                      err_msg=name)
        assert res.padded == bool(z[f"km/{name}/padded"]), name
    with pytest.raises(ShapeError):
        quantize_seed(np.ones((2, 4)), np.ones((2, 5)), 2)
    with pytest.raises(ParameterError):
        quantize_seed(np.ones((1, 4)), None, 1)
    with pytest.raises(ParameterError):
        kmeans_1d_weighted(np.ones(4), np.zeros(4), 2)
    with pytest.raises(ShapeError):
        kmeans_1d_weighted(np.ones((2, 2)), np.ones((2, 2)), 2)


def test_upscale_bit_exact_vs_reference():
    """upscale (quantizer.py:310-367): the interval path (value-contiguous codes,
    incl. identical members and an empty cluster) and the per-cluster general
    path (scrambled codes, a zero-weight cluster, duplicates, an empty cluster)
    give the reference's codes and float64 centroids bit for bit."""
    from paper_2402_10517_b200.errors import ParameterError, ShapeError
    from paper_2402_10517_b200.quantizer import ChannelQuantization, upscale

    z = np.load(GOLDEN)
    for name in z["up_cases"]:
        name = str(name)
        cq = ChannelQuantization(int(z[f"up/{name}/bits"]), z[f"up/{name}/codes_in"], z[f"up/{name}/centroids_in"])
        up = upscale(cq, z[f"up/{name}/row"], z[f"up/{name}/sens"])
        assert up.bit_width == cq.bit_width + 1
        np.testing.assert_array_equal(up.codes, z[f"up/{name}/codes"], err_msg=name)
        np.testing.assert_array_equal(up.centroids.view(np.uint64), z[f"up/{name}/centroids"].view(np.uint64),
                                      err_msg=name)
    cq = ChannelQuantization(2, np.zeros(4, dtype=np.int64), np.zeros(4))
    with pytest.raises(ShapeError):
        upscale(cq, np.ones(3), np.ones(3))
    with pytest.raises(ParameterError):
        upscale(ChannelQuantization(8, np.zeros(4, dtype=np.int64), np.zeros(256)), np.ones(4), np.ones(4))


def test_build_matches_seed_plus_repeated_upscale():
    """test_quantizer.py:197-210 restated: per channel, quantize_seed then
    upscale to n_max gives build_any_precision's codes and (rounded) tables."""
    from paper_2402_10517_b200.quantizer import build_any_precision, quantize_seed, upscale

    rng = np.random.default_rng(8)
    w = rng.standard_normal((5, 300))
    s = rng.random((5, 300))
    layer = build_any_precision(w, s, 2, 5)
    for r in range(5):
        cq = quantize_seed(w[r][None, :], s[r][None, :], 2)[0]
        np.testing.assert_array_equal(cq.centroids.astype(np.float16), layer.centroid_tables[2][r])
        for k in range(3, 6):
            cq = upscale(cq, w[r], s[r])
            np.testing.assert_array_equal(cq.centroids.astype(np.float16), layer.centroid_tables[k][r])
        np.testing.assert_array_equal(cq.codes, layer.codes[r])


def test_clustering_mirror_vs_reference():
    """clustering.cluster_rows / split_boundaries (clustering.py:204-302) on rows
    with many, 3 (padded) and repeated values: bounds, order, padded flags and
    the 2-means splits equal the reference's."""
    from paper_2402_10517_b200 import clustering

    z = np.load(GOLDEN)
    b, order, sv, sw, padded = clustering.cluster_rows(z["cl/values"], z["cl/weights"], 8)
    np.testing.assert_array_equal(b, z["cl/bounds"])
    np.testing.assert_array_equal(order, z["cl/order"])
    np.testing.assert_array_equal(padded, z["cl/padded"])
    split = clustering.split_boundaries(sv, sw, None, None, None, b)
    np.testing.assert_array_equal(split, z["cl/split"])
