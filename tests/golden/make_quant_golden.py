"""Golden quantizer fixtures from the REFERENCE implementation
(quantizer.build_any_precision of anyprec 0.1.0, imported read-only from
/root/reference/pkg/src in the build container).

    python tests/golden/make_quant_golden.py

Writes quant_golden.npz next to this script: per case the inputs (weights,
sensitivities or none) and the reference's outputs (parent codes, fp16 tables
for every k, float64 channel_sse for every k, level codes).  The cases cover
random rows with zero-sensitivity entries and a dead (all-zero) row,
low-distinct rows (k_eff < 2^n_min, padded tables, unsplittable clusters),
duplicates, -0.0 / +0.0 ties, n_min = 2, and a row wider than 8192 (deep
pairwise-summation tree), n_min == n_max and a 32-cluster seed; plus
continue_upscale of a 3..5-bit layer to 8 bits ("cont/*") and its error message
for codes that are not value-contiguous; quantize_seed ("seed/*") and
kmeans_1d_weighted at non-power-of-two k ("km/*"); upscale on both of its paths
("up/*"); clustering.cluster_rows / split_boundaries ("cl/*").  Nothing at test or bench time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def cases():
    rng = np.random.default_rng(2402)
    # random rows, random sensitivities with exact zeros, one dead row
    w = rng.standard_normal((12, 700))
    s = rng.random((12, 700))
    s[rng.random((12, 700)) < 0.1] = 0.0
    s[3] = 0.0
    yield "rand_12x700_3_8", w, s, 3, 8
    # low-distinct rows: row i has i+1 distinct values (1..10), uniform sensitivity
    w = np.stack([rng.choice(rng.standard_normal(i + 1), size=300) for i in range(10)])
    yield "lowdistinct_10x300_3_6", w, None, 3, 6
    # n_min = 2, odd width above one tile
    w = rng.standard_normal((6, 1030)) * rng.uniform(0.01, 3.0, (6, 1))
    s = rng.random((6, 1030)) ** 4
    yield "nmin2_6x1030_2_5", w, s, 2, 5
    # signed zeros, heavy ties, integer-valued weights
    w = rng.integers(-3, 4, (5, 257)).astype(np.float64)
    w[w == 0] = np.where(rng.random(int((w == 0).sum())) < 0.5, -0.0, 0.0)
    s = rng.integers(0, 3, (5, 257)).astype(np.float64)
    yield "ties_5x257_2_8", w, s, 2, 8
    # a row wider than 8192: deeper split tree for the SSE / mean reductions
    w = rng.standard_normal((2, 9000))
    s = rng.random((2, 9000))
    yield "wide_2x9000_3_5", w, s, 3, 5
    # seed only (n_min == n_max) and a 32-cluster seed (many DP layers)
    w = rng.standard_normal((6, 500))
    yield "single_6x500_4_4", w, rng.random((6, 500)), 4, 4
    w = rng.standard_normal((4, 1200)) * rng.uniform(0.1, 2.0, (4, 1))
    yield "seed5_4x1200_5_7", w, rng.random((4, 1200)), 5, 7


def main():
    sys.path.insert(0, REF_SRC)
    from anyprec.quantizer import build_any_precision  # noqa: E402

    out = {}
    names = []
    for name, w, s, n_min, n_max in cases():
        layer = build_any_precision(w, s, n_min, n_max, record_levels=True)
        names.append(name)
        out[f"{name}/weights"] = w
        if s is not None:
            out[f"{name}/sens"] = s
        out[f"{name}/bits"] = np.array([n_min, n_max])
        out[f"{name}/codes"] = layer.codes
        for k in range(n_min, n_max + 1):
            out[f"{name}/table{k}"] = layer.centroid_tables[k]
            out[f"{name}/sse{k}"] = layer.channel_sse[k]
            out[f"{name}/level{k}"] = layer.level_codes[k]
    out["cases"] = np.array(names)
    # continue_upscale (quantizer.py:438-512): a 3..5-bit layer extended to 8 bits
    from anyprec.quantizer import continue_upscale  # noqa: E402
    from anyprec.errors import ParameterError  # noqa: E402

    rng = np.random.default_rng(77)
    w = rng.standard_normal((9, 640))
    s = rng.random((9, 640))
    s[2] = 0.0  # dead row -> uniform
    base = build_any_precision(w, s, 3, 5)
    ext = continue_upscale(w, s, base, 8)
    out["cont/weights"], out["cont/sens"] = w, s
    out["cont/base_codes"] = base.codes
    for k in range(3, 6):
        out[f"cont/base_table{k}"] = base.centroid_tables[k]
    out["cont/codes"] = ext.codes
    for k in range(3, 9):
        out[f"cont/table{k}"] = ext.centroid_tables[k]
        out[f"cont/sse{k}"] = ext.channel_sse[k]
    out["cont/bad_codes"] = rng.integers(0, 32, size=(9, 640), dtype=np.uint8)
    # quantize_seed / kmeans_1d_weighted (quantizer.py:122-157, 281-307)
    from anyprec.quantizer import SensitivityMap, kmeans_1d_weighted, quantize_seed  # noqa: E402

    seeds = {
        "sign": (np.sign(rng.standard_normal((3, 40))) * 2.5, None, 2),
        "eight": (rng.permutation(np.arange(8.0))[None, :].repeat(2, 0), None, 3),
        "rand": (rng.standard_normal((5, 300)), rng.random((5, 300)), 2),
        "dead": (rng.standard_normal((4, 100)), np.vstack([rng.random((3, 100)), np.zeros((1, 100))]), 3),
        "tiny": (np.array([[1.0], [2.0]]), None, 2),
    }
    for name, (sw_, ss_, n1) in seeds.items():
        cqs = quantize_seed(sw_, SensitivityMap(ss_) if ss_ is not None else None, n1)
        out[f"seed/{name}/weights"] = sw_
        if ss_ is not None:
            out[f"seed/{name}/sens"] = ss_
        out[f"seed/{name}/n1"] = np.array(n1)
        out[f"seed/{name}/codes"] = np.stack([c.codes for c in cqs])
        out[f"seed/{name}/centroids"] = np.stack([c.centroids for c in cqs])
    kms = [("k1", 1), ("k3", 3), ("k5", 5), ("k7", 7), ("k12", 12)]
    for name, k in kms:
        v = rng.standard_normal(257) * 3.0
        wt = rng.random(257)
        res = kmeans_1d_weighted(v, wt, k)
        out[f"km/{name}/values"], out[f"km/{name}/weights"], out[f"km/{name}/k"] = v, wt, np.array(k)
        out[f"km/{name}/centroids"], out[f"km/{name}/assignments"] = res.centroids, res.assignments
        out[f"km/{name}/padded"] = np.array(res.padded)
    v = np.array([1.0, 1.0, 2.0, 2.0, 2.0])  # fewer distinct values than clusters
    res = kmeans_1d_weighted(v, np.ones(5), 4)
    out["km/pad/values"], out["km/pad/weights"], out["km/pad/k"] = v, np.ones(5), np.array(4)
    out["km/pad/centroids"], out["km/pad/assignments"] = res.centroids, res.assignments
    out["km/pad/padded"] = np.array(res.padded)
    out["km_cases"] = np.array([n for n, _ in kms] + ["pad"])
    # upscale (quantizer.py:310-367): interval and general paths
    from anyprec.quantizer import ChannelQuantization, upscale  # noqa: E402

    ups = {}
    row = rng.standard_normal(200)
    sens = rng.random(200)
    ups["contig"] = (quantize_seed(row[None, :], sens[None, :], 2)[0], row, sens)
    ups["ident"] = (ChannelQuantization(2, np.zeros(4, dtype=np.int64), np.array([1.0, 1.0, 1.0, 1.0])),
                    np.ones(4), np.ones(4))
    rowe = np.concatenate([rng.standard_normal(30) - 3, rng.standard_normal(30) + 3])
    ups["empty"] = (ChannelQuantization(2, np.where(rowe > 0, 3, 0).astype(np.int64), np.array([-3.0, -1.0, 1.0, 3.0])),
                    rowe, rng.random(60))
    cq = quantize_seed(row[None, :], sens[None, :], 3)[0]
    shuffled = ChannelQuantization(3, rng.permutation(cq.codes), cq.centroids)
    ups["general"] = (shuffled, row, sens)
    sz = sens.copy()
    sz[shuffled.codes == 2] = 0.0  # a zero-weight cluster: uniform weights
    ups["general_zw"] = (shuffled, row, sz)
    rowd = np.round(rng.standard_normal(90), 1)
    ups["general_dup"] = (ChannelQuantization(2, rng.integers(0, 3, 90), np.array([-1.0, 0.0, 1.0, 2.0])),
                          rowd, rng.random(90))  # code 3 empty, duplicates within clusters
    for name, (cq_, r_, s_) in ups.items():
        up = upscale(cq_, r_, s_)
        out[f"up/{name}/codes_in"], out[f"up/{name}/centroids_in"] = np.asarray(cq_.codes), cq_.centroids
        out[f"up/{name}/bits"] = np.array(cq_.bit_width)
        out[f"up/{name}/row"], out[f"up/{name}/sens"] = r_, s_
        out[f"up/{name}/codes"], out[f"up/{name}/centroids"] = up.codes, up.centroids
    out["up_cases"] = np.array(list(ups))
    # clustering.cluster_rows / split_boundaries (clustering.py:204-302)
    from anyprec import clustering as cl  # noqa: E402

    vals = np.vstack([rng.standard_normal(150), np.repeat(rng.standard_normal(3), 50),
                      np.round(rng.standard_normal(150), 1)])
    wts = rng.random((3, 150))
    b, order, sv_, sw_, padded = cl.cluster_rows(vals, wts, 8)
    pw, pwv, pwv2 = cl._prefix_sums(sv_, sw_)
    sb = cl.split_boundaries(sv_, sw_, pw, pwv, pwv2, b)
    out["cl/values"], out["cl/weights"] = vals, wts
    out["cl/bounds"], out["cl/order"], out["cl/padded"], out["cl/split"] = b, order, padded, sb
    out["seed_cases"] = np.array(list(seeds))
    try:
        continue_upscale(w, s, type(base)(n_min=3, n_max=5, codes=out["cont/bad_codes"],
                                          centroid_tables=base.centroid_tables, shape=base.shape), 8)
        out["cont/bad_msg"] = np.array("")
    except ParameterError as e:
        out["cont/bad_msg"] = np.array(str(e))
    np.savez_compressed(os.path.join(OUT, "quant_golden.npz"), **out)
    print("wrote", len(names), "cases")


if __name__ == "__main__":
    main()
