"""Generate golden vectors for the hot path from the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports anyprec 0.1.0 straight from /root/reference/pkg/src (read-only) and
writes small compressed .npz fixtures next to this script.  Nothing at test
or bench time reads /root/reference; the fixtures travel with the repo.

Each case records the reference's own outputs for:
  bitplane.pack_bitplanes / permute_layout / unpack_codes  (bitplane.py:76-136)
  engine.bit_transpose / transpose_any_width               (engine.py:48-92)
  engine._merged_index_stream                              (engine.py:249-260)
  engine.gemv / gemm (both paths) / dequantize + ExecutionReport counters
                                                           (engine.py:284-362)
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _random_layer(rng, rows, cols, n_min, n_max):
    # pkg/tests/helpers.py:108-120, verbatim semantics
    from anyprec import AnyPrecisionLayer

    codes = rng.integers(0, 1 << n_max, size=(rows, cols), dtype=np.uint8)
    tables = {}
    for k in range(n_min, n_max + 1):
        t = rng.normal(size=(rows, 1 << k)).astype(np.float64)
        t.sort(axis=1)
        tables[k] = t.astype(np.float16)
    return AnyPrecisionLayer(n_min=n_min, n_max=n_max, codes=codes, centroid_tables=tables,
                             shape=(rows, cols))


def main():
    sys.path.insert(0, REF_SRC)
    import anyprec
    from anyprec import bitplane, engine

    assert anyprec.__version__ == "0.1.0", anyprec.__version__

    # ---- bitplane packing / permutation / prefix reads ----------------------
    pack_cases = [
        ("allzero", np.zeros((3, 10), dtype=np.uint8), 4),
        ("single101", np.array([[0b101]], dtype=np.uint8), 3),
        ("rand16x2048n8", np.random.default_rng(0).integers(0, 256, (16, 2048), dtype=np.uint8), 8),
        ("rand5x1500n3", np.random.default_rng(1).integers(0, 8, (5, 1500), dtype=np.uint8), 3),
        ("full2x100n8", np.full((2, 100), 255, dtype=np.uint8), 8),
        ("rand7x300n6", np.random.default_rng(2).integers(0, 64, (7, 300), dtype=np.uint8), 6),
        ("rand6x2000n5", np.random.default_rng(7).integers(0, 32, (6, 2000), dtype=np.uint8), 5),
        ("rand9x3100n7", np.random.default_rng(70).integers(0, 128, (9, 3100), dtype=np.uint8), 7),
        ("rand1x1024n1", np.random.default_rng(5).integers(0, 2, (1, 1024), dtype=np.uint8), 1),
    ]
    arrs = {}
    for name, codes, n_max in pack_cases:
        t = bitplane.pack_bitplanes(codes, n_max)
        p = bitplane.permute_layout(t)
        arrs[f"{name}/codes"] = codes
        arrs[f"{name}/n_max"] = np.array(n_max)
        arrs[f"{name}/linear"] = t.planes
        arrs[f"{name}/permuted"] = p.planes
        arrs[f"{name}/padded"] = np.array(t.padded_cols)
        for k in range(1, n_max + 1):
            arrs[f"{name}/unpack{k}"] = bitplane.unpack_codes(p, k)
    arrs["tile_permutation"] = bitplane.tile_permutation()
    arrs["lane_weight_indices"] = np.stack([bitplane.lane_weight_indices(l) for l in range(32)])
    np.savez_compressed(os.path.join(OUT, "bitplane_golden.npz"), **arrs)

    # ---- SWAR transpose -------------------------------------------------------
    arrs = {}
    rng = np.random.default_rng(555)
    for b in (2, 4, 8):
        w = rng.integers(0, 2**32, size=(b, 257), dtype=np.uint32)
        arrs[f"bt{b}/in"] = w
        arrs[f"bt{b}/out"] = engine.bit_transpose(w)
    for k in range(2, 9):
        w = rng.integers(0, 2**32, size=(k, 257), dtype=np.uint32)
        arrs[f"taw{k}/in"] = w
        arrs[f"taw{k}/out"] = engine.transpose_any_width(w, k)
    np.savez_compressed(os.path.join(OUT, "transpose_golden.npz"), **arrs)

    # ---- GEMV / GEMM / dequantize --------------------------------------------
    arrs = {}
    engine_cases = [
        # name, seed, rows, cols, n_min, n_max
        ("L16x2000", 40, 16, 2000, 2, 8),
        ("L6x1100", 6, 6, 1100, 2, 6),
        ("L8x2048", 7, 8, 2048, 3, 5),
        ("L3x1024", 8, 3, 1024, 3, 4),
        ("L33x3000", 99, 33, 3000, 3, 8),
        ("L20x4096", 4242, 20, 4096, 3, 8),
        ("L5x300", 11, 5, 300, 2, 7),
    ]
    for name, seed, rows, cols, n_min, n_max in engine_cases:
        rng = np.random.default_rng(seed)
        layer = _random_layer(rng, rows, cols, n_min, n_max)
        prep = engine.prepare(layer)
        # stored as float32 (exactly what _prep_x feeds the engine) to keep fixtures small
        x = rng.normal(size=cols).astype(np.float32).astype(np.float64)
        X = rng.normal(size=(17, cols)).astype(np.float32).astype(np.float64)
        arrs[f"{name}/codes"] = layer.codes
        arrs[f"{name}/meta"] = np.array([rows, cols, n_min, n_max])
        arrs[f"{name}/x"] = x.astype(np.float32)
        arrs[f"{name}/X"] = X.astype(np.float32)
        arrs[f"{name}/permuted"] = prep.tensor.planes
        for k in layer.supported_bits():
            arrs[f"{name}/table{k}"] = layer.centroid_tables[k]
            rep = engine.ExecutionReport()
            arrs[f"{name}/gemv{k}"] = engine.gemv(prep, x, engine.GemvConfig(bit_width=k), report=rep)
            arrs[f"{name}/gemv{k}/counters"] = np.array(
                [rep.planes_bytes_read, rep.table_bytes_read])
            arrs[f"{name}/gemv{k}/path"] = np.array(rep.path_taken)
            arrs[f"{name}/gemv16_{k}"] = engine.gemv(
                prep, x, engine.GemvConfig(bit_width=k, activations_fp16=True))
            if k == 3:
                arrs[f"{name}/gemv3_plain"] = engine.gemv(
                    prep, x, engine.GemvConfig(bit_width=3, use_merged_table=False))
            if rows * cols <= 40000:
                arrs[f"{name}/dequant{k}"] = engine.dequantize(layer, k)
            for m in (1, 2, 8, 16, 17):
                rep = engine.ExecutionReport()
                arrs[f"{name}/gemm{k}_m{m}"] = engine.gemm(
                    prep, X[:m], engine.GemvConfig(bit_width=k), report=rep)
                arrs[f"{name}/gemm{k}_m{m}/path"] = np.array(rep.path_taken)
                arrs[f"{name}/gemm{k}_m{m}/counters"] = np.array(
                    [rep.planes_bytes_read, rep.table_bytes_read])
        if n_min <= 3 <= n_max:
            arrs[f"{name}/merged_stream"] = engine._merged_index_stream(prep)
    np.savez_compressed(os.path.join(OUT, "engine_golden.npz"), **arrs)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
