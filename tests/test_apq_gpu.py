"""The .apq container on the GPU: read_apq (GPU unpack) returns the reference's
layer bit for bit, serialize (GPU pack) reproduces the reference's bytes, and
load_prepared serves the file's planes section as-is (planes and GEMV outputs
bit-identical to engine.prepare of the same layer)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cases():
    d = np.load(os.path.join(GOLD, "apq_golden.npz"))
    meta = json.loads(bytes(d["meta_json"]).decode())
    return d, {n: m for n, m in meta.items() if not n.startswith("_")}


def test_read_apq_and_serialize_roundtrip():
    from paper_2402_10517_b200 import apq

    d, cases = _cases()
    for name, m in cases.items():
        path = os.path.join(GOLD, f"apq_{name}.apq")
        layer, tensor = apq.read_apq(path)
        assert np.array_equal(layer.codes, d[f"{name}/codes"]), name
        for k in range(m["n_min"], m["n_max"] + 1):
            assert np.array_equal(layer.centroid_tables[k].view(np.uint16), d[f"{name}/table{k}"].view(np.uint16))
        with open(path, "rb") as f:
            ref = f.read()
        assert apq.serialize(layer, layout=m["layout"]) == ref, name  # GPU pack (+ permute)
        assert apq.layers_equal(layer, layer)


def test_load_prepared_serves_planes_as_is():
    import torch

    from paper_2402_10517_b200 import AnyPrecisionLayer, apq, engine

    d, cases = _cases()
    for name, m in cases.items():
        prep_f = apq.load_prepared(os.path.join(GOLD, f"apq_{name}.apq"))
        layer = AnyPrecisionLayer(n_min=m["n_min"], n_max=m["n_max"], codes=d[f"{name}/codes"],
                                  centroid_tables={k: d[f"{name}/table{k}"] for k in range(m["n_min"], m["n_max"] + 1)},
                                  shape=(m["rows"], m["cols"]))
        prep = engine.prepare(layer)
        assert torch.equal(prep_f.planes, prep.planes), name
        x = np.random.default_rng(1).standard_normal(m["cols"])
        for k in range(max(3, m["n_min"]), m["n_max"] + 1):
            cfg = engine.GemvConfig(bit_width=k)
            assert np.array_equal(engine.gemv(prep_f, x, cfg), engine.gemv(prep, x, cfg)), (name, k)
