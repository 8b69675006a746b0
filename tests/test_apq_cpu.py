"""The .apq container (reference apq.py): header / length / CRC validation with
the reference's exact messages and offsets, and bit-exact serialisation of a
given tensor -- host-only parts, no GPU.  Fixtures: tests/golden/make_apq_golden.py."""

import json
import os
import struct

import numpy as np
import pytest

from paper_2402_10517_b200 import AnyPrecisionLayer, apq
from paper_2402_10517_b200.bitplane import BitplaneTensor
from paper_2402_10517_b200.errors import ApqFormatError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    d = np.load(os.path.join(GOLD, "apq_golden.npz"))
    return d, json.loads(bytes(d["meta_json"]).decode())


def _bytes(name):
    with open(os.path.join(GOLD, f"apq_{name}.apq"), "rb") as f:
        return f.read()


def _corruptions(data: bytes):  # same recipes as make_apq_golden.corruptions
    out = {"truncated": bytes(data[:10])}
    b = bytearray(data); b[0:4] = b"APQ2"; out["magic"] = bytes(b)
    b = bytearray(data); b[4] = 7; b[5] = 3; out["bit_range"] = bytes(b)
    b = bytearray(data); b[6] = 2; out["layout_flag"] = bytes(b)
    b = bytearray(data); b[7] = 1; out["reserved"] = bytes(b)
    b = bytearray(data); struct.pack_into("<I", b, 16, 1000); out["padded"] = bytes(b)
    out["length"] = bytes(data[:-1])
    b = bytearray(data); b[len(b) // 2] ^= 0x40; out["crc"] = bytes(b)
    return out


def test_headers_parse(gold):
    _, meta = gold
    for name, m in meta.items():
        if name.startswith("_"):
            continue
        h = apq._parse(_bytes(name))
        assert (h["rows"], h["cols"], h["n_min"], h["n_max"], h["layout"]) == (
            m["rows"], m["cols"], m["n_min"], m["n_max"], m["layout"])


def test_corruptions_match_reference_messages(gold):
    _, meta = gold
    first = [n for n in meta if not n.startswith("_")][0]
    for cname, bad in _corruptions(_bytes(first)).items():
        want = meta["_errors"][cname]
        with pytest.raises(ApqFormatError) as ei:
            apq._parse(bad)
        assert str(ei.value) == want["message"], cname
        assert ei.value.offset == want["offset"], cname


def test_serialize_given_tensor_bit_exact(gold):
    d, meta = gold
    for name, m in meta.items():
        if name.startswith("_"):
            continue
        data = _bytes(name)
        h = apq._parse(data)
        tables, planes = apq._sections(data, h)
        tensor = BitplaneTensor(np.array(planes), h["rows"], h["cols"], h["padded"], h["layout"])
        layer = AnyPrecisionLayer(n_min=m["n_min"], n_max=m["n_max"], codes=d[f"{name}/codes"],
                                  centroid_tables={k: d[f"{name}/table{k}"] for k in tables},
                                  shape=(m["rows"], m["cols"]))
        assert apq.serialize(layer, tensor, layout=m["layout"]) == data, name
        for k, t in tables.items():
            assert np.array_equal(t.view(np.uint16), d[f"{name}/table{k}"].view(np.uint16))
