"""Golden .apq fixtures from the REFERENCE implementation (apq.py of anyprec
0.1.0, imported read-only from /root/reference/pkg/src in the build container).

    python tests/golden/make_apq_golden.py

Writes, next to this script:
  apq_<name>.apq           the reference's serialize() bytes of a random layer
  apq_golden.npz           per case: the layer's codes and tables (what
                           deserialize must return), and the reference's
                           ApqFormatError message for a set of corruptions of the
                           first case (truncation, magic, bit range, layout,
                           reserved byte, size, CRC; recipes in corruptions(),
                           replayed by tests/test_apq_cpu.py).
Nothing at test or bench time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

CASES = [  # name, rows, cols, n_min, n_max, layout
    ("perm_37x1500_3_8", 37, 1500, 3, 8, "permuted"),
    ("lin_64x1024_2_4", 64, 1024, 2, 4, "linear"),
    ("perm_16x3000_3_6", 16, 3000, 3, 6, "permuted"),
]


def corruptions(data: bytes):
    hdr = bytearray(data)
    out = {"truncated": bytes(data[:10])}
    b = bytearray(data); b[0:4] = b"APQ2"; out["magic"] = bytes(b)
    b = bytearray(data); b[4] = 7; b[5] = 3; out["bit_range"] = bytes(b)
    b = bytearray(data); b[6] = 2; out["layout_flag"] = bytes(b)
    b = bytearray(data); b[7] = 1; out["reserved"] = bytes(b)
    b = bytearray(data); struct.pack_into("<I", b, 16, 1000); out["padded"] = bytes(b)
    out["length"] = bytes(data[:-1])
    b = bytearray(data); b[len(b) // 2] ^= 0x40; out["crc"] = bytes(b)
    del hdr
    return out


def main():
    sys.path.insert(0, REF_SRC)
    from anyprec import AnyPrecisionLayer, apq
    from anyprec.errors import ApqFormatError

    rng = np.random.default_rng(2402)
    arrays, meta = {}, {}
    for name, rows, cols, n_min, n_max, layout in CASES:
        codes = rng.integers(0, 1 << n_max, size=(rows, cols), dtype=np.uint8)
        tables = {}
        for k in range(n_min, n_max + 1):
            t = rng.normal(size=(rows, 1 << k))
            t.sort(axis=1)
            tables[k] = t.astype(np.float16)
        layer = AnyPrecisionLayer(n_min=n_min, n_max=n_max, codes=codes, centroid_tables=tables,
                                  shape=(rows, cols))
        data = apq.serialize(layer, layout=layout)
        with open(os.path.join(OUT, f"apq_{name}.apq"), "wb") as f:
            f.write(data)
        arrays[f"{name}/codes"] = codes
        for k, t in tables.items():
            arrays[f"{name}/table{k}"] = t
        meta[name] = {"rows": rows, "cols": cols, "n_min": n_min, "n_max": n_max, "layout": layout}
    first = CASES[0][0]
    with open(os.path.join(OUT, f"apq_{first}.apq"), "rb") as f:
        data = f.read()
    errors = {}
    for cname, bad in corruptions(data).items():
        try:
            apq.deserialize(bad)
            errors[cname] = None
        except ApqFormatError as e:
            errors[cname] = {"message": str(e), "offset": e.offset}
    meta["_errors"] = errors
    arrays["meta_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "apq_golden.npz"), **arrays)
    print("wrote", len(CASES), "cases,", len(errors), "corruptions")


if __name__ == "__main__":
    main()
