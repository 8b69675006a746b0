"""End to end through the B200 components in the order a user chains them:
GPU quantizer (build_any_precision) -> .apq file -> load_prepared (planes
uploaded as-is) -> GEMV at every bit-width, against the layer's own
dequantised weights; plus continue_upscale -> serialize round trip."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_quantize_save_load_serve(tmp_path):
    import torch

    from paper_2402_10517_b200 import apq, engine
    from paper_2402_10517_b200.quantizer import build_any_precision, continue_upscale

    rng = np.random.default_rng(4)
    W = rng.standard_normal((700, 1536)) * 0.05
    S = rng.random((700, 1536))
    layer = build_any_precision(W, S, 3, 6)
    path = tmp_path / "layer.apq"
    apq.write_apq(path, layer)
    prep = apq.load_prepared(path)
    x = torch.randn(1536, device="cuda").half()
    for k in range(3, 7):
        y = engine.gemv(prep, x, engine.GemvConfig(bit_width=k, activations_fp16=True))
        Wk = torch.from_numpy(engine.dequantize(layer, k)).cuda()
        ref = Wk @ x.float()
        assert float((y - ref).norm() / ref.norm()) < 1e-5, k
        # the quantizer's k-bit model approximates the weights (SSE shrinks with k)
        assert np.all(layer.channel_sse[k] >= 0)
    ext = continue_upscale(W, S, layer, 8)
    back, _ = apq.deserialize(apq.serialize(ext))
    assert apq.layers_equal(back, ext)
    assert np.array_equal(ext.codes >> 2, layer.codes)  # the 6-bit codes are the prefix of the 8-bit ones
