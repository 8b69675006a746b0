"""Decode step (BASELINE config C5): the fused glue kernels + quantized GEMVs
give the hidden state of an fp32 PyTorch reference built from the dequantized
weights (engine.dequantize), at every bit-width."""

import pytest

pytestmark = pytest.mark.gpu


def _reference_hidden(torch, engine, model, k):
    cfg, ctx = model.cfg, model.context
    nh, hd, H = cfg.heads, cfg.head_dim, cfg.hidden
    w = model.norm_w.float()

    def rms(v):
        return v * torch.rsqrt(v.pow(2).mean() + 1e-5) * w

    def rope(t):
        a, b = t[:, : hd // 2], t[:, hd // 2:]
        return torch.cat([a * model.cos - b * model.sin, b * model.cos + a * model.sin], dim=-1)

    x = model.embed[model.token].view(H).float()
    for li, blk in enumerate(model.blocks):
        W = {n: engine.dequantize(p, k).float() for n, p in blk.items()}
        h = rms(x).half().float()
        q, kk, v = (W[n] @ h for n in ("q", "k", "v"))
        q, kk = rope(q.half().float().view(nh, hd)), rope(kk.half().float().view(nh, hd))
        kc = model.k_cache[li].float().clone()
        vc = model.v_cache[li].float().clone()
        kc[0, :, ctx] = kk
        vc[0, :, ctx] = v.half().float().view(nh, hd)
        att = torch.softmax((q.view(nh, 1, hd) @ kc[0].transpose(1, 2)) / hd ** 0.5, dim=-1) @ vc[0]
        x = x + (W["o"] @ att.reshape(H).half().float()).half().float()
        h = rms(x).half().float()
        g, u = W["gate"] @ h, W["up"] @ h
        a = (torch.nn.functional.silu(g.half().float()) * u.half().float()).half().float()
        x = x + (W["down"] @ a).half().float()
    return rms(x)


def test_decode_step_matches_dequantized_reference():
    import torch

    from paper_2402_10517_b200 import engine
    from paper_2402_10517_b200.decode import DecodeModel, LlamaConfig

    cfg = LlamaConfig(hidden=512, intermediate=1376, heads=4, layers=2, vocab=1000)
    model = DecodeModel(cfg, context=64, seed=3)
    model.token.fill_(17)
    for k in (3, 5, 8):
        model.step(k)  # eager
        torch.cuda.synchronize()
        got = model.hbuf.float().view(-1)
        want = _reference_hidden(torch, engine, model, k)
        err = float((got - want).norm() / want.norm())
        assert err < 2e-2, (k, err)
        model.capture(k)  # graph replay gives the same bits
        model.step(k)
        torch.cuda.synchronize()
        assert torch.equal(model.hbuf.float().view(-1), got), k
