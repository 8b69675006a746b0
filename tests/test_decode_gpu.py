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
        W["gate"], W["up"] = W["gate_up"][0::2], W["gate_up"][1::2]  # interleaved rows
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
        assert err < 1e-2, (k, err)  # north_star's bar
        model.capture(k)  # graph replay gives the same bits
        model.step(k)
        torch.cuda.synchronize()
        assert torch.equal(model.hbuf.float().view(-1), got), k


@pytest.mark.parametrize("heads,pos", [(1, 0), (4, 1), (4, 63), (4, 64), (32, 200), (32, 1024), (4, 2047), (4, 2048), (8, 4095)])
def test_attention_decode_vs_fp32(heads, pos):
    """apb_attention_decode (RoPE + cache append + split-chunk attention) against
    fp32 torch on the same fp16 inputs; twice in a row gives the same bits (the
    per-head tickets reset themselves)."""
    import torch

    from paper_2402_10517_b200 import _device as dev
    from paper_2402_10517_b200._lib import check, load

    lib, hd = load(), 128
    g = torch.Generator(device="cuda").manual_seed(pos * 7 + heads)
    stride = (pos + 1 + 5) * hd  # slack rows after pos: must stay untouched
    q, k, v = (torch.randn(heads * hd, device="cuda", generator=g).half() for _ in range(3))
    kc = torch.randn(heads * stride, device="cuda", generator=g).half()
    vc = torch.randn(heads * stride, device="cuda", generator=g).half()
    kc0, vc0 = kc.clone(), vc.clone()
    ang = (pos + 1.5) / (10000.0 ** (torch.arange(0, hd, 2, device="cuda").float() / hd))
    cos, sin = torch.cos(ang).contiguous(), torch.sin(ang).contiguous()
    nbytes = lib.apb_attention_decode_workspace(heads, hd, pos + 1)
    ws = torch.zeros(nbytes, device="cuda", dtype=torch.uint8)
    nxt = torch.randn(2, heads * stride, device="cuda", generator=g).half()  # prefetch target only
    outs = []
    for _ in range(2):
        out = torch.empty(heads * hd, device="cuda", dtype=torch.float16)
        P = dev.ptr
        check(lib.apb_attention_decode(P(q), P(k), P(v), P(cos), P(sin), P(kc), P(vc), heads, hd, stride, pos,
                                       hd ** -0.5, P(ws), nbytes, P(out), P(nxt[0]), P(nxt[1]), dev.stream_ptr()),
              "apb_attention_decode")
        torch.cuda.synchronize()
        outs.append(out)
    assert torch.equal(outs[0], outs[1])

    def rope(t):
        a, b = t[:, : hd // 2], t[:, hd // 2:]
        return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)

    qr = rope(q.float().view(heads, hd))
    kr = rope(k.float().view(heads, hd)).half()
    K = kc0.view(heads, -1, hd)[:, : pos + 1].float().clone()
    V = vc0.view(heads, -1, hd)[:, : pos + 1].float().clone()
    K[:, pos], V[:, pos] = kr.float(), v.float().view(heads, hd)
    att = torch.softmax((qr.unsqueeze(1) @ K.transpose(1, 2)) * hd ** -0.5, dim=-1) @ V
    want = att.view(-1)
    err = float((outs[0].float() - want).abs().max())
    assert err < 2e-3, err
    # cache: row pos now holds rot(k) / v; every other row untouched
    kcv, vcv = kc.view(heads, -1, hd), vc.view(heads, -1, hd)
    assert torch.equal(kcv[:, pos], kr) and torch.equal(vcv[:, pos], v.view(heads, hd))
    mask = torch.ones(kcv.shape[1], dtype=torch.bool, device="cuda")
    mask[pos] = False
    assert torch.equal(kcv[:, mask], kc0.view(heads, -1, hd)[:, mask])
    assert torch.equal(vcv[:, mask], vc0.view(heads, -1, hd)[:, mask])


def test_attention_decode_rejects_bad_arguments():
    from paper_2402_10517_b200._lib import load

    lib = load()
    assert lib.apb_attention_decode_workspace(4, 64, 10) == -1
    assert lib.apb_attention_decode_workspace(4, 128, 0) == -1


@pytest.mark.parametrize("n", [4096, 4097, 11008, 20000])
def test_rms_residual_and_silu_vs_fp32(n):
    """Vector (n % 4 == 0, n <= 16K) and scalar paths of the RMS kernel, with and
    without the residual add; SiLU*up at even and odd n."""
    import torch

    from paper_2402_10517_b200 import _device as dev
    from paper_2402_10517_b200._lib import check, load

    lib, P, st = load(), dev.ptr, dev.stream_ptr()
    g = torch.Generator(device="cuda").manual_seed(n)
    resid = torch.randn(n, device="cuda", generator=g)
    add = torch.randn(n, device="cuda", generator=g).half()
    w = (torch.rand(n, device="cuda", generator=g) + 0.5).half()
    for use_add in (False, True):
        r = resid.clone()
        out = torch.empty(n, device="cuda", dtype=torch.float16)
        check(lib.apb_rms_residual(P(r), P(add) if use_add else None, P(w), P(out), n, 1e-5, st),
              "apb_rms_residual")
        torch.cuda.synchronize()
        want_r = resid + add.float() if use_add else resid
        assert torch.allclose(r, want_r, rtol=0, atol=1e-6)
        want = want_r * torch.rsqrt(want_r.pow(2).mean() + 1e-5) * w.float()
        assert float((out.float() - want).abs().max()) < 4e-3
    gate, up = (torch.randn(n, device="cuda", generator=g).half() for _ in range(2))
    out = torch.empty(n, device="cuda", dtype=torch.float16)
    check(lib.apb_silu_mul(P(gate), P(up), P(out), n, st), "apb_silu_mul")
    torch.cuda.synchronize()
    want = torch.nn.functional.silu(gate.float()) * up.float()
    assert float((out.float() - want).abs().max()) < 1e-2


def test_embed_rms_and_argmax():
    import torch

    from paper_2402_10517_b200 import _device as dev
    from paper_2402_10517_b200._lib import check, load

    lib, P, st = load(), dev.ptr, dev.stream_ptr()
    g = torch.Generator(device="cuda").manual_seed(1)
    emb = torch.randn(100, 4096, device="cuda", generator=g).half()
    w = (torch.rand(4096, device="cuda", generator=g) + 0.5).half()
    tok = torch.tensor([37], device="cuda")
    resid = torch.empty(4096, device="cuda")
    out = torch.empty(4096, device="cuda", dtype=torch.float16)
    check(lib.apb_embed_rms(P(emb), P(tok), 4096, P(resid), P(w), P(out), 1e-5, st), "apb_embed_rms")
    torch.cuda.synchronize()
    r = emb[37].float()
    assert torch.equal(resid, r)
    want = r * torch.rsqrt(r.pow(2).mean() + 1e-5) * w.float()
    assert float((out.float() - want).abs().max()) < 4e-3
    for n in (1, 1000, 32000):
        x = torch.randn(n, device="cuda", generator=g).half()
        x[n // 2] = 60000.0
        if n > 10:
            x[n // 3] = 60000.0  # tie: the first index wins
        o = torch.empty(1, dtype=torch.int64, device="cuda")
        check(lib.apb_argmax_f16(P(x), n, P(o), st), "apb_argmax_f16")
        torch.cuda.synchronize()
        assert int(o) == (n // 3 if n > 10 else 0), (n, int(o))


def test_decode_step_llama7b_block_shapes():
    """Two decoder blocks at the real Llama-2-7B shapes (hidden 4096,
    intermediate 11008, 32 heads, context 256): the folded RMSNorm / GLU
    epilogues and the attention kernel at production sizes, against the same
    fp32 reference built from the dequantized weights."""
    import torch

    from paper_2402_10517_b200 import engine
    from paper_2402_10517_b200.decode import DecodeModel, LlamaConfig

    cfg = LlamaConfig(layers=2, vocab=1000)
    model = DecodeModel(cfg, context=256, seed=5)
    model.token.fill_(123)
    # k = 6 -> 7 -> 8 on ONE model: the RMSNorm producers' grids shrink (down:
    # 256 -> 148 CTAs, o: 256 -> 148 at k = 8), so partial-sum slots the smaller
    # grid does not own must not keep the previous k's values
    for k in (3, 6, 7, 8, 6):
        model.step(k)
        torch.cuda.synchronize()
        got = model.hbuf.float().view(-1)
        want = _reference_hidden(torch, engine, model, k)
        err = float((got - want).norm() / want.norm())
        assert err < 1e-2, (k, err)  # north_star's bar
