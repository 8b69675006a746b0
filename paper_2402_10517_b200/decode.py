"""Single-token decode step of a Llama-2-style decoder with any-precision
quantized linears (BASELINE config C5).

Every linear of every decoder block (q/k/v/o, gate/up/down; arch.py:74-81 of
the reference lists the same seven per block) is one n_max-bit bitplane parent
served at a per-step bit-width k through the B200 GEMV (plan.GemvPlan, grouped
q/k/v launch, fp16 outputs, PDL chain); gate and up are one layer with
interleaved rows whose GEMV epilogue computes SiLU(gate)*up (APB_FLAG_GLU)
straight into the down projection's input.  The glue around them is two fused
sm_100a kernels of csrc/apb_decode.cu (residual add + RMSNorm writing the next
GEMV's activation buffer; RoPE + KV-cache append + split-chunk single-query
attention writing the o-projection's activation buffer), all in the GEMVs' PDL
chain, plus a cuBLAS fp16 LM head; the whole step is captured in one CUDA graph
per k.  Weights are random-init (codes uniform in [0, 2^n_max),
sorted N(0,1) centroid rows, helpers.random_layer semantics), activations are
real (embedding lookup of a token id, norms with unit weights).

This is a measurement vehicle for the quantized hot path inside a full decode
step, not a model loader: there is no tokenizer, no checkpoint, no sampling
beyond argmax.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _device as dev
from .layer import AnyPrecisionLayer


@dataclass
class LlamaConfig:
    hidden: int = 4096
    intermediate: int = 11008
    heads: int = 32
    layers: int = 32
    vocab: int = 32000
    rope_theta: float = 10000.0
    n_min: int = 3
    n_max: int = 8

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def _random_prepared(torch, engine, rows, cols, cfg, g):
    codes = torch.randint(0, 1 << cfg.n_max, (rows, cols), dtype=torch.uint8, device="cuda", generator=g)
    tables = {k: torch.sort(torch.randn(rows, 1 << k, device="cuda", generator=g), dim=1).values.half() * 0.02
              for k in range(cfg.n_min, cfg.n_max + 1)}
    layer = AnyPrecisionLayer(n_min=cfg.n_min, n_max=cfg.n_max, codes=codes, centroid_tables=tables,
                              shape=(rows, cols))
    prep = engine.prepare(layer)
    del codes
    return prep


class DecodeModel:
    """Random-init quantized decoder; ``step(k)`` decodes one token at bit-width k."""

    def __init__(self, cfg: LlamaConfig = LlamaConfig(), context: int = 1024, seed: int = 0):
        torch = dev.require_cuda()
        from . import engine, plan
        from ._lib import load

        self.cfg, self.context = cfg, context
        H, I, nh, hd = cfg.hidden, cfg.intermediate, cfg.heads, cfg.head_dim
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.blocks = []
        for _ in range(cfg.layers):
            # gate and up as ONE layer with interleaved rows (2i = gate_i, 2i+1 = up_i):
            # the GEMV's GLU epilogue writes silu(gate) * up for the down projection
            names = [("q", H, H), ("k", H, H), ("v", H, H), ("o", H, H), ("gate_up", 2 * I, H), ("down", H, I)]
            self.blocks.append({n: _random_prepared(torch, engine, r, c, cfg, g) for n, r, c in names})
        self.embed = (torch.randn(cfg.vocab, H, device="cuda", generator=g) * 0.02).half()
        self.lm_head = (torch.randn(cfg.vocab, H, device="cuda", generator=g) * 0.02).half()
        self.norm_w = torch.ones(H, device="cuda", dtype=torch.float16)
        # KV cache filled with `context` random past positions; the new token is position `context`
        self.k_cache = [torch.randn(1, nh, context + 1, hd, device="cuda", generator=g).half()
                        for _ in range(cfg.layers)]
        self.v_cache = [torch.randn(1, nh, context + 1, hd, device="cuda", generator=g).half()
                        for _ in range(cfg.layers)]
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, device="cuda").float() / hd))
        ang = float(context) * inv
        self.cos, self.sin = torch.cos(ang).contiguous(), torch.sin(ang).contiguous()
        self.resid = torch.zeros(H, device="cuda", dtype=torch.float32)
        ws_bytes = load().apb_attention_decode_workspace(nh, hd, context + 1)
        self.attn_ws = torch.zeros(ws_bytes, device="cuda", dtype=torch.uint8)
        self.hbuf = torch.zeros(1, H, device="cuda", dtype=torch.float16)
        # per-CTA sums of squares of the two RMSNorm producers of a block (zero-filled
        # once; a CTA index is written by the same launch shape every step)
        self.part_a = torch.zeros(320, device="cuda", dtype=torch.float32)
        self.part_b = torch.zeros(320, device="cuda", dtype=torch.float32)
        self.token = torch.zeros(1, dtype=torch.long, device="cuda")
        self.next_token = torch.zeros(1, dtype=torch.long, device="cuda")
        self.kv_prefetch = True
        self._plans, self._graphs = {}, {}
        self._plan_mod = plan

    # ---- per-k launch plans: x / y buffers shared by every block -----------------
    def _plans_for(self, k: int):
        """Per block: qkv | o | gate_up | down.  RMSNorm lives in the epilogues:
        o and down are producers (residual add, fp16(resid * w) straight into the
        next GEMV's activation buffer, per-CTA sums of squares), q/k/v (from block
        1 on) and gate_up are consumers (row sums scaled by the norm factor)."""
        if k in self._plans:
            return self._plans[k]
        plan, cfg = self._plan_mod, self.cfg
        H, eps = cfg.hidden, 1e-5
        per_block = []
        for li, blk in enumerate(self.blocks):
            qkv_norm = None if li == 0 else ("consumer", self.part_b, H, eps)
            qkv = plan.GemvPlan([blk["q"], blk["k"], blk["v"]], k, grouped=True, pdl=True, shared_x=True,
                                y_fp16=True, norm=qkv_norm)
            o = plan.GemvPlan([blk["o"]], k, grouped=True, pdl=True, y_fp16=True,
                              norm=("producer", self.resid, self.norm_w, self.part_a))
            gu = plan.GemvPlan([blk["gate_up"]], k, grouped=True, pdl=True, y_fp16=True, glu=True,
                               norm=("consumer", self.part_a, H, eps))
            dn = plan.GemvPlan([blk["down"]], k, grouped=True, pdl=True, y_fp16=True,
                               norm=("producer", self.resid, self.norm_w, self.part_b))
            o.rebind(o.x, gu.x)    # fp16(resid * w) after the attention block -> gate_up's input
            gu.rebind(gu.x, dn.x)  # silu(gate) * up lands in the down projection's input
            per_block.append((qkv, o, gu, dn))
        for (_, _, _, dn), (qkv, _, _, _) in zip(per_block, per_block[1:]):
            dn.rebind(dn.x, qkv.x[:1])  # fp16(resid * w) after the MLP -> the next block's q/k/v input
        self._plans[k] = per_block
        return per_block

    def _forward(self, k: int):
        torch = dev.require_cuda()
        from ._lib import check, load

        lib, st = load(), dev.stream_ptr()
        cfg, ctx = self.cfg, self.context
        nh, hd, H = cfg.heads, cfg.head_dim, cfg.hidden
        P = dev.ptr
        blocks = self._plans_for(k)
        # embedding row -> fp32 residual and the first block's normalised input, one kernel
        check(lib.apb_embed_rms(P(self.embed), P(self.token), H, P(self.resid), P(self.norm_w),
                                P(blocks[0][0].x[0]), 1e-5, st), "apb_embed_rms")
        for li, (qkv, o, gu, dn) in enumerate(blocks):
            qkv.run()
            check(lib.apb_attention_decode(P(qkv.y[0]), P(qkv.y[1]), P(qkv.y[2]), P(self.cos), P(self.sin),
                                           P(self.k_cache[li]), P(self.v_cache[li]), nh, hd, (ctx + 1) * hd, ctx,
                                           hd ** -0.5, P(self.attn_ws), self.attn_ws.numel(), P(o.x[0]),
                                           *self._next_kv(li), st),
                  "apb_attention_decode")
            o.run()   # resid += o(att); gate_up's input = fp16(resid * w)
            gu.run()  # scaled by the norm factor; GLU epilogue -> dn.x
            dn.run()  # resid += down(.); the next block's input = fp16(resid * w)
        check(lib.apb_rms_residual(P(self.resid), None, P(self.norm_w), P(self.hbuf), H, 1e-5, st),
              "apb_rms_residual")
        logits = self.hbuf @ self.lm_head.t()
        check(lib.apb_argmax_f16(P(logits), cfg.vocab, P(self.next_token), st), "apb_argmax_f16")

    def _next_kv(self, li):
        """The next block's cache for the attention kernel's L2 prefetch (none after the last)."""
        if li + 1 >= self.cfg.layers or not self.kv_prefetch:
            return None, None
        return dev.ptr(self.k_cache[li + 1]), dev.ptr(self.v_cache[li + 1])

    def capture(self, k: int):
        torch = dev.require_cuda()
        self._forward(k)  # warm-up: plans, kernel attributes, library workspaces
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            self._forward(k)
        self._graphs[k] = gr
        return gr

    def step(self, k: int):
        """Decode one token at bit-width k (graph replay once captured)."""
        gr = self._graphs.get(k)
        if gr is None:
            self._forward(k)
        else:
            gr.replay()
        return self.next_token

    def quantized_bytes(self, k: int) -> int:
        """Algorithmic bytes the quantized linears read per token."""
        tot = 0
        for blk in self.blocks:
            for p in blk.values():
                r, c = p.tensor.rows, p.tensor.cols
                tot += r * c * k // 8 + r * (1 << k) * 2 + c * 2 + r * 2
        return tot
