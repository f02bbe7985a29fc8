"""TEST INFRASTRUCTURE: plain-PyTorch fp32 reference of one LLaMA-shaped pipeline stage.

Used only by the GPU parity tests to check the hand-written stage step
(paper_2602_05754_b200/csrc/device/stage.cpp). It reads the same flat parameter
buffer layout (engine.param_layout) and recomputes loss and gradients in fp32
with the bf16-rounded weights the device GEMMs consume. The reference repo has
no transformer math, so this part of parity is "unpinned by the reference"
(SURVEY 8(c)).
"""
from __future__ import annotations

import torch
import torch.nn.functional as F


class _RoundBF16(torch.autograd.Function):
    """bf16 storage point: the value and its gradient are both rounded to bf16, as the device
    stores that activation and its gradient in bf16 between kernels."""

    @staticmethod
    def forward(ctx, x):
        return x.bfloat16().float()

    @staticmethod
    def backward(ctx, g):
        return g.bfloat16().float()


class _FlashRefAttention(torch.autograd.Function):
    """Causal softmax attention at flash-attention storage precision (faithful mode): scores and
    softmax in fp32, P rounded to bf16 for the P.V and P^T.dO products, dS = P (dP - D) rounded to
    bf16 for the dQ and dK products, D = rowsum(dO * O) on the bf16-stored output. All products
    accumulate in fp32. q, k, v: [B, H, S, D] (k, v already expanded to H heads)."""

    @staticmethod
    def forward(ctx, q, k, v):
        scale = q.shape[-1] ** -0.5
        s = (q @ k.transpose(-1, -2)) * scale
        S = s.shape[-1]
        causal = torch.ones(S, S, dtype=torch.bool, device=s.device).triu(1)
        s = s.masked_fill(causal, float("-inf"))
        p = torch.exp(s - torch.logsumexp(s, -1, keepdim=True))
        del s
        pb = p.bfloat16().float()
        o = pb @ v
        ctx.save_for_backward(q, k, v, p, o.bfloat16().float())
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, p, o = ctx.saved_tensors
        scale = q.shape[-1] ** -0.5
        dv = p.bfloat16().float().transpose(-1, -2) @ do
        dp = do @ v.transpose(-1, -2)
        ds = p * (dp - (do * o).sum(-1, keepdim=True))
        del dp
        dsb = ds.bfloat16().float()
        dq = (dsb @ k) * scale
        dk = (dsb.transpose(-1, -2) @ q) * scale
        return dq, dk, dv


class _RoundFwdBF16(torch.autograd.Function):
    """bf16 rounding of the value only: the gradient passes through in fp32 (the device rounds it
    later, at an upstream storage point)."""

    @staticmethod
    def forward(ctx, x):
        return x.bfloat16().float()

    @staticmethod
    def backward(ctx, g):
        return g


def _q(x, faithful: bool):
    return _RoundBF16.apply(x) if faithful else x


def unflatten(flat: torch.Tensor, layout: dict) -> dict:
    out = {}
    for ent in layout["units"] + layout["dense"]:
        n = ent["rows"] * ent["cols"]
        t = flat[ent["offset"]:ent["offset"] + n]
        out[ent["name"]] = t.view(ent["rows"], ent["cols"]) if ent["rows"] > 1 else t.view(ent["cols"])
    return out


def rms(x, g, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def rope(x, seq, theta):
    # x [B, S, H, D] rotate-half
    d = x.shape[-1]
    half = d // 2
    j = torch.arange(half, dtype=torch.float64, device=x.device)
    inv = theta ** (-2.0 * j / d)
    pos = torch.arange(seq, dtype=torch.float64, device=x.device)
    ang = pos[:, None] * inv[None, :]
    c = torch.cos(ang).float()[None, :, None, :]
    s = torch.sin(ang).float()[None, :, None, :]
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * c - b * s, b * c + a * s], dim=-1)


def gate_index(ffn, device=None):
    """Columns of gate j in the gate|up output: rows of Wgu interleave 128-blocks
    [gate b | up b] (kernels.cu gate_col); up j is 128 columns further."""
    import torch

    j = torch.arange(ffn, device=device)
    return (j // 128) * 256 + j % 128


def stage_loss(params: dict, shape, layers: range, tokens: torch.Tensor, targets: torch.Tensor, first: bool,
               last: bool, x_in: torch.Tensor | None = None, faithful: bool = False):
    """tokens/targets: [T] int64 of one microbatch. Returns (loss or output activations).

    faithful=True rounds every activation (and its gradient) to bf16 where the device stage
    stores it in bf16 between kernels (stage.cpp forward/backward): x, h1, qkv (after RoPE),
    the attention output, x2, h2, gate|up, the SwiGLU output, hf and the logits. The math between
    those points stays fp32, as in the device's fp32-accumulating kernels; the attention keeps
    flash attention's bf16 P and dS operands (_FlashRefAttention)."""
    B, S, h = shape.micro_batch, shape.seq, shape.hidden
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    Q = lambda t: _q(t, faithful)  # noqa: E731
    x = params["emb"][tokens] if first else x_in
    x = Q(x)
    for layer in layers:
        p = lambda n: params[f"l{layer}.{n}"]  # noqa: E731
        h1 = Q(rms(x, p("g1"), shape.norm_eps))
        qkv = Q(h1 @ p("wqkv").t())
        q = qkv[:, : nh * hd].view(B, S, nh, hd)
        k = qkv[:, nh * hd:(nh + nkv) * hd].view(B, S, nkv, hd)
        v = qkv[:, (nh + nkv) * hd:].view(B, S, nkv, hd)
        # the device rotates the bf16 q / k in fp32 and rounds the result (qkv GEMM epilogue); its
        # backward rotates the fp32 dq / dk accumulators and rounds once, into dqkv (flash_attn.cu)
        Qf = (lambda t: _RoundFwdBF16.apply(t)) if faithful else (lambda t: t)  # noqa: E731
        q, k = Qf(rope(q, S, shape.rope_theta)), Qf(rope(k, S, shape.rope_theta))
        rep = nh // nkv
        k = k.repeat_interleave(rep, dim=2)
        v = v.repeat_interleave(rep, dim=2)
        if faithful:
            att = _FlashRefAttention.apply(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2))
        else:
            att = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                                 is_causal=True)
        att = Q(att.transpose(1, 2).reshape(B * S, nh * hd))
        x = Q(x + att @ p("wo").t())
        h2 = Q(rms(x, p("g2"), shape.norm_eps))
        gu = Q(h2 @ p("wgu").t())
        gi = gate_index(shape.ffn, gu.device)
        g, u = gu[:, gi], gu[:, gi + 128]
        x = Q(x + Q(F.silu(g) * u) @ p("wd").t())
    if not last:
        return x
    hf = Q(rms(x, params["gf"], shape.norm_eps))
    logits = Q(hf @ params["wlm"].t())
    return F.cross_entropy(logits, targets)
