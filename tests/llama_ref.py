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
               last: bool, x_in: torch.Tensor | None = None):
    """tokens/targets: [T] int64 of one microbatch. Returns (loss or output activations)."""
    B, S, h = shape.micro_batch, shape.seq, shape.hidden
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    x = params["emb"][tokens] if first else x_in
    for layer in layers:
        p = lambda n: params[f"l{layer}.{n}"]  # noqa: E731
        h1 = rms(x, p("g1"), shape.norm_eps)
        qkv = h1 @ p("wqkv").t()
        q = qkv[:, : nh * hd].view(B, S, nh, hd)
        k = qkv[:, nh * hd:(nh + nkv) * hd].view(B, S, nkv, hd)
        v = qkv[:, (nh + nkv) * hd:].view(B, S, nkv, hd)
        q, k = rope(q, S, shape.rope_theta), rope(k, S, shape.rope_theta)
        rep = nh // nkv
        k = k.repeat_interleave(rep, dim=2)
        v = v.repeat_interleave(rep, dim=2)
        att = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), is_causal=True)
        att = att.transpose(1, 2).reshape(B * S, nh * hd)
        x = x + att @ p("wo").t()
        h2 = rms(x, p("g2"), shape.norm_eps)
        gu = h2 @ p("wgu").t()
        gi = gate_index(shape.ffn, gu.device)
        g, u = gu[:, gi], gu[:, gi + 128]
        x = x + (F.silu(g) * u) @ p("wd").t()
    if not last:
        return x
    hf = rms(x, params["gf"], shape.norm_eps)
    logits = hf @ params["wlm"].t()
    return F.cross_entropy(logits, targets)
