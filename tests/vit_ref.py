"""TEST INFRASTRUCTURE: plain PyTorch fp32 restatement of the ViT encoder stage (VitStage,
csrc/device/vit_stage.cpp) and of its synthetic patch input, for parity tests."""
import numpy as np
import torch
import torch.nn.functional as F

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def synthetic_patches(seed: int, microbatch: int, rows: int, cols: int) -> torch.Tensor:
    """launch_synthetic_patches (vit_kernels.cu): splitmix64 of the element index, seeded with
    seed * golden + microbatch (uint64 wrap), mapped to [-1, 1) and rounded to bf16."""
    s = (seed * GOLDEN + microbatch) & MASK64
    i = np.arange(rows * cols, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(s) + (i + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    v = (z >> np.uint64(40)).astype(np.float64) * 2.0 ** -23 - 1.0
    return torch.tensor(v.astype(np.float32)).to(torch.bfloat16).float().view(rows, cols)


def stage_loss(params: dict, shape, layers, patches, labels, first: bool, last: bool, x_in=None):
    """Forward of layers [b, e) (+ patch embedding on the first stage, head + mean CE on the last)."""
    B, S, h = shape.micro_batch, shape.seq, shape.hidden
    nh = shape.n_heads
    hd = shape.head_dim
    eps = shape.norm_eps
    p = params.__getitem__
    if first:
        E = patches @ p("patch_w").t() + p("patch_b")
        tok = torch.cat([p("cls").expand(B, 1, h), E.view(B, S - 1, h)], dim=1) + p("pos").view(1, S, h)
        x = tok.reshape(B * S, h)
    else:
        x = x_in
    for i in layers:
        q = lambda n: p(f"l{i}.{n}")  # noqa: E731
        h1 = F.layer_norm(x, (h,), q("ln1g"), q("ln1b"), eps)
        qkv = h1 @ q("wqkv").t() + q("bqkv")
        qh, kh, vh = (qkv[:, j * h:(j + 1) * h].view(B, S, nh, hd).transpose(1, 2) for j in range(3))
        att = F.scaled_dot_product_attention(qh, kh, vh, is_causal=False)
        att = att.transpose(1, 2).reshape(B * S, h)
        x = x + att @ q("wo").t() + q("bo")
        h2 = F.layer_norm(x, (h,), q("ln2g"), q("ln2b"), eps)
        x = x + F.gelu(h2 @ q("w1").t() + q("b1")) @ q("w2").t() + q("b2")
    if not last:
        return x
    xc = x.view(B, S, h)[:, 0]
    hc = F.layer_norm(xc, (h,), p("lnfg"), p("lnfb"), eps)
    logits = hc @ p("head").t() + p("headb")
    return F.cross_entropy(logits, labels)
