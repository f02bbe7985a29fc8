"""K7 attention (flash_attn.cu, hand-written tcgen05/TMEM/TMA kernels) vs plain PyTorch fp32.

Shapes: the north-star configurations (LLaMA-8B 32/8 heads and LLaMA-13B 40/40 heads at head_dim
128, LLaMA-1B 32/8 at head_dim 64, S = 2048), the tiny test preset, and a bidirectional
(ViT-style) case. The reference is fp32 scaled-dot-product attention on the same bf16 q, k, v
(and, for the backward, the same bf16 dO), with RoPE applied in fp32 where the kernel applies its
backward. Stated tolerances (relative Frobenius norm per tensor): out 1e-2, LSE 1e-4 absolute
(log2 units), dq / dk / dv 2e-2 -- the kernel's P and dS are bf16 MMA operands, as in every flash
attention.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def lib():
    from paper_2602_05754_b200 import _native

    return _native.device()


def chk(rc, what=""):
    assert rc == 0, f"{what}: {rc} {lib().pf_engine_last_error().decode()}"


def sp():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


CASES = [
    # B, S, nh, nkv, hd, causal, rope_theta
    (2, 2048, 32, 8, 128, True, 500000.0),   # LLaMA-8B layer (configs[2])
    (1, 2048, 40, 40, 128, True, 10000.0),   # LLaMA-13B layer (configs[3])
    (2, 2048, 32, 8, 64, True, 500000.0),    # LLaMA-1B layer (configs[1])
    (2, 128, 4, 2, 64, True, 500000.0),      # tiny preset
    (1, 384, 6, 3, 128, True, 0.0),          # 3 blocks, GQA 2, no RoPE
    (4, 256, 8, 8, 64, False, 0.0),          # bidirectional (ViT-style, S % 128 == 0)
]


@pytest.mark.parametrize("B,S,nh,nkv,hd,causal,theta", CASES)
def test_flash_attention_matches_fp32_reference(cuda, B, S, nh, nkv, hd, causal, theta):
    import torch
    import torch.nn.functional as F

    from llama_ref import rope

    T = B * S
    W = (nh + 2 * nkv) * hd
    g = torch.Generator(device="cpu").manual_seed(B * 1000 + S + nh + hd)
    qkv = (torch.randn(T, W, generator=g) * 1.0).bfloat16().cuda()
    dout = (torch.randn(T, nh * hd, generator=g) * 0.1).bfloat16().cuda()
    out = torch.empty(T, nh * hd, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(B, nh, S, dtype=torch.float32, device=cuda)
    scale = hd ** -0.5
    chk(lib().pf_flash_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, nkv, hd, scale, int(causal),
                                sp()), "fwd")
    dqkv = torch.empty_like(qkv)
    chk(lib().pf_flash_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dqkv.data_ptr(), B, S,
                                nh, nkv, hd, scale, int(causal), theta, sp()), "bwd")
    torch.cuda.synchronize()

    # fp32 reference: q, k are the rotated activations the kernel read; the gradients w.r.t. the
    # un-rotated q, k follow through the fp32 rotation (the kernel's RoPE backward)
    x = qkv.float().view(B, S, nh + 2 * nkv, hd)
    q0 = x[:, :, :nh].clone()
    k0 = x[:, :, nh:nh + nkv].clone()
    v = x[:, :, nh + nkv:].clone().requires_grad_(True)
    if theta > 0:
        # the kernel's inputs are already rotated; a rotation by -angle recovers pre-RoPE inputs
        # whose forward rotation reproduces them (to fp32 rounding)
        qp = _unrope(q0, S, theta).requires_grad_(True)
        kp = _unrope(k0, S, theta).requires_grad_(True)
        q, k = rope(qp, S, theta), rope(kp, S, theta)
    else:
        qp = q0.requires_grad_(True)
        kp = k0.requires_grad_(True)
        q, k = qp, kp
    rep = nh // nkv
    ke, ve = k.repeat_interleave(rep, 2), v.repeat_interleave(rep, 2)
    ref = F.scaled_dot_product_attention(q.transpose(1, 2), ke.transpose(1, 2), ve.transpose(1, 2), is_causal=causal,
                                         scale=scale)
    ref = ref.transpose(1, 2).reshape(T, nh * hd)
    ref.backward(dout.float())
    got = out.float()
    assert _rel(got, ref) <= 1e-2, _rel(got, ref)

    s = torch.einsum("bqhd,bkhd->bhqk", q.detach(), ke.detach()) * scale
    if causal:
        s = s.masked_fill(torch.ones(S, S, dtype=torch.bool, device=cuda).triu(1), float("-inf"))
    lse_ref = torch.logsumexp(s, -1) / np.log(2.0)
    assert (lse - lse_ref).abs().max().item() <= 1e-3 * max(1.0, lse_ref.abs().max().item())

    d = dqkv.float().view(B, S, nh + 2 * nkv, hd)
    errs = {"dq": _rel(d[:, :, :nh], qp.grad), "dk": _rel(d[:, :, nh:nh + nkv], kp.grad),
            "dv": _rel(d[:, :, nh + nkv:], v.grad)}
    print(f"B{B} S{S} nh{nh} nkv{nkv} hd{hd} causal={causal}: out {_rel(got, ref):.2e}", {k: f"{e:.2e}" for k, e in errs.items()})
    for name, e in errs.items():
        assert e <= 2e-2, (name, e)


def _unrope(x, S, theta):
    """Inverse of llama_ref.rope (rotation by -angle), fp32."""
    import torch

    d = x.shape[-1]
    half = d // 2
    j = torch.arange(half, dtype=torch.float64, device=x.device)
    inv = theta ** (-2.0 * j / d)
    pos = torch.arange(S, dtype=torch.float64, device=x.device)
    ang = pos[:, None] * inv[None, :]
    c = torch.cos(ang).float()[None, :, None, :]
    s = torch.sin(ang).float()[None, :, None, :]
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * c + b * s, b * c - a * s], dim=-1)


def test_flash_attention_in_place_dqkv(cuda):
    """The stage writes dq|dk|dv over qkv itself: same result as a separate output buffer."""
    import torch

    B, S, nh, nkv, hd = 2, 512, 8, 2, 128
    T, W = B * S, (nh + 2 * nkv) * hd
    g = torch.Generator(device="cpu").manual_seed(5)
    qkv = torch.randn(T, W, generator=g).bfloat16().cuda()
    dout = (torch.randn(T, nh * hd, generator=g) * 0.1).bfloat16().cuda()
    out = torch.empty(T, nh * hd, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(B, nh, S, dtype=torch.float32, device=cuda)
    scale = hd ** -0.5
    chk(lib().pf_flash_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, nkv, hd, scale, 1, sp()))
    sep = torch.empty_like(qkv)
    chk(lib().pf_flash_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), sep.data_ptr(), B, S,
                                nh, nkv, hd, scale, 1, 500000.0, sp()))
    inplace = qkv.clone()
    chk(lib().pf_flash_attn_bwd(inplace.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                inplace.data_ptr(), B, S, nh, nkv, hd, scale, 1, 500000.0, sp()))
    torch.cuda.synchronize()
    # dq sums fp32 partials by atomics (order-dependent); dk, dv are exact
    d_sep, d_in = sep.float().view(T, -1, hd), inplace.float().view(T, -1, hd)
    assert torch.equal(d_sep[:, nh:], d_in[:, nh:])
    assert _rel(d_in[:, :nh], d_sep[:, :nh]) <= 1e-2


def test_flash_attention_rejects_unsupported_shapes(cuda):
    import torch

    buf = torch.zeros(1 << 20, dtype=torch.bfloat16, device=cuda)
    lse = torch.zeros(1 << 16, dtype=torch.float32, device=cuda)
    assert lib().pf_flash_attn_fwd(buf.data_ptr(), buf.data_ptr(), lse.data_ptr(), 1, 100, 2, 2, 64, 0.1, 1, sp()) == 4
    assert lib().pf_flash_attn_fwd(buf.data_ptr(), buf.data_ptr(), lse.data_ptr(), 1, 128, 2, 2, 96, 0.1, 1, sp()) == 4
    assert lib().pf_flash_attn_fwd(buf.data_ptr(), buf.data_ptr(), lse.data_ptr(), 1, 128, 3, 2, 64, 0.1, 1, sp()) == 4


@pytest.mark.parametrize("hd,causal", [(128, True), (64, True), (128, False)])
def test_flash_forward_lane_divergent_rescale(cuda, hd, causal):
    """Rows of one warp whose running max grows past the lazy-rescale threshold at different key
    blocks (alternating query rows see a +-12 log2-unit spike in key block 1): the O rescale must
    be warp-uniform (tcgen05.ld / st are warp-collective; a lane-divergent TMEM access hung the
    LLaMA-8B step). Forward output and LSE vs fp32."""
    import torch
    import torch.nn.functional as F

    B, S, nh, nkv = 1, 512, 4, 2
    T, W = B * S, (nh + 2 * nkv) * hd
    g = torch.Generator(device="cpu").manual_seed(77)
    x = torch.randn(T, nh + 2 * nkv, hd, generator=g) * 0.5
    sign = torch.where(torch.arange(S) % 2 == 0, 1.0, -1.0)
    x[:, :nh, 0] = 5.0 * sign[:, None]           # q: +-5 along dim 0, alternating rows
    x[128:256, nh:nh + nkv, 0] = 2.2 * hd ** 0.5  # k: spike along dim 0 in key block 1
    qkv = x.reshape(T, W).bfloat16().cuda()
    out = torch.empty(T, nh * hd, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(B, nh, S, dtype=torch.float32, device=cuda)
    scale = hd ** -0.5
    chk(lib().pf_flash_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, nkv, hd, scale, int(causal),
                                sp()), "fwd")
    torch.cuda.synchronize()
    xf = qkv.float().view(B, S, nh + 2 * nkv, hd)
    q, k, v = xf[:, :, :nh], xf[:, :, nh:nh + nkv], xf[:, :, nh + nkv:]
    rep = nh // nkv
    ke, ve = k.repeat_interleave(rep, 2), v.repeat_interleave(rep, 2)
    ref = F.scaled_dot_product_attention(q.transpose(1, 2), ke.transpose(1, 2), ve.transpose(1, 2), is_causal=causal,
                                         scale=scale).transpose(1, 2).reshape(T, nh * hd)
    assert _rel(out, ref) <= 1e-2, _rel(out, ref)
    s = torch.einsum("bqhd,bkhd->bhqk", q, ke) * scale
    if causal:
        s = s.masked_fill(torch.ones(S, S, dtype=torch.bool, device=cuda).triu(1), float("-inf"))
    lse_ref = torch.logsumexp(s, -1) / np.log(2.0)
    assert (lse - lse_ref).abs().max().item() <= 1e-3 * max(1.0, lse_ref.abs().max().item())


_BWD_PATH_SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2602_05754_b200 import _native
lib = _native.device()
B, S, nh, nkv, hd = 2, 512, 8, 2, {hd}
T, W = B * S, (nh + 2 * nkv) * hd
g = torch.Generator().manual_seed(3)
qkv = torch.randn(T, W, generator=g).bfloat16().cuda()
dout = (torch.randn(T, nh * hd, generator=g) * 0.1).bfloat16().cuda()
out = torch.empty(T, nh * hd, dtype=torch.bfloat16, device='cuda')
lse = torch.empty(B, nh, S, device='cuda')
st = torch.cuda.current_stream().cuda_stream
assert lib.pf_flash_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, nkv, hd, hd ** -0.5, 1, st) == 0
d = torch.empty_like(qkv)
assert lib.pf_flash_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), d.data_ptr(), B, S, nh, nkv,
                             hd, hd ** -0.5, 1, 500000.0, st) == 0
torch.cuda.synchronize()
np.save(sys.argv[1], d.float().cpu().numpy())
"""


@pytest.mark.parametrize("hd", [128, 64])
def test_flash_backward_separate_dq_matches_fused(cuda, tmp_path, hd):
    """PF_ATTN_BWD=2 computes dQ in its own kernel (no fp32 atomics) before the dK / dV kernel; the
    default keeps dQ inside the dK / dV kernel. dk / dv come from the same code (bitwise equal); dq
    differs only by fp32 summation order."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("2", "1"):
        f = tmp_path / f"d{mode}.npy"
        env = dict(os.environ, PF_ATTN_BWD=mode)
        subprocess.run([sys.executable, "-c", _BWD_PATH_SNIPPET.replace("{hd}", str(hd)), str(f)], cwd=root, env=env,
                       check=True, timeout=300)
        outs[mode] = np.load(f)
    nh, nkv = 8, 2
    a = outs["2"].reshape(outs["2"].shape[0], nh + 2 * nkv, hd)
    b = outs["1"].reshape(a.shape)
    assert np.array_equal(a[:, nh:], b[:, nh:])
    dq_a, dq_b = a[:, :nh], b[:, :nh]
    assert np.linalg.norm(dq_a - dq_b) <= 1e-2 * np.linalg.norm(dq_b)


_FWD_PATH_SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2602_05754_b200 import _native
lib = _native.device()
B, S, nh, nkv, hd = 2, 640, 8, 2, {hd}
T, W = B * S, (nh + 2 * nkv) * hd
g = torch.Generator().manual_seed(9)
qkv = torch.randn(T, W, generator=g).bfloat16().cuda()
out = torch.empty(T, nh * hd, dtype=torch.bfloat16, device='cuda')
lse = torch.empty(B, nh, S, device='cuda')
st = torch.cuda.current_stream().cuda_stream
assert lib.pf_flash_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, nkv, hd, hd ** -0.5, {causal}, st) == 0
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([out.float().cpu().numpy().ravel(), lse.cpu().numpy().ravel()]))
"""


@pytest.mark.parametrize("hd,causal", [(128, 1), (64, 1), (128, 0)])
def test_flash_forward_two_tile_matches_one_tile(cuda, tmp_path, hd, causal):
    """The default two-tile (ping-pong) forward and the one-tile forward (PF_ATTN_FWD=1) on the same
    inputs; S = 640 is 5 query blocks, so the last CTA of the two-tile kernel has no tile B."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for mode in ("2", "1"):
        f = tmp_path / f"o{mode}.npy"
        code = _FWD_PATH_SNIPPET.replace("{hd}", str(hd)).replace("{causal}", str(causal))
        subprocess.run([sys.executable, "-c", code, str(f)], cwd=root, env=dict(os.environ, PF_ATTN_FWD=mode),
                       check=True, timeout=300)
        outs[mode] = np.load(f)
    a, b = outs["2"], outs["1"]
    n_out = 2 * 640 * 8 * hd
    assert np.linalg.norm(a[:n_out] - b[:n_out]) <= 1e-2 * np.linalg.norm(b[:n_out])
    assert np.abs(a[n_out:] - b[n_out:]).max() <= 1e-3 * max(1.0, np.abs(b[n_out:]).max())
