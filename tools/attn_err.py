"""Numerical error of the hand-written flash attention vs torch's bf16 SDPA (cuDNN / flash), both
against the same fp32 reference, at the LLaMA layer shapes (no RoPE: q, k, v as given).

    python tools/attn_err.py
"""
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05754_b200 import _native  # noqa: E402


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm()).item()


def main():
    lib = _native.device()
    for (B, S, nh, nkv, hd, std) in [(2, 2048, 32, 8, 128, 1.0), (1, 2048, 40, 40, 128, 1.0), (2, 2048, 32, 8, 128, 1.6),
                                     (2, 2048, 32, 8, 64, 1.0)]:
        T, W = B * S, (nh + 2 * nkv) * hd
        g = torch.Generator(device="cpu").manual_seed(1)
        qkv = (torch.randn(T, W, generator=g) * std).bfloat16().cuda()
        dout = (torch.randn(T, nh * hd, generator=g) * 0.1).bfloat16().cuda()
        out = torch.empty(T, nh * hd, dtype=torch.bfloat16, device="cuda")
        lse = torch.empty(B, nh, S, device="cuda")
        dqkv = torch.empty_like(qkv)
        sc = hd ** -0.5
        st = torch.cuda.current_stream().cuda_stream
        assert lib.pf_flash_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, nkv, hd, sc, 1, st) == 0
        assert lib.pf_flash_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dqkv.data_ptr(),
                                     B, S, nh, nkv, hd, sc, 1, 0.0, st) == 0
        x = qkv.view(B, S, nh + 2 * nkv, hd)
        rep = nh // nkv

        def run(dtype):
            q = x[:, :, :nh].to(dtype).transpose(1, 2).contiguous().requires_grad_(True)
            k = x[:, :, nh:nh + nkv].to(dtype).transpose(1, 2).contiguous().requires_grad_(True)
            v = x[:, :, nh + nkv:].to(dtype).transpose(1, 2).contiguous().requires_grad_(True)
            o = F.scaled_dot_product_attention(q, k.repeat_interleave(rep, 1), v.repeat_interleave(rep, 1),
                                               is_causal=True, scale=sc)
            o.backward(dout.view(B, S, nh, hd).transpose(1, 2).to(dtype))
            return (o.transpose(1, 2).reshape(T, -1), q.grad.transpose(1, 2).reshape(T, -1),
                    k.grad.transpose(1, 2).reshape(T, -1), v.grad.transpose(1, 2).reshape(T, -1))

        ref = run(torch.float32)
        lib_bf = run(torch.bfloat16)
        d = dqkv.view(T, nh + 2 * nkv, hd)
        ours = (out, d[:, :nh].reshape(T, -1), d[:, nh:nh + nkv].reshape(T, -1), d[:, nh + nkv:].reshape(T, -1))
        names = ("out", "dq", "dk", "dv")
        print(f"B{B} S{S} nh{nh}/{nkv} hd{hd} std{std}: ours " +
              " ".join(f"{n} {rel(a, r):.2e}" for n, a, r in zip(names, ours, ref)) + " | torch bf16 " +
              " ".join(f"{n} {rel(a, r):.2e}" for n, a, r in zip(names, lib_bf, ref)), flush=True)


if __name__ == "__main__":
    main()
