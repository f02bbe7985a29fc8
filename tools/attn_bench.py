"""Times the hand-written flash attention (flash_attn.cu) forward and backward at the LLaMA layer
shapes with CUDA events, next to torch's cuDNN SDPA on the same shapes (for comparison only).

    python tools/attn_bench.py [--iters 20]
"""
import argparse
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05754_b200 import _native  # noqa: E402

SHAPES = {"llama-8b": (2, 2048, 32, 8, 128), "llama-13b": (1, 2048, 40, 40, 128), "llama-1b": (2, 2048, 32, 8, 64)}


def timeit(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--shapes", default="llama-8b,llama-13b,llama-1b")
    a = ap.parse_args()
    lib = _native.device()
    for name in a.shapes.split(","):
        B, S, nh, nkv, hd = SHAPES[name]
        T, W = B * S, (nh + 2 * nkv) * hd
        qkv = torch.randn(T, W, device="cuda").bfloat16()
        dout = (torch.randn(T, nh * hd, device="cuda") * 0.1).bfloat16()
        out = torch.empty(T, nh * hd, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(B, nh, S, device="cuda")
        dqkv = torch.empty_like(qkv)
        scale = hd ** -0.5
        st = torch.cuda.current_stream().cuda_stream
        fwd = lambda: lib.pf_flash_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, nkv, hd, scale, 1, st)  # noqa
        bwd = lambda: lib.pf_flash_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),  # noqa
                                            dqkv.data_ptr(), B, S, nh, nkv, hd, scale, 1, 500000.0, st)
        assert fwd() == 0 and bwd() == 0
        f_ms, b_ms = timeit(fwd, a.iters), timeit(bwd, a.iters)
        if os.environ.get("PF_ATTN_PROF", "0") in ("1", "3"):
            import ctypes

            import numpy as np

            buf = np.zeros(32, dtype=np.uint64)
            lib.pf_flash_attn_prof(buf.ctypes.data_as(ctypes.c_void_p))  # reset
            fwd()
            torch.cuda.synchronize()
            lib.pf_flash_attn_prof(buf.ctypes.data_as(ctypes.c_void_p))
            print(f"{name} fwd CTA0 cycles: mma wait_p {buf[0]} wait_kv {buf[1]} total {buf[2]} | softmax wait_s {buf[3]} "
                  f"bar {buf[4]} compute {buf[7]} total {buf[5]} | producer wait_empty {buf[6]}")
            bwd()
            torch.cuda.synchronize()
            lib.pf_flash_attn_prof(buf.ctypes.data_as(ctypes.c_void_p))
            print(f"{name} bwd CTA0 cycles: mma wait_qdo {buf[8]} wait_dqempty {buf[9]} wait_p {buf[10]} total {buf[11]} | "
                  f"softmax wait_s {buf[12]} bar {buf[17]} compute {buf[14]} (tld {buf[18]} bar+math {buf[19]} tst {buf[20]} "
                  f"st_wait {buf[21]}) wait_dq {buf[13]} drain {buf[15]} (tld {buf[22]}) total {buf[16]}")
        flops_f = 4.0 * B * S * S * nh * hd / 2  # causal
        line = f"{name:9s} ours: fwd {f_ms * 1e3:7.1f} us ({flops_f / f_ms / 1e9:6.1f} TF/s)  bwd {b_ms * 1e3:7.1f} us " \
               f"({2.5 * flops_f / b_ms / 1e9:6.1f} TF/s)"
        try:
            x = qkv.view(B, S, nh + 2 * nkv, hd)
            q = x[:, :, :nh].transpose(1, 2).contiguous().requires_grad_(True)
            k = x[:, :, nh:nh + nkv].repeat_interleave(nh // nkv, 2).transpose(1, 2).contiguous().requires_grad_(True)
            v = x[:, :, nh + nkv:].repeat_interleave(nh // nkv, 2).transpose(1, 2).contiguous().requires_grad_(True)
            do = dout.view(B, S, nh, hd).transpose(1, 2).contiguous()
            from torch.nn.attention import SDPBackend, sdpa_kernel

            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
                cf = timeit(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True), a.iters)
                cb = timeit(lambda: torch.autograd.grad(o, (q, k, v), do, retain_graph=True), a.iters)
            line += f"   | cuDNN SDPA (K/V expanded): fwd {cf * 1e3:7.1f} us  bwd {cb * 1e3:7.1f} us"
        except Exception as e:  # pragma: no cover
            line += f"   | cuDNN SDPA unavailable: {e}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
