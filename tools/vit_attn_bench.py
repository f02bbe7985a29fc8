"""ViT short-sequence attention backward at the ViT-L/32 microbatch (64 images x 50 tokens, 16 heads of 64),
CUDA events on one B200: the kernel alone, with the fused qkv bias gradient, and the torch column sum it
replaces (the stage's former separate bias-gradient pass)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2602_05754_b200 import _native  # noqa: E402


def timed(fn, iters=50):
    for _ in range(5):
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
    lib = _native.device()
    B, S, nh, hd = int(os.environ.get("B", 64)), 50, 16, 64
    qkv = torch.randn(B * S, 3 * nh * hd, device="cuda").to(torch.bfloat16)
    dout = torch.randn(B * S, nh * hd, device="cuda").to(torch.bfloat16)
    out = torch.empty(B * S, nh * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * nh * S, device="cuda")
    dqkv = torch.empty_like(qkv)
    db = torch.zeros(3 * nh * hd, device="cuda")
    sc = 1.0 / math.sqrt(hd)
    st = torch.cuda.current_stream().cuda_stream
    _native.check(lib.pf_vit_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, hd, sc, st), "fwd")
    fwd = timed(lambda: lib.pf_vit_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, hd, sc, st))
    plain = timed(lambda: lib.pf_vit_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                              dqkv.data_ptr(), None, B, S, nh, hd, sc, st))
    fused = timed(lambda: lib.pf_vit_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                              dqkv.data_ptr(), db.data_ptr(), B, S, nh, hd, sc, st))
    colsum = timed(lambda: db.add_(dqkv.float().sum(0)))
    # bytes: qkv + dout read, dqkv written (bf16), lse read (D comes from P and dP: O is not read)
    nbytes = B * S * (3 * nh * hd * 2 * 2 + nh * hd * 2) + B * nh * S * 4
    print(f"B={B} S={S} nh={nh}: fwd {fwd * 1e3:.1f} us | bwd {plain * 1e3:.1f} us "
          f"({nbytes / (plain * 1e-3) / 1e9:.0f} GB/s) | bwd + fused bias grad {fused * 1e3:.1f} us | "
          f"torch column sum {colsum * 1e3:.1f} us")


if __name__ == "__main__":
    main()
