"""qkv projection + RoPE at LLaMA-1B shapes: fused epilogue vs GEMM + rope_fwd (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2602_05754_b200 import _native  # noqa: E402
lib = _native.device()
T, S, nh, nkv, hd, D = 4096, 2048, 32, 8, 64, 2048
N = (nh + 2 * nkv) * hd
x = torch.randn(T, D, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, D, device="cuda") * 0.05).to(torch.bfloat16)
qkv = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
def timed(fn, iters=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3
fused = timed(lambda: lib.pf_gemm_rope(x.data_ptr(), D, w.data_ptr(), D, qkv.data_ptr(), T, S, nh, nkv, hd, D, 500000.0, s))
gemm = timed(lambda: lib.pf_gemm_bf16(x.data_ptr(), 0, D, w.data_ptr(), 0, D, qkv.data_ptr(), N, T, N, D, 1.0, 0, 512, None, 0, s))
rope = timed(lambda: lib.pf_rope_fwd(qkv.data_ptr(), T, S, nh, nkv, hd, 500000.0, s))
print(f"qkv + RoPE T={T} N={N} K={D}: fused {fused:.1f} us | gemm {gemm:.1f} + rope {rope:.1f} = {gemm + rope:.1f} us")
