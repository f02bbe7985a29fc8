"""One o-proj-shaped CTA-pair GEMM (4096 x 2048 x 2048) under a given PF_GEMM_STREAMK mode (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2602_05754_b200 import _native  # noqa: E402
lib = _native.device()
M, N, K = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 2048, 2048))]
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    assert lib.pf_gemm_bf16(A.data_ptr(), 0, K, B.data_ptr(), 0, K, C.data_ptr(), N, M, N, K, 1.0, 0, 512, None, 0, s) == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    lib.pf_gemm_bf16(A.data_ptr(), 0, K, B.data_ptr(), 0, K, C.data_ptr(), N, M, N, K, 1.0, 0, 512, None, 0, s)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 50
print(f"mode {os.environ.get('PF_GEMM_STREAMK', 'default')} {M}x{N}x{K}: {ms * 1e3:.1f} us {2 * M * N * K / ms / 1e9:.0f} TF/s")
