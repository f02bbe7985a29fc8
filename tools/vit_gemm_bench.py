"""The ViT-L/32 microbatch GEMMs (T = 3200 tokens, h = 1024, mlp 4096) through pf_gemm_bf16 (CTA-pair
kernel, plain bf16 store), CUDA events over back-to-back launches: TF/s per shape and the tile-wave
count (256 x 256 tiles over 74 CTA pairs)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_05754_b200 import _native  # noqa: E402

lib = _native.device()
s = torch.cuda.current_stream().cuda_stream


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


T = int(os.environ.get("T", 3200))
shapes = [("qkv fwd", T, 3072, 1024, 0), ("o fwd", T, 1024, 1024, 0), ("fc1 fwd", T, 4096, 1024, 0),
          ("fc2 fwd", T, 1024, 4096, 0), ("qkv dX", T, 1024, 3072, 1), ("o dX", T, 1024, 1024, 1),
          ("fc1 dX", T, 1024, 4096, 1), ("fc2 dX", T, 4096, 1024, 1)]
for name, M, N, K, bmn in shapes:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    # fwd: W stored [N][K]; dX: W stored [K][N] (read MN-major)
    w = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).to(torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ldb = N if bmn else K
    row = []
    for bn in (512, 256, 128):
        ms = timed(lambda: _native.check(lib.pf_gemm_bf16(a.data_ptr(), 0, K, w.data_ptr(), bmn, ldb, c.data_ptr(), N,
                                                          M, N, K, 1.0, 0, bn, None, 0, s), name))
        row.append(f"bn{bn} {ms * 1e3:6.1f} us {2 * M * N * K / ms / 1e9:5.0f} TF/s")
    tiles = math.ceil(M / 256) * math.ceil(N / 256)
    print(f"{name:8s} {M}x{N}x{K} ({tiles / 74:.2f} pair waves): " + " | ".join(row), flush=True)
