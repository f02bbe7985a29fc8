"""LLaMA-8B N = 4096 GEMM shapes (3.46 CTA-pair waves of 256 x 256 tiles): stream-K modes A/B.
    PF_GEMM_STREAMK=0|1|2 python tools/gemm_bench8b.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gemm_bench import bench  # noqa: E402

T = 4096
for name, M, N, K, b_mn in [("gu dX", T, 4096, 28672, 1), ("d fwd", T, 4096, 14336, 0), ("qkv dX", T, 4096, 6144, 1),
                            ("o dX", T, 4096, 4096, 1), ("o fwd", T, 4096, 4096, 0), ("lm dX", T, 4096, 128256, 1)]:
    tf, ms = bench(M, N, K, 0, b_mn, 512)
    print(f"mode {os.environ.get('PF_GEMM_STREAMK', 'default')} {name:7s} {M}x{N}x{K}: {tf:7.1f} TF/s ({ms:.3f} ms)",
          flush=True)
