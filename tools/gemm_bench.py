"""Throughput of the tcgen05 GEMM variants on the LLaMA stage shapes (CUDA events, live)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_05754_b200 import _native  # noqa: E402

lib = _native.device()


def bench(M, N, K, a_mn, b_mn, bn, epi=0, iters=20):
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi in (2, 3) else torch.bfloat16)
    st = torch.zeros(((M + 127) // 128) * ((N + 127) // 128), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def call():
        rc = lib.pf_gemm_bf16(A.data_ptr(), a_mn, A.stride(0), B.data_ptr(), b_mn, B.stride(0), C.data_ptr(), N, M, N,
                              K, 1.0, epi, bn, st.data_ptr(), 1, s)
        assert rc == 0, rc

    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return 2.0 * M * N * K / (ms * 1e-3) / 1e12, ms


if __name__ == "__main__":
    T = 4096
    shapes = [("qkv fwd", T, 3072, 2048, 0, 0), ("o fwd", T, 2048, 2048, 0, 0), ("gu fwd", T, 16384, 2048, 0, 0),
              ("d fwd", T, 2048, 8192, 0, 0), ("lm fwd", T, 128256, 2048, 0, 0), ("gu dX", T, 2048, 16384, 0, 1),
              ("d dX", T, 8192, 2048, 0, 1), ("qkv dX", T, 2048, 3072, 0, 1), ("lm dX", T, 2048, 128256, 0, 1),
              ("gu dW", 16384, 2048, T, 1, 1), ("8b gu fwd", T, 28672, 4096, 0, 0), ("8b d dX", T, 14336, 4096, 0, 1)]
    for name, M, N, K, a_mn, b_mn in shapes:
        row = [name, f"{M}x{N}x{K}"]
        for bn in (256, 512) if not a_mn else (128,):
            try:
                tf, ms = bench(M, N, K, a_mn, b_mn, bn, epi=2 if a_mn else 0)
                row.append(f"bn{bn}: {tf:7.1f} TF/s ({ms:.3f} ms)")
            except AssertionError as e:
                row.append(f"bn{bn}: err {e}")
        print(" | ".join(row), flush=True)
