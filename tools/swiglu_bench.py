"""SwiGLU fused into the CTA-pair GEMM epilogues vs GEMM + separate kernel (CUDA events, live)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2602_05754_b200 import _native  # noqa: E402

lib = _native.device()


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def ok(rc):
    assert rc == 0, rc


for T, D, ffn in [(4096, 2048, 8192), (4096, 4096, 14336)]:
    s = torch.cuda.current_stream().cuda_stream
    h = torch.randn(T, D, device="cuda").to(torch.bfloat16)
    w = (torch.randn(2 * ffn, D, device="cuda") * 0.05).to(torch.bfloat16)
    wd = (torch.randn(D, ffn, device="cuda") * 0.05).to(torch.bfloat16)
    dy = torch.randn(T, D, device="cuda").to(torch.bfloat16)
    gu = torch.empty(T, 2 * ffn, device="cuda", dtype=torch.bfloat16)
    a = torch.empty(T, ffn, device="cuda", dtype=torch.bfloat16)
    da = torch.empty(T, ffn, device="cuda", dtype=torch.bfloat16)
    dgu = torch.empty_like(gu)
    fl_f = 2.0 * T * 2 * ffn * D
    fl_b = 2.0 * T * ffn * D
    t_gemm = timed(lambda: ok(lib.pf_gemm_bf16(h.data_ptr(), 0, D, w.data_ptr(), 0, D, gu.data_ptr(), 2 * ffn, T,
                                               2 * ffn, D, 1.0, 0, 512, None, 0, s)))
    t_act = timed(lambda: ok(lib.pf_swiglu_fwd(gu.data_ptr(), a.data_ptr(), T, ffn, s)))
    t_fused = timed(lambda: ok(lib.pf_gemm_swiglu(h.data_ptr(), D, w.data_ptr(), D, gu.data_ptr(), a.data_ptr(), T,
                                                  ffn, D, s)))
    print(f"fwd T={T} D={D} ffn={ffn}: gemm {t_gemm:.3f} ms ({fl_f / t_gemm / 1e9:.0f} TF/s) + swiglu {t_act:.3f} ms"
          f" = {t_gemm + t_act:.3f} | fused {t_fused:.3f} ms ({fl_f / t_fused / 1e9:.0f} TF/s)", flush=True)
    t_gemm = timed(lambda: ok(lib.pf_gemm_bf16(dy.data_ptr(), 0, D, wd.data_ptr(), 1, ffn, da.data_ptr(), ffn, T,
                                               ffn, D, 1.0, 0, 512, None, 0, s)))
    t_act = timed(lambda: ok(lib.pf_swiglu_bwd(gu.data_ptr(), da.data_ptr(), dgu.data_ptr(), T, ffn, s)))
    t_fused = timed(lambda: ok(lib.pf_gemm_dswiglu(dy.data_ptr(), D, wd.data_ptr(), ffn, gu.data_ptr(),
                                                   dgu.data_ptr(), T, ffn, D, s)))
    print(f"bwd T={T} D={D} ffn={ffn}: gemm {t_gemm:.3f} ms ({fl_b / t_gemm / 1e9:.0f} TF/s) + dswiglu {t_act:.3f} ms"
          f" = {t_gemm + t_act:.3f} | fused {t_fused:.3f} ms ({fl_b / t_fused / 1e9:.0f} TF/s)", flush=True)
