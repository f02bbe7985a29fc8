"""ViT MLP GEMMs with the GELU epilogues vs the plain CTA-pair GEMM of the same shape (T = 3200 / 25600,
h = 1024, mlp = 4096), CUDA events over back-to-back launches."""
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
    return e0.elapsed_time(e1) / iters * 1e3


def ck(rc):
    assert rc == 0, rc


for T in (3200, 25600):
    h, f = 1024, 4096
    x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    w1 = (0.05 * torch.randn(f, h, device="cuda")).to(torch.bfloat16)   # [ffn][h]
    b1 = torch.randn(f, device="cuda").to(torch.bfloat16)
    w2 = (0.05 * torch.randn(h, f, device="cuda")).to(torch.bfloat16)   # [h][ffn]
    dy = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    pre = torch.empty(T, f, device="cuda", dtype=torch.bfloat16)
    act = torch.empty_like(pre)
    dpre = torch.empty_like(pre)
    db = torch.zeros(f, device="cuda")
    fl = 2.0 * T * f * h
    plain_f = timed(lambda: ck(lib.pf_gemm_bf16(x.data_ptr(), 0, h, w1.data_ptr(), 0, h, pre.data_ptr(), f, T, f, h, 1.0,
                                                0, 512, None, 0, s)))
    gelu = timed(lambda: ck(lib.pf_gemm_gelu(x.data_ptr(), h, w1.data_ptr(), h, b1.data_ptr(), pre.data_ptr(),
                                             act.data_ptr(), T, f, h, s)))
    plain_b = timed(lambda: ck(lib.pf_gemm_bf16(dy.data_ptr(), 0, h, w2.data_ptr(), 1, f, dpre.data_ptr(), f, T, f, h,
                                                1.0, 0, 512, None, 0, s)))
    dgelu = timed(lambda: ck(lib.pf_gemm_dgelu(dy.data_ptr(), h, w2.data_ptr(), f, pre.data_ptr(), dpre.data_ptr(),
                                               None, T, f, h, s)))
    dgelu_db = timed(lambda: ck(lib.pf_gemm_dgelu(dy.data_ptr(), h, w2.data_ptr(), f, pre.data_ptr(), dpre.data_ptr(),
                                                  db.data_ptr(), T, f, h, s)))
    print(f"T={T}: fc1 plain {plain_f:.1f} us ({fl / plain_f / 1e6:.0f} TF/s) | +bias+GELU {gelu:.1f} us | "
          f"fc2 dX plain {plain_b:.1f} us ({fl / plain_b / 1e6:.0f} TF/s) | +GELU' {dgelu:.1f} us | +GELU' +db {dgelu_db:.1f} us",
          flush=True)
