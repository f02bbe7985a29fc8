"""LayerNorm forward / fused backward (residual, dg, db, dsum) at the ViT-L/32 microbatch (T = 3200, h = 1024)
through the C ABI: CUDA events, back-to-back launches (the step's inputs are L2-resident: 6.5 MB each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_05754_b200 import _native  # noqa: E402

lib = _native.device()
s = torch.cuda.current_stream().cuda_stream


def timed(fn, iters=100):
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


for T, h in [(3200, 1024), (25600, 1024)]:
    x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    dy = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    res = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    g = torch.ones(h, device="cuda").to(torch.bfloat16)
    b = torch.zeros(h, device="cuda").to(torch.bfloat16)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    mean, rstd = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
    dg, db, dsum = (torch.zeros(h, device="cuda") for _ in range(3))
    fwd = timed(lambda: lib.pf_layernorm_fwd(x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
                                             rstd.data_ptr(), T, h, 1e-6, s))
    bwd = timed(lambda: lib.pf_layernorm_bwd(x.data_ptr(), g.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                             dy.data_ptr(), res.data_ptr(), dx.data_ptr(), dg.data_ptr(), db.data_ptr(),
                                             dsum.data_ptr(), T, h, s))
    print(f"T={T} h={h}: fwd {fwd:.1f} us ({2 * T * h * 2 / fwd / 1e3:.0f} GB/s) | bwd {bwd:.1f} us "
          f"({4 * T * h * 2 / bwd / 1e3:.0f} GB/s: x, dy, residual in, dx out)", flush=True)
