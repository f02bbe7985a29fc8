"""RMSNorm backward (dx with residual + dg) and forward at LLaMA shapes through the C ABI: CUDA events, L2 flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2602_05754_b200 import _native  # noqa: E402
lib = _native.device()
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
for T, h, rows in [(4096, 4096, "1"), (4096, 4096, "2"), (2048, 5120, "1"), (2048, 5120, "2")]:
    os.environ["PF_NORM_ROWS"] = rows  # 1: row-block backward without prefetch, 0: warp-per-row (A/B)
    x = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    dy = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    res = torch.randn(T, h, device="cuda").to(torch.bfloat16)
    g = torch.ones(h, device="cuda").to(torch.bfloat16)
    rstd = torch.ones(T, device="cuda")
    dx = torch.empty_like(x)
    dg = torch.zeros(h, device="cuda")
    tot = 0.0
    for k in range(23):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert lib.pf_rmsnorm_bwd(x.data_ptr(), g.data_ptr(), rstd.data_ptr(), dy.data_ptr(), res.data_ptr(),
                                  dx.data_ptr(), dg.data_ptr(), T, h, s) == 0
        e1.record(); torch.cuda.synchronize()
        if k >= 3: tot += e0.elapsed_time(e1)
    us = tot / 20 * 1e3
    print(f"rmsnorm_bwd T={T} h={h} rows={rows}: {us:.1f} us, {4 * T * h * 2 / us / 1e3:.0f} GB/s (x, dy, residual in; dx out)")
    y = torch.empty_like(x)
    tot = 0.0
    for k in range(23):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert lib.pf_rmsnorm_fwd(x.data_ptr(), g.data_ptr(), y.data_ptr(), rstd.data_ptr(), T, h, 1e-5, s) == 0
        e1.record(); torch.cuda.synchronize()
        if k >= 3: tot += e0.elapsed_time(e1)
    us = tot / 20 * 1e3
    print(f"rmsnorm_fwd T={T} h={h} rows={rows}: {us:.1f} us, {2 * T * h * 2 / us / 1e3:.0f} GB/s (x in; y out)")
