"""Cross-entropy kernel time at the LLaMA LM-head shape (T=4096, V=128256), CUDA events, L2 flushed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2602_05754_b200 import _native  # noqa: E402
lib = _native.device()
s = torch.cuda.current_stream().cuda_stream
for T, V in [(4096, 128256), (2048, 32000)]:
    src = (3 * torch.randn(T, V, device="cuda")).to(torch.bfloat16)
    lg = src.clone()
    tgt = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    ls = torch.zeros(1, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
    tot = 0.0
    for k in range(13):
        lg.copy_(src); flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert lib.pf_cross_entropy(lg.data_ptr(), tgt.data_ptr(), ls.data_ptr(), T, V, 1.0 / T, 1.0 / T, s) == 0
        e1.record(); torch.cuda.synchronize()
        if k >= 3: tot += e0.elapsed_time(e1)
    ms = tot / 10
    print(f"CE T={T} V={V}: {ms * 1e3:.1f} us, {2 * T * V * 2 / ms / 1e6:.0f} GB/s (read + write once)")
