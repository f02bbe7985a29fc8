"""Masked dW (K3) throughput on the LLaMA-1B stage shapes: the 1-CTA unit-list kernel
(pf_gemm_dw_units over K5 lists) vs the CTA-pair kernel (pf_gemm_dw_pairs over K5p pair
lists), at a given frozen fraction. TF/s counts the unfrozen units' FLOPs only (padding
partners are not credited). CUDA events, live; prints one line per shape."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_05754_b200 import _native  # noqa: E402
from test_kernels_gpu import pair_list_ref, rowpair_list_ref  # noqa: E402

lib = _native.device()


def bench(name, T, O, I, frac, iters=20):
    tm, tn = -(-O // 128), -(-I // 128)
    U = tm * tn
    rng = np.random.default_rng(1)
    frozen = np.zeros(U, dtype=bool)
    frozen[rng.permutation(U)[:int(frac * U)]] = True
    units = [u for u in range(U) if not frozen[u]]
    plist = pair_list_ref(frozen, tm, tn)
    rlist = rowpair_list_ref(frozen, tm, tn)
    dY = torch.randn(T, O, device="cuda").to(torch.bfloat16)
    X = torch.randn(T, I, device="cuda").to(torch.bfloat16)
    G = torch.zeros(O, I, device="cuda")
    st = torch.zeros(U, dtype=torch.int32, device="cuda")
    ul = torch.tensor(units + [0], dtype=torch.int32, device="cuda")
    uc = torch.tensor([len(units)], dtype=torch.int32, device="cuda")
    pl = torch.tensor(plist + [0], dtype=torch.int32, device="cuda")
    pc = torch.tensor([len(plist)], dtype=torch.int32, device="cuda")
    rl = torch.tensor(rlist + [0, 0], dtype=torch.int32, device="cuda")
    rc_ = torch.tensor([len(rlist) // 2], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")

    def old(k):
        return lib.pf_gemm_dw_units(dY.data_ptr(), 1, dY.stride(0), X.data_ptr(), 1, X.stride(0), G.data_ptr(),
                                    G.stride(0), O, I, T, 1.0, ul.data_ptr(), uc.data_ptr(), U, st.data_ptr(), 0, k, s)

    def new(k):
        return lib.pf_gemm_dw_pairs(dY.data_ptr(), dY.stride(0), X.data_ptr(), X.stride(0), G.data_ptr(), G.stride(0),
                                    O, I, T, pl.data_ptr(), pc.data_ptr(), st.data_ptr(), 0, k, s)

    def rows(k):
        return lib.pf_gemm_dw_rowpairs(dY.data_ptr(), dY.stride(0), X.data_ptr(), X.stride(0), G.data_ptr(),
                                       G.stride(0), O, I, T, rl.data_ptr(), rc_.data_ptr(), st.data_ptr(), 0, k, s)

    out = []
    for fn in (old, new, rows):
        for k in range(3):
            assert fn(k + 1) == 0
        tot = 0.0
        for k in range(iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert fn(100 + k) == 0
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        ms = tot / iters
        out.append((2.0 * len(units) * 128 * 128 * T / (ms * 1e-3) / 1e12, ms))
    pad = sum(1 for u in plist if u < 0)
    print(f"{name:10s} {O}x{I} T={T} units {len(units)}/{U} pad {pad} | 1-CTA {out[0][0]:7.1f} TF/s "
          f"({out[0][1]:.3f} ms) | CTA pair {out[1][0]:7.1f} TF/s ({out[1][1]:.3f} ms) | row pair {out[2][0]:7.1f} "
          f"TF/s ({out[2][1]:.3f} ms)", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--frac", type=float, default=0.8)
    ap.add_argument("--only", nargs="*", default=None, help="shape names to run")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    T = 4096
    for name, O, I in [("gu", 16384, 2048), ("d", 2048, 8192), ("qkv", 3072, 2048), ("o", 2048, 2048),
                       ("lm", 128256, 2048), ("8b gu", 28672, 4096), ("8b d", 4096, 14336)]:
        if a.only is None or name in a.only:
            bench(name, T, O, I, a.frac, a.iters)
