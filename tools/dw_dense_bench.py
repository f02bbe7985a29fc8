"""Dense-cell dW at the LLaMA-8B layer shapes: row-pair kernel (every unit listed) vs the 256 x 256
CTA-pair dense kernel, CUDA events, T = 4096.  python tools/dw_dense_bench.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_05754_b200 import _native  # noqa: E402


def main():
    lib = _native.device()
    st = torch.cuda.current_stream().cuda_stream
    T = 4096
    for name, O, I in [("qkv", 6144, 4096), ("o", 4096, 4096), ("gu", 28672, 4096), ("d", 4096, 14336)]:
        tm, tn = O // 128, I // 128
        dY = torch.randn(T, O, device="cuda").bfloat16()
        X = torch.randn(T, I, device="cuda").bfloat16()
        G = torch.zeros(O, I, device="cuda")
        stamps = torch.zeros(tm * tn, dtype=torch.int32, device="cuda")
        ents = []
        for r in range(tm):
            for c in range(0, tn, 2):
                ents += [r * tn + c, r * tn + c + 1 if c + 1 < tn else -1]
        el = torch.tensor(ents + [0, 0], dtype=torch.int32, device="cuda")
        cnt = torch.tensor([len(ents) // 2], dtype=torch.int32, device="cuda")
        flops = 2.0 * T * O * I
        res = {}
        for kind in ("rows", "dense"):
            def run():
                if kind == "rows":
                    return lib.pf_gemm_dw_rowpairs(dY.data_ptr(), O, X.data_ptr(), I, G.data_ptr(), I, O, I, T,
                                                   el.data_ptr(), cnt.data_ptr(), stamps.data_ptr(), 0, 1, st)
                return lib.pf_gemm_dw_dense(dY.data_ptr(), O, X.data_ptr(), I, G.data_ptr(), I, O, I, T,
                                            stamps.data_ptr(), 0, 1, st)
            assert run() == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            res[kind] = (ms, flops / ms / 1e9)
        print(f"{name:4s} {O}x{I} T={T}: rows {res['rows'][0] * 1e3:7.1f} us ({res['rows'][1]:6.1f} TF/s) | "
              f"dense {res['dense'][0] * 1e3:7.1f} us ({res['dense'][1]:6.1f} TF/s)", flush=True)


if __name__ == "__main__":
    main()
