"""One profiled training step of the stage engine (for ncu; capture window = cudaProfilerStart/Stop).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file out.csv \
        python tools/profile_step.py --model llama-1b --ratio 0.8
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-1b")
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--ratio", type=float, default=0.8)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import torch

    from paper_2602_05754_b200.engine import PRESETS, Trainer

    tr = Trainer(PRESETS[args.model], "gpipe", 1, 1, args.microbatches, lr=1e-4)
    tr.set_override(args.ratio)
    for t in range(1, args.warmup + 1):
        tr.step(t)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    r = tr.step(args.warmup + 1)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print({k: r[k] for k in ("batch_ms", "optimizer_ms", "mean_ratio", "loss")})
    tr.close()


if __name__ == "__main__":
    main()
