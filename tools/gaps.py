"""Where the step time goes between kernels: per-action CUDA-event durations, the idle gaps between
consecutive actions, and the host time spent enqueueing a step vs its device time.

    python tools/gaps.py --model llama-1b --ratio 0.8
"""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-1b")
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--ratio", type=float, default=0.8)
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2602_05754_b200.engine import PRESETS, Trainer

    tr = Trainer(PRESETS[args.model], "gpipe", 1, 1, args.microbatches, lr=1e-4)
    tr.set_override(args.ratio)
    for t in range(1, 4):
        tr.step(t)
    torch.cuda.synchronize()
    for t in range(4, 4 + args.steps):
        w0 = time.perf_counter()
        r = tr.step(t)
        wall = (time.perf_counter() - w0) * 1e3
        start, end, kinds, mbs, stages = tr.action_times()
        gaps = start[1:] - end[:-1]
        busy = float(np.sum(end - start))
        print(f"step {t}: wall {wall:.2f} ms  batch {r['batch_ms']:.2f}  opt {r['optimizer_ms']:.2f}  "
              f"mask {r['mask_ms']:.2f}  sum(actions) {busy:.2f}  inter-action gaps {float(gaps.sum()):.3f} "
              f"(max {float(gaps.max()):.3f})")
    fw = [e - s for s, e, k in zip(start, end, kinds) if k == 0]
    bw = [e - s for s, e, k in zip(start, end, kinds) if k == 1]
    print(f"forward actions: mean {np.mean(fw):.3f} ms; backward: mean {np.mean(bw):.3f} ms")
    tr.close()


if __name__ == "__main__":
    main()
