"""Device timeline of one training step (torch.profiler / CUPTI activity records, no serialisation):
sum of kernel busy time vs the step's device span, and the idle gaps between consecutive kernels,
bucketed. Answers "how much of the step is launch / dependency bubbles" without nsys.

    python tools/timeline_gaps.py --model llama-1b --ratio 0.8
"""
from __future__ import annotations

import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-1b")
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--ratio", type=float, default=0.8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--top", type=int, default=12)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2602_05754_b200.engine import PRESETS, Trainer

    tr = Trainer(PRESETS[args.model], "gpipe", 1, 1, args.microbatches, lr=1e-4)
    tr.set_override(args.ratio)
    for t in range(1, args.warmup + 1):
        tr.step(t)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = tr.step(args.warmup + 1)
        torch.cuda.synchronize()
    kern = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
            and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
    kern.sort(key=lambda e: e.time_range.start)
    t0, t1 = kern[0].time_range.start, max(e.time_range.end for e in kern)
    busy = sum(e.time_range.end - e.time_range.start for e in kern)
    gaps = collections.Counter()
    gap_us = collections.defaultdict(float)
    by_prev = collections.defaultdict(float)
    end = kern[0].time_range.end
    for a, b in zip(kern, kern[1:]):
        g = b.time_range.start - max(end, a.time_range.end)
        end = max(end, a.time_range.end)
        if g <= 0:
            continue
        k = "<2us" if g < 2 else "2-5us" if g < 5 else "5-20us" if g < 20 else "20-100us" if g < 100 else ">=100us"
        gaps[k] += 1
        gap_us[k] += g
        by_prev[b.name[:70]] += g
    span = t1 - t0
    print(f"step batch_ms {r['batch_ms']:.2f} | device span {span / 1e3:.2f} ms | kernel busy {busy / 1e3:.2f} ms "
          f"({busy / span:.1%}) | {len(kern)} kernels | idle {(span - busy) / 1e3:.2f} ms")
    for k in ("<2us", "2-5us", "5-20us", "20-100us", ">=100us"):
        print(f"  gaps {k:>8}: {gaps[k]:5d}  total {gap_us[k] / 1e3:7.2f} ms")
    print("idle before (top kernels):")
    for name, g in sorted(by_prev.items(), key=lambda kv: -kv[1])[:args.top]:
        print(f"  {g / 1e3:7.2f} ms  {name}")
    tr.close()


if __name__ == "__main__":
    main()
