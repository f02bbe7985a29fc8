"""One or more stage steps of a north-star-shaped slice with timings (hang / regression probe).

    python tools/step_probe.py [--model llama-8b] [--layers 2] [--vocab 32768] [--M 2] [--ratio 0.5] [--steps 2]
"""
import argparse
import dataclasses
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-8b")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--vocab", type=int, default=32768)
    ap.add_argument("--M", type=int, default=2)
    ap.add_argument("--ratio", type=float, default=0.5)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--schedule", default="1f1b")
    a = ap.parse_args()
    import torch

    from paper_2602_05754_b200.engine import PRESETS, Trainer

    shape = PRESETS[a.model]
    kw = {}
    if a.layers:
        kw["layers"] = a.layers
    if a.vocab:
        kw["vocab"] = a.vocab
    shape = dataclasses.replace(shape, **kw)
    tr = Trainer(shape, a.schedule, 1, 1, a.M, lr=1e-4, seed=1)
    tr.set_override(a.ratio)
    for t in range(1, a.steps + 1):
        w0 = time.perf_counter()
        r = tr.step(t)
        torch.cuda.synchronize()
        print(f"step {t}: loss {r['loss']:.4f} batch {r['batch_ms']:.2f} ms wall {1e3 * (time.perf_counter() - w0):.1f} ms",
              flush=True)
    tr.close()
    print("ok", flush=True)


if __name__ == "__main__":
    main()
