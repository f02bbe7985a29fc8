"""Per-tensor gradient error of the device stage step at the LLaMA-8B layer shapes (2 layers, 32768
vocab slice, 1 microbatch, nothing frozen) vs the faithful-bf16 torch reference and vs pure fp32;
wqkv split into its q / k / v row blocks.  python tools/northstar_diag.py [--model llama-8b]"""
import argparse
import dataclasses
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-8b")
    a = ap.parse_args()
    from gpu_util import device_view
    from llama_ref import stage_loss, unflatten
    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout

    kw = dict(layers=2, vocab=32768) if a.model == "llama-8b" else dict(layers=2)
    shape = dataclasses.replace(PRESETS[a.model], **kw)
    tr = Trainer(shape, "1f1b", 1, 1, 1, lr=0.5, seed=7)
    tr.set_override(0.0)
    lay = param_layout(shape, 1, 1)
    buf = tr.stage_buffers(0)
    n = buf["n_params"]
    rng = np.random.default_rng(11)
    tok = rng.integers(0, shape.vocab, size=(1, shape.tokens), dtype=np.int32)
    tgt = rng.integers(0, shape.vocab, size=(1, shape.tokens), dtype=np.int32)
    w0 = device_view(buf["weights"], n, torch.bfloat16).clone()
    tr.step(1, tok, tgt)
    torch.cuda.synchronize()
    g_dev = unflatten(device_view(buf["grad"], n).clone(), lay)
    refs = {}
    for faithful in (True, False):
        params = {k: v.detach().clone().requires_grad_(True) for k, v in unflatten(w0.float(), lay).items()}
        loss = stage_loss(params, shape, range(shape.layers), torch.tensor(tok[0], device="cuda").long(),
                          torch.tensor(tgt[0], device="cuda").long(), True, True, faithful=faithful)
        loss.backward()
        refs[faithful] = {k: v.grad.detach() for k, v in params.items()}
        del params
    nh, nkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim

    def rel(x, y):
        return (x - y).norm().item() / max(y.norm().item(), 1e-30)

    for name in sorted(g_dev):
        parts = {"all": slice(None)}
        if name.endswith("wqkv"):
            parts = {"q": slice(0, nh * hd), "k": slice(nh * hd, (nh + nkv) * hd), "v": slice((nh + nkv) * hd, None)}
        for pn, sl in parts.items():
            d, rf, r32 = g_dev[name][sl], refs[True][name][sl], refs[False][name][sl]
            print(f"{name:10s} {pn:3s} |g| {rf.norm().item():.3e}  dev-vs-faithful {rel(d, rf):.2e}  "
                  f"dev-vs-fp32 {rel(d, r32):.2e}  faithful-vs-fp32 {rel(rf, r32):.2e}", flush=True)
    tr.close()


if __name__ == "__main__":
    main()
