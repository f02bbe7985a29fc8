"""Stage step at the north-star layer shapes vs the plain PyTorch fp32 restatement (tests/llama_ref.py).

BASELINE configs[2] (LLaMA-8B: h 4096, head_dim 128, GQA 32/8, 2 x 2048 tokens per microbatch) and
configs[3] (LLaMA-13B: h 5120, MHA 40/40, head_dim 128, vocab 32000, 1 x 2048 tokens), each as a
2-layer stage that is both first and last (embedding, 2 decoder layers, final norm, LM head; the
8B head is a 32768-row slice of its 128256-row vocabulary). Three consecutive training steps with
half of every cell's 128x128 units frozen (exact-count masks), 2 microbatches per step.

Per step, on the same bf16 weights and masks the device used:
  * loss: |loss_dev - loss_ref| <= 2e-3 * |loss_ref|;
  * every parameter tensor's accumulated gradient G = sum_m U_m . g_m (the device's fp32 grad
    buffer over the units touched this step) and its update theta += -(lr / M) G
    (sandbox.cpp:221,250; the reference update rounded in fp32 like the device's):
    ||x_dev - x_ref|| <= tol * ||x_ref|| (relative Frobenius norm, per tensor) against the
    bf16-faithful reference, tol = max(2e-2, 1.1 x that tensor's bf16 noise floor), the floor
    being the faithful reference's own distance from the pure fp32 gradient (above 2e-2 only for
    the top layer's q / k / g1 gradients: ~3 %);
  * and the device gradient is no farther from the pure fp32 gradient than the faithful bf16
    evaluation is (<= 1.1 x floor + 2e-3);
  * units frozen in every microbatch are bit-for-bit untouched;
  * the bf16 GEMM copy equals bf16(master) after the step.
The reference rounds activations (and their gradients) to bf16 where the device stores them in bf16
(llama_ref.stage_loss faithful=True); its math is fp32. The transformer math has no counterpart in
the reference repo ("parity unpinned by the reference"), so this is the stated tolerance.
"""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_TENSOR = 2e-2
TOL_LOSS = 2e-3

CASES = {
    "llama-8b": dict(layers=2, vocab=32768),
    "llama-13b": dict(layers=2),
}


def _expand_unit_mask(frozen_bits: np.ndarray, ent: dict) -> np.ndarray:
    r, c = ent["rows"], ent["cols"]
    tn = ent["tiles_n"]
    tm = (r + 127) // 128
    bits = frozen_bits[ent["unit_offset"]:ent["unit_offset"] + ent["units"]].reshape(tm, tn)
    return np.kron((~bits).astype(np.float32), np.ones((128, 128), dtype=np.float32))[:r, :c]


@pytest.mark.parametrize("model", ["llama-8b", "llama-13b"])
def test_stage_steps_north_star_shapes(cuda, model):
    import torch

    from gpu_util import device_view
    from llama_ref import stage_loss, unflatten
    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout

    shape = dataclasses.replace(PRESETS[model], **CASES[model])
    M, lr, steps = 2, 0.5, 3
    tr = Trainer(shape, "1f1b", 1, 1, M, lr=lr, seed=7)
    tr.set_override(0.5)
    lay = param_layout(shape, 1, 1)
    buf = tr.stage_buffers(0)
    assert buf["n_params"] == lay["n_params"] and buf["n_units"] == lay["n_units"]
    n = buf["n_params"]
    rng = np.random.default_rng(11)
    T = shape.tokens
    worst = {}
    for t in range(1, steps + 1):
        tokens = rng.integers(0, shape.vocab, size=(M, T), dtype=np.int32)
        targets = rng.integers(0, shape.vocab, size=(M, T), dtype=np.int32)
        theta0 = device_view(buf["master"], n).clone()
        w0 = device_view(buf["weights"], n, torch.bfloat16).clone()
        res = tr.step(t, tokens, targets)
        torch.cuda.synchronize()
        theta1 = device_view(buf["master"], n).clone()
        w1 = device_view(buf["weights"], n, torch.bfloat16).clone()
        g_dev_all = unflatten(device_view(buf["grad"], n).clone(), lay)
        assert torch.equal(w1, theta1.bfloat16()), "bf16 weights != bf16(master)"
        masks = tr.last_masks(0)
        frozen = [pf.unpack_mask(masks[m], lay["n_units"]) for m in range(M)]
        assert abs(res["mean_ratio"] - 0.5) < 0.01

        refs = {}
        for faithful in (True, False):
            params = {k: v.detach().clone().requires_grad_(True) for k, v in unflatten(w0.float(), lay).items()}
            grads = {k: torch.zeros_like(v) for k, v in params.items()}
            losses = []
            for m in range(M):
                for v in params.values():
                    v.grad = None
                loss = stage_loss(params, shape, range(shape.layers), torch.tensor(tokens[m], device=cuda).long(),
                                  torch.tensor(targets[m], device=cuda).long(), True, True, faithful=faithful)
                loss.backward()
                losses.append(loss.item())
                for ent in lay["units"]:
                    upd = torch.tensor(_expand_unit_mask(frozen[m], ent), device=cuda)
                    grads[ent["name"]] += params[ent["name"]].grad * upd
                for ent in lay["dense"]:
                    grads[ent["name"]] += params[ent["name"]].grad
            del params
            refs[faithful] = (grads, losses)
        grads, losses = refs[True]
        grads32 = refs[False][0]
        ref_loss = float(np.mean(losses))
        assert abs(res["loss"] - ref_loss) <= TOL_LOSS * abs(ref_loss), (t, res["loss"], ref_loss)

        th0 = unflatten(theta0, lay)
        d_dev = unflatten(theta1 - theta0, lay)
        all_frozen = np.logical_and.reduce(frozen)
        # the device's SGD in fp32 (kernels.cu masked_sgd_units / sgd_dense): theta += (-(lr/M)) * G
        step_scale = torch.tensor(-(lr * (1.0 / M)), dtype=torch.float32, device=cuda)
        checked = 0
        for ent in lay["units"] + lay["dense"]:
            name = ent["name"]
            got = d_dev[name]
            touched = torch.ones_like(got, dtype=torch.bool)
            if ent["freezable"]:
                frozen_all = torch.tensor(_expand_unit_mask(all_frozen, ent), device=cuda) == 0
                assert torch.count_nonzero(got[frozen_all]).item() == 0, (t, name)
                touched = ~frozen_all
            if grads[name].abs().max().item() == 0:
                continue
            # (1) the accumulated gradient sum_m U_m . g_m itself (grad buffer, units touched this step)
            ref_g, dev_g, g32 = grads[name][touched], g_dev_all[name][touched], grads32[name][touched]
            rel_g = (dev_g - ref_g).norm().item() / ref_g.norm().item()
            # bf16 noise floor of this tensor: how far the faithful bf16 evaluation itself lands from
            # the exact fp32 gradient (rounding flips at the bf16 storage points compound through the
            # layers: 1.4-3.1 % at these shapes, tools/northstar_diag.py)
            floor = (ref_g - g32).norm().item() / g32.norm().item()
            rel_32 = (dev_g - g32).norm().item() / g32.norm().item()
            tol = max(TOL_TENSOR, 1.1 * floor)
            # (2) the parameter update, with the reference update rounded like the device's (the fp32
            # subtraction theta1 - theta0 of a ~1e-8 update to a ~2e-2 weight is exact only to an ulp)
            exp = (th0[name] + step_scale * grads[name]) - th0[name]
            rel = (got - exp).norm().item() / exp.norm().item()
            worst[name] = max(worst.get(name, 0.0), rel, rel_g)
            assert rel_g <= tol, (t, name, "grad", rel_g, floor)
            assert rel <= tol, (t, name, "update", rel, floor)
            # no noisier than a bf16-faithful evaluation: as close to the exact fp32 gradient
            assert rel_32 <= 1.1 * floor + 2e-3, (t, name, "grad vs fp32", rel_32, floor)
            checked += 1
        assert checked >= 12
        del grads, d_dev, g_dev_all, th0
    print(f"{model}: worst per-tensor relative error over {steps} steps:",
          {k: f"{v:.2e}" for k, v in sorted(worst.items(), key=lambda kv: -kv[1])[:6]})
    tr.close()
