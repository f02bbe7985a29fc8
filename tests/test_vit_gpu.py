"""ViT encoder stage (ViT-L/32 family) vs a plain PyTorch fp32 restatement
(tests/vit_ref.py) on the same bf16 weights, synthetic patches and freeze masks: loss, and the
masked update of every parameter (frozen-in-every-microbatch units untouched)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _expand_unit_mask(frozen_bits: np.ndarray, ent: dict) -> np.ndarray:
    r, c = ent["rows"], ent["cols"]
    tn = ent["tiles_n"]
    tm = (r + 127) // 128
    bits = frozen_bits[ent["unit_offset"]:ent["unit_offset"] + ent["units"]].reshape(tm, tn)
    return np.kron((~bits).astype(np.float32), np.ones((128, 128), dtype=np.float32))[:r, :c]


def _run_and_compare(cuda, schedule, stages_per_rank, override, M=2, lr=0.5, seed=5, steps=1):
    import torch

    from gpu_util import device_view
    from llama_ref import unflatten
    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout
    from vit_ref import stage_loss, synthetic_patches

    shape = PRESETS["vit-tiny"]
    S = stages_per_rank
    tr = Trainer(shape, schedule, 1, S, M, lr=lr, seed=seed)
    tr.set_override(override)
    lays = [param_layout(shape, s, S) for s in range(1, S + 1)]
    bufs = [tr.stage_buffers(i) for i in range(S)]
    for b, lay in zip(bufs, lays):
        assert b["n_params"] == lay["n_params"] and b["n_units"] == lay["n_units"]
    theta0 = [device_view(b["master"], b["n_params"]).clone() for b in bufs]
    w0 = [device_view(b["weights"], b["n_params"], torch.bfloat16).clone() for b in bufs]
    rng = np.random.default_rng(2)
    T = shape.tokens
    tokens = np.zeros((M, T), dtype=np.int32)
    targets = rng.integers(0, shape.vocab, size=(M, T), dtype=np.int32)
    res = tr.step(1, tokens, targets)
    torch.cuda.synchronize()
    theta1 = [device_view(b["master"], b["n_params"]).clone() for b in bufs]
    frozen = [[pf.unpack_mask(mk, lays[i]["n_units"]) for mk in tr.last_masks(i)] for i in range(S)]

    params = {}
    for i in range(S):
        params.update({k: v.detach().clone().requires_grad_(True) for k, v in unflatten(w0[i].float(), lays[i]).items()})
    grads = {k: torch.zeros_like(v) for k, v in params.items()}
    losses = []
    pd = shape.patch_dim
    np_ = shape.seq - 1
    for m in range(M):
        for v in params.values():
            v.grad = None
        patches = synthetic_patches(seed, m + 1, shape.micro_batch * np_, pd).to(cuda)
        labels = torch.tensor(targets[m][: shape.micro_batch], device=cuda).long()
        loss = stage_loss(params, shape, range(shape.layers), patches, labels, True, True)
        loss.backward()
        losses.append(loss.item())
        for i in range(S):
            for ent in lays[i]["units"]:
                upd = torch.tensor(_expand_unit_mask(frozen[i][m], ent), device=cuda)
                grads[ent["name"]] += params[ent["name"]].grad * upd
            for ent in lays[i]["dense"]:
                grads[ent["name"]] += params[ent["name"]].grad
    assert abs(res["loss"] - np.mean(losses)) < 2e-2 * abs(np.mean(losses)), (res["loss"], losses)
    d_dev = {}
    for i in range(S):
        d_dev.update(unflatten(theta1[i] - theta0[i], lays[i]))
    all_frozen = [np.logical_and.reduce(frozen[i]) for i in range(S)]
    checked = 0
    for i in range(S):
        for ent in lays[i]["units"] + lays[i]["dense"]:
            name = ent["name"]
            exp = -(lr / M) * grads[name]
            got = d_dev[name]
            if ent["freezable"]:
                keep = torch.tensor(1 - _expand_unit_mask(all_frozen[i], ent), device=cuda).bool()
                assert torch.count_nonzero(got[keep]).item() == 0, name
            if exp.abs().max().item() == 0:
                continue
            rel = (got - exp).norm().item() / exp.norm().item()
            assert rel < 6e-2, (name, rel)
            checked += 1
    assert checked >= 20
    tr.close()


@pytest.mark.parametrize("override", [0.0, 0.5])
def test_vit_stage_matches_torch_reference(cuda, override):
    _run_and_compare(cuda, "gpipe", 1, override)


@pytest.mark.parametrize("schedule,stages_per_rank", [("interleaved-1f1b", 2), ("zbv-split", 2)])
def test_vit_multi_stage_matches_torch_reference(cuda, schedule, stages_per_rank):
    _run_and_compare(cuda, schedule, stages_per_rank, 0.5)


def test_vit_controller_plan_and_training(cuda):
    """Warm-up, monitoring, LP at T_m and the freeze ramp on the ViT stage; the loss decreases."""
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    tr = Trainer(PRESETS["vit-tiny"], "gpipe", 1, 1, 4, phases=(2, 6, 8, 14), r_max=0.8, lr=0.05, seed=3)
    losses = [tr.step(t)["loss"] for t in range(1, 15)]
    assert all(np.isfinite(losses))
    p = tr.get_plan()
    assert p is not None and p["ratios"].mean() <= 0.8 + 1e-6
    assert np.mean(losses[-3:]) < np.mean(losses[:3])
    tr.close()
