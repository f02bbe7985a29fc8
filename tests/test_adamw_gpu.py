"""Masked AdamW step (§8(f) rank 4; the paper trains with AdamW, the reference sandbox only has SGD,
sandbox.cpp:250, so this is pinned against a plain torch fp64 AdamW restatement instead).

Semantics checked: g = G / M over the accumulated unfrozen-unit gradient; a unit frozen in every
microbatch of a step keeps theta, m, v and its step count; touched units use their own step count
for the bias correction; dense parameters (norm gains, embedding) step every time."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _unit_element_mask(lay: dict, n: int) -> np.ndarray:
    """Per-element unit index (-1 for dense / padding) of the stage's flat parameter buffer."""
    idx = np.full(n, -1, dtype=np.int64)
    for ent in lay["units"]:
        r, c = ent["rows"], ent["cols"]
        rb = np.arange(r)[:, None] // 128
        cb = np.arange(c)[None, :] // 128
        idx[ent["offset"]:ent["offset"] + r * c] = (ent["unit_offset"] + rb * ent["tiles_n"] + cb).reshape(-1)
    return idx


def _dense_mask(lay: dict, n: int) -> np.ndarray:
    d = np.zeros(n, dtype=bool)
    for ent in lay["dense"]:
        d[ent["offset"]:ent["offset"] + ent["rows"] * ent["cols"]] = True
    return d


@pytest.mark.parametrize("override", [0.0, 0.5])
def test_masked_adamw_matches_torch_restatement(cuda, override):
    import torch

    from gpu_util import device_view
    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout

    shape = PRESETS["tiny"]
    M, lr, b1, b2, eps, wd = 2, 1e-3, 0.9, 0.99, 1e-8, 0.1
    tr = Trainer(shape, "gpipe", 1, 1, M, lr=lr, seed=7, optimizer="adamw", betas=(b1, b2), eps=eps,
                 weight_decay=wd)
    tr.set_override(override)
    lay = param_layout(shape, 1, 1)
    buf = tr.stage_buffers(0)
    n, units = buf["n_params"], buf["n_units"]
    unit_of = torch.tensor(_unit_element_mask(lay, n), device=cuda)
    dense = torch.tensor(_dense_mask(lay, n), device=cuda)
    theta = device_view(buf["master"], n).double().clone()
    m = torch.zeros(n, dtype=torch.float64, device=cuda)
    v = torch.zeros_like(m)
    steps = torch.zeros(units, dtype=torch.int64, device=cuda)
    dense_steps = 0
    rng = np.random.default_rng(3)
    saw_frozen_unit = False
    for t in range(1, 4):
        tokens = rng.integers(0, shape.vocab, size=(M, shape.tokens), dtype=np.int32)
        targets = rng.integers(0, shape.vocab, size=(M, shape.tokens), dtype=np.int32)
        tr.step(t, tokens, targets)
        torch.cuda.synchronize()
        G = device_view(buf["grad"], n).double()
        stamps = device_view(buf["stamps"], units, torch.int32).long()
        touched_unit = stamps == t
        saw_frozen_unit |= bool((~touched_unit).any().item())
        steps = steps + touched_unit.long()
        dense_steps += 1
        upd = dense | ((unit_of >= 0) & touched_unit[unit_of.clamp(min=0)])
        k = torch.where(dense, torch.full_like(unit_of, dense_steps), steps[unit_of.clamp(min=0)]).double()
        g = G / M
        m_new = b1 * m + (1 - b1) * g
        v_new = b2 * v + (1 - b2) * g * g
        bc1, bc2 = 1 - b1 ** k, 1 - b2 ** k
        th_new = theta * (1 - lr * wd) - (lr / bc1) * m_new / (v_new.sqrt() / bc2.sqrt() + eps)
        theta = torch.where(upd, th_new, theta)
        m = torch.where(upd, m_new, m)
        v = torch.where(upd, v_new, v)

        st = tr.optim_state(0)
        dm = device_view(st["m"], n).double()
        dv = device_view(st["v"], n).double()
        dth = device_view(buf["master"], n).double()
        dsteps = device_view(st["unit_steps"], units, torch.int32).long()
        assert torch.equal(dsteps, steps)
        sel = (unit_of >= 0) | dense
        assert (dm - m)[sel].abs().max().item() <= 1e-5 * m[sel].abs().max().item() + 1e-12
        assert (dv - v)[sel].abs().max().item() <= 1e-5 * v[sel].abs().max().item() + 1e-16
        # theta: fp32 (two roundings of theta itself) vs fp64; the step of size ~lr to 1e-6 relative
        ratio = ((dth - theta).abs() / (3e-7 * theta.abs() + 1e-6 * lr)) * sel
        worst = int(ratio.argmax().item())
        assert ratio[worst].item() <= 1.0, (
            f"i={worst} unit={int(unit_of[worst])} theta={theta[worst].item():.9e} dev={dth[worst].item():.9e} "
            f"g={g[worst].item():.6e} m={m[worst].item():.6e} v={v[worst].item():.6e} k={k[worst].item()}")
        # frozen-in-every-microbatch units: theta, m, v untouched this step
        frozen_el = (unit_of >= 0) & ~touched_unit[unit_of.clamp(min=0)]
        if frozen_el.any():
            assert torch.equal(dm[frozen_el], m[frozen_el]) and torch.equal(dth[frozen_el], theta[frozen_el])
        theta, m, v = dth.clone(), dm.clone(), dv.clone()  # re-anchor on the device state (fp32 drift)
    if override > 0:
        assert saw_frozen_unit
    tr.close()


def test_adamw_bias_correction_first_step_is_sign_like(cuda):
    """With zero state the first AdamW step of an unfrozen element is lr * g / (|g| + eps) (+ decay)."""
    import torch

    from gpu_util import device_view
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    shape = PRESETS["tiny"]
    lr = 1e-2
    tr = Trainer(shape, "gpipe", 1, 1, 2, lr=lr, seed=1, optimizer="adamw", weight_decay=0.0)
    tr.set_override(0.0)
    buf = tr.stage_buffers(0)
    n = buf["n_params"]
    th0 = device_view(buf["master"], n).double().clone()
    tr.step(1)
    torch.cuda.synchronize()
    G = device_view(buf["grad"], n).double()
    d = device_view(buf["master"], n).double() - th0
    big = G.abs() > 1e-3 * G.abs().max()
    exp = -lr * torch.sign(G[big])
    assert (d[big] - exp).abs().max().item() < 1e-3 * lr
    tr.close()


def test_adamw_rejects_bad_config():
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    with pytest.raises(ValueError):
        Trainer(PRESETS["tiny"], optimizer="lion")
