"""Stage step (forward, masked backward, masked optimizer) vs a plain PyTorch fp32 reference,
and the Alg. 1 controller driving it (phases, monitoring -> LP plan -> bit-exact masks)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _expand_unit_mask(frozen_bits: np.ndarray, ent: dict) -> np.ndarray:
    """Per-element update mask (1 = updated) of one matrix from the stage's unit bits."""
    r, c = ent["rows"], ent["cols"]
    tn = ent["tiles_n"]
    tm = (r + 127) // 128
    bits = frozen_bits[ent["unit_offset"]:ent["unit_offset"] + ent["units"]].reshape(tm, tn)
    upd = (~bits).astype(np.float32)
    return np.kron(upd, np.ones((128, 128), dtype=np.float32))[:r, :c]


@pytest.mark.parametrize("override,dw", [(0.0, "rows"), (0.5, "rows"), (0.5, "units"), (0.5, "pairs")])
def test_stage_step_matches_torch_reference(cuda, override, dw, monkeypatch):
    """One stage step vs an fp32 torch restatement on the same bf16 weights and masks, with each
    masked-dW kernel (row pairs: the default; 1-CTA units; CTA-pair column pairs)."""
    import torch

    monkeypatch.setenv("PF_DW_KERNEL", dw)
    from gpu_util import device_view
    from llama_ref import stage_loss, unflatten
    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout

    shape = PRESETS["tiny"]
    M, lr = 2, 0.5
    tr = Trainer(shape, "gpipe", 1, 1, M, lr=lr, seed=3)
    tr.set_override(override)
    lay = param_layout(shape, 1, 1)
    buf = tr.stage_buffers(0)
    assert buf["n_params"] == lay["n_params"] and buf["n_units"] == lay["n_units"]
    n = buf["n_params"]
    theta0 = device_view(buf["master"], n).clone()
    w0 = device_view(buf["weights"], n, torch.bfloat16).clone()
    rng = np.random.default_rng(0)
    T = shape.tokens
    tokens = rng.integers(0, shape.vocab, size=(M, T), dtype=np.int32)
    targets = rng.integers(0, shape.vocab, size=(M, T), dtype=np.int32)
    res = tr.step(1, tokens, targets)
    torch.cuda.synchronize()
    theta1 = device_view(buf["master"], n).clone()
    masks = tr.last_masks(0)
    frozen = [pf.unpack_mask(masks[m], lay["n_units"]) for m in range(M)]
    assert abs(res["mean_ratio"] - override) < 0.01

    # fp32 reference on the same bf16 weights
    params = {k: v.detach().clone().requires_grad_(True) for k, v in unflatten(w0.float(), lay).items()}
    grads = {k: torch.zeros_like(v) for k, v in params.items()}
    losses = []
    for m in range(M):
        for v in params.values():
            v.grad = None
        loss = stage_loss(params, shape, range(shape.layers), torch.tensor(tokens[m], device=cuda).long(),
                          torch.tensor(targets[m], device=cuda).long(), True, True, faithful=True)
        loss.backward()
        losses.append(loss.item())
        for ent in lay["units"]:
            upd = torch.tensor(_expand_unit_mask(frozen[m], ent), device=cuda)
            grads[ent["name"]] += params[ent["name"]].grad * upd
        for ent in lay["dense"]:
            grads[ent["name"]] += params[ent["name"]].grad
    assert abs(res["loss"] - np.mean(losses)) < 2e-2 * abs(np.mean(losses))

    d_dev = unflatten(theta1 - theta0, lay)
    all_frozen = np.logical_and.reduce(frozen)
    checked = 0
    for ent in lay["units"] + lay["dense"]:
        name = ent["name"]
        exp = -(lr / M) * grads[name]
        got = d_dev[name]
        if ent["freezable"]:
            mask_all = torch.tensor(1 - _expand_unit_mask(all_frozen, ent), device=cuda).bool()
            # units frozen in every microbatch are not updated at all (sandbox.cpp:250)
            assert torch.count_nonzero(got[mask_all]).item() == 0, name
        if exp.abs().max().item() == 0:
            continue
        rel = (got - exp).norm().item() / exp.norm().item()
        assert rel < 6e-2, (name, rel)
        checked += 1
    assert checked >= 10
    tr.close()


@pytest.mark.parametrize("schedule,stages_per_rank",
                         [("interleaved-1f1b", 2), ("interleaved-1f1b", 4), ("zbv", 2), ("zbv-split", 2)])
def test_multi_stage_rank_matches_torch_reference(cuda, schedule, stages_per_rank):
    """Several virtual stages on one GPU: activations and gradients hand over between local
    stages; the update must equal the single-model reference. zbv-split runs each cell's dW as
    a separate W action after its B (gradients kept in the slot), which must not change it."""
    import torch

    from gpu_util import device_view
    from llama_ref import stage_loss, unflatten
    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout

    shape = PRESETS["tiny"]
    M, lr, S = 2, 0.5, stages_per_rank
    tr = Trainer(shape, schedule, 1, S, M, lr=lr, seed=5)
    tr.set_override(0.5)
    lays = [param_layout(shape, s, S) for s in range(1, S + 1)]
    bufs = [tr.stage_buffers(i) for i in range(S)]
    theta0 = [device_view(b["master"], b["n_params"]).clone() for b in bufs]
    w0 = [device_view(b["weights"], b["n_params"], torch.bfloat16).clone() for b in bufs]
    rng = np.random.default_rng(1)
    T = shape.tokens
    tokens = rng.integers(0, shape.vocab, size=(M, T), dtype=np.int32)
    targets = rng.integers(0, shape.vocab, size=(M, T), dtype=np.int32)
    res = tr.step(1, tokens, targets)
    torch.cuda.synchronize()
    theta1 = [device_view(b["master"], b["n_params"]).clone() for b in bufs]
    frozen = [[pf.unpack_mask(mk, lays[i]["n_units"]) for mk in tr.last_masks(i)] for i in range(S)]

    params = {}
    for i in range(S):
        params.update({k: v.detach().clone().requires_grad_(True) for k, v in unflatten(w0[i].float(), lays[i]).items()})
    owner = {ent["name"]: i for i in range(S) for ent in lays[i]["units"] + lays[i]["dense"]}
    grads = {k: torch.zeros_like(v) for k, v in params.items()}
    losses = []
    for m in range(M):
        for v in params.values():
            v.grad = None
        loss = stage_loss(params, shape, range(shape.layers), torch.tensor(tokens[m], device=cuda).long(),
                          torch.tensor(targets[m], device=cuda).long(), True, True, faithful=True)
        loss.backward()
        losses.append(loss.item())
        for i in range(S):
            for ent in lays[i]["units"]:
                upd = torch.tensor(_expand_unit_mask(frozen[i][m], ent), device=cuda)
                grads[ent["name"]] += params[ent["name"]].grad * upd
            for ent in lays[i]["dense"]:
                grads[ent["name"]] += params[ent["name"]].grad
    assert abs(res["loss"] - np.mean(losses)) < 2e-2 * abs(np.mean(losses))
    d_dev = {}
    for i in range(S):
        d_dev.update(unflatten(theta1[i] - theta0[i], lays[i]))
    for name, exp_g in grads.items():
        exp = -(lr / M) * exp_g
        if exp.abs().max().item() == 0:
            continue
        rel = (d_dev[name] - exp).norm().item() / exp.norm().item()
        assert rel < 6e-2, (name, owner[name], rel)
    tr.close()


def test_hybrid_apf_reconcile_masks(cuda):
    """Hybrid TimelyFreeze+APF: each freezing-phase cell holds exactly floor(AFR*units) frozen units
    and relates to the APF base set as reconcile_mask (Alg. 2) does: superset when growing,
    subset when shrinking."""
    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    shape = PRESETS["tiny"]
    M, phases = 2, (2, 8, 10, 14)
    # threshold 1.0: every element whose EMA update direction is not constant is eligible
    tr = Trainer(shape, "gpipe", 1, 1, M, phases=phases, r_max=0.8, lr=1e-2, seed=3, apf=True,
                 apf_threshold=0.999, hybrid=True, hybrid_unit_fraction=0.5)
    units = tr.stage_buffers(0)["n_units"]
    checked = 0
    for t in range(1, phases[3] + 1):
        base = tr.apf_base(0)  # base used by this step = last step's APF result
        r = tr.step(t)
        if t <= phases[1] or base is None:
            continue
        plan = tr.get_plan()
        bset = set(np.flatnonzero(pf.unpack_mask(base, units)).tolist())
        ms = tr.last_masks(0)
        for m in range(M):
            target = int(np.floor(pf.actual_freeze_ratio(t, pf.PhasePlan(*phases), plan["ratios"][m]) * units))
            got = set(np.flatnonzero(pf.unpack_mask(ms[m], units)).tolist())
            assert len(got) == target
            if target >= len(bset):
                assert bset <= got
            else:
                assert got <= bset
            checked += 1
        assert np.isfinite(r["loss"])
    assert checked >= 4
    tr.close()


def test_controller_phases_plan_and_bit_exact_masks(cuda):
    import torch  # noqa: F401

    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    shape = PRESETS["tiny"]
    M, phases = 4, (2, 8, 10, 20)
    tr = Trainer(shape, "gpipe", 1, 1, M, phases=phases, r_max=0.8, lr=1e-3, seed=11)
    plan = pf.PhasePlan(*phases)
    units = tr.stage_buffers(0)["n_units"]
    results = []
    for t in range(1, 13):
        r = tr.step(t)
        results.append(r)
        assert r["phase"] == int(pf.phase_of(t, plan))
        assert np.isfinite(r["loss"])
        if t == 7:  # MonitorLower: every unit frozen
            assert r["mean_ratio"] == 1.0
        if t <= 5:
            assert r["mean_ratio"] == 0.0
        p = tr.get_plan()
        assert (p is None) == (t < plan.t_monitor)
        if p is not None:
            # masks are the reference stream (run_freezing_masks order), regenerated by jump-ahead
            ms = pf.MaskStream(p["ratios"], plan, M, 1, units, 11)
            assert np.array_equal(tr.last_masks(0), ms.stage_step(t, 1))
    p = tr.get_plan()
    assert p["makespan_opt"] < p["makespan_base"]
    assert np.all(p["ratios"] <= 1.0) and p["ratios"].mean() <= 0.8 + 1e-6
    stable = results[-1]
    assert abs(stable["mean_ratio"] - p["ratios"].mean()) < 0.02
    assert stable["predicted_ms"] > 0
    tr.close()


def test_zbv_split_controller_plan_over_w_nodes(cuda):
    """zbv-split through warm-up, monitoring (w nodes frozen in MonitorLower), the LP at T_m over
    the w nodes, and the ramp: masks stay the reference stream keyed by the w cells."""
    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    shape = PRESETS["tiny"]
    M, phases = 4, (2, 8, 10, 16)
    tr = Trainer(shape, "zbv-split", 1, 2, M, phases=phases, r_max=0.8, lr=1e-3, seed=13)
    plan = pf.PhasePlan(*phases)
    units = [tr.stage_buffers(i)["n_units"] for i in range(2)]
    for t in range(1, 13):
        r = tr.step(t)
        assert np.isfinite(r["loss"])
        p = tr.get_plan()
        if p is not None:
            ms = pf.MaskStream(p["ratios"], plan, M, 2, units, 13)
            for i, s in enumerate((1, 2)):
                assert np.array_equal(tr.last_masks(i), ms.stage_step(t, s))
    _, kinds, mbs, stages = tr.action_ms()
    assert sorted(np.bincount(kinds).tolist()) == [2 * M] * 3  # f, b, w for both local stages
    p = tr.get_plan()
    n = 2 * M
    assert len(p["w_min"]) == 3 * n
    assert np.allclose(p["w_min"][n:2 * n], p["w_max"][n:2 * n])  # b fixed
    assert np.all(p["w_min"][2 * n:] <= p["w_max"][2 * n:])
    assert np.all(p["ratios"] <= 1.0) and p["ratios"].mean() <= 0.8 + 1e-6
    assert p["makespan_opt"] <= p["makespan_base"]
    tr.close()


@pytest.mark.parametrize("schedule,ranks,C", [("1f1b", 4, 1), ("interleaved-1f1b", 4, 2), ("zbv", 2, 2),
                                              ("zbv-split", 4, 2)])
def test_trainer_p2p_links_match_host_rule(cuda, schedule, ranks, C):
    """The device trainer's NCCL link list (one communicator per cross-rank edge class) is the one
    the gloo replay of the issue program validated (pipefreeze.p2p_links)."""
    from paper_2602_05754_b200 import pipefreeze as pf
    from paper_2602_05754_b200.engine import PRESETS, Trainer

    import dataclasses

    cfg = pf.PipelineConfig(schedule, ranks, C, 4)
    tr = Trainer(dataclasses.replace(PRESETS["tiny"], layers=8), schedule, ranks, C, 4, rank=1)
    assert tr.links() == pf.p2p_links(cfg)
    with pytest.raises(Exception):
        tr.step(1)  # remote neighbours and no init_comm(): refused, not silently local
    tr.close()


@pytest.mark.parametrize("dense_kernel", ["1", "0"])
def test_mixed_dense_and_partial_cells_match_torch_reference(cuda, dense_kernel, monkeypatch):
    """One step whose microbatch cells mix partial masks (row-pair dW over K5r lists) and a cell with
    no frozen unit (the dense CTA-pair dW, chosen per cell from the host mask), given as caller-owned
    masks: the unit stamps must hand the accumulation across the two kernels (a unit first written by
    a partial cell is accumulated by the dense one and vice versa). The accumulated gradient (fp32
    grad buffer) vs the fp32 torch reference; PF_DW_DENSE=0 runs every cell on the row-pair kernel."""
    import torch

    monkeypatch.setenv("PF_DW_DENSE", dense_kernel)
    from gpu_util import device_view
    from llama_ref import stage_loss, unflatten
    from paper_2602_05754_b200.engine import PRESETS, Trainer, param_layout

    shape = PRESETS["tiny"]
    M = 3
    tr = Trainer(shape, "gpipe", 1, 1, M, lr=0.5, seed=21)
    lay = param_layout(shape, 1, 1)
    buf = tr.stage_buffers(0)
    n, units = buf["n_params"], buf["n_units"]
    words = (units + 63) // 64
    rng = np.random.default_rng(5)
    bits = np.stack([rng.random(units) < 0.5, np.zeros(units, dtype=bool), rng.random(units) < 0.3])
    host = np.zeros((M, words), dtype=np.uint64)
    for m in range(M):
        for u in np.flatnonzero(bits[m]):
            host[m, u // 64] |= np.uint64(1) << np.uint64(u % 64)
    tok = rng.integers(0, shape.vocab, size=(M, shape.tokens), dtype=np.int32)
    tgt = rng.integers(0, shape.vocab, size=(M, shape.tokens), dtype=np.int32)
    w0 = device_view(buf["weights"], n, torch.bfloat16).clone()
    tr.step(1, tok, tgt, masks=host)
    torch.cuda.synchronize()
    g_dev = unflatten(device_view(buf["grad"], n).clone(), lay)
    params = {k: v.detach().clone().requires_grad_(True) for k, v in unflatten(w0.float(), lay).items()}
    grads = {k: torch.zeros_like(v) for k, v in params.items()}
    for m in range(M):
        for v in params.values():
            v.grad = None
        loss = stage_loss(params, shape, range(shape.layers), torch.tensor(tok[m], device=cuda).long(),
                          torch.tensor(tgt[m], device=cuda).long(), True, True, faithful=True)
        loss.backward()
        for ent in lay["units"]:
            grads[ent["name"]] += params[ent["name"]].grad * torch.tensor(_expand_unit_mask(bits[m], ent), device=cuda)
    checked = 0
    for ent in lay["units"]:
        name = ent["name"]
        touched = torch.tensor(_expand_unit_mask(np.logical_and.reduce(bits), ent), device=cuda).bool()
        exp, got = grads[name][touched], g_dev[name][touched]
        if exp.abs().max().item() == 0:
            continue
        rel = (got - exp).norm().item() / exp.norm().item()
        assert rel < 6e-2, (name, rel)
        checked += 1
    assert checked >= 8
    tr.close()
