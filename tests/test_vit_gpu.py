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


@pytest.mark.parametrize("B,S,nh", [(4, 50, 16), (3, 64, 2), (5, 10, 4), (2, 1, 3)])
def test_short_sequence_attention_vs_torch(cuda, B, S, nh):
    """Per-(image, head) attention kernels vs torch fp32 softmax attention: O, LSE and the packed
    dq|dk|dv (also written in place over qkv)."""
    import math

    import torch

    from paper_2602_05754_b200 import _native

    lib = _native.device()
    hd = 64
    g = torch.Generator().manual_seed(B * 100 + S)
    qkv = torch.randn(B * S, 3 * nh * hd, generator=g).to(torch.bfloat16).cuda()
    dout = torch.randn(B * S, nh * hd, generator=g).to(torch.bfloat16).cuda()
    out = torch.empty(B * S, nh * hd, dtype=torch.bfloat16, device=cuda)
    lse = torch.empty(B * nh * S, device=cuda)
    scale = 1.0 / math.sqrt(hd)
    st = torch.cuda.current_stream().cuda_stream
    _native.check(lib.pf_vit_attn_fwd(qkv.data_ptr(), out.data_ptr(), lse.data_ptr(), B, S, nh, hd, scale, st), "fwd")
    dqkv = torch.empty_like(qkv)
    _native.check(lib.pf_vit_attn_bwd(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(), dqkv.data_ptr(),
                                      None, B, S, nh, hd, scale, st), "bwd")
    inplace = qkv.clone()
    dbias = torch.full((3 * nh * hd,), 0.5, device=cuda)  # accumulated into, like the stage's grad buffer
    _native.check(lib.pf_vit_attn_bwd(inplace.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                      inplace.data_ptr(), dbias.data_ptr(), B, S, nh, hd, scale, st), "bwd in place")
    torch.cuda.synchronize()
    x = qkv.float().view(B, S, 3, nh, hd).permute(2, 0, 3, 1, 4)  # [3, B, nh, S, hd]
    q, k, v = (t.clone().requires_grad_(True) for t in x)
    sc = q @ k.transpose(-1, -2) * scale
    ref_lse = torch.logsumexp(sc, -1)
    o = torch.softmax(sc, -1) @ v
    o.backward(dout.float().view(B, S, nh, hd).permute(0, 2, 1, 3))
    o_ref = o.permute(0, 2, 1, 3).reshape(B * S, nh * hd)
    assert (out.float() - o_ref).abs().max().item() <= 2e-2 * o_ref.abs().max().item()
    assert torch.allclose(lse.view(B, nh, S), ref_lse, atol=2e-2, rtol=1e-2)
    grads = torch.stack([q.grad, k.grad, v.grad]).permute(1, 3, 0, 2, 4).reshape(B * S, 3 * nh * hd)
    assert (dqkv.float() - grads).abs().max().item() <= 3e-2 * grads.abs().max().item()
    assert torch.equal(inplace, dqkv)
    # fused bias gradient = column sums of the stored bf16 dqkv (fp32 atomics: order-dependent rounding only)
    db_ref = dqkv.float().sum(0) + 0.5
    assert torch.allclose(dbias, db_ref, atol=1e-3, rtol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("T,h", [(3200, 1024), (777, 512), (129, 256), (300, 768)])
def test_layernorm_fwd_bwd_vs_torch(cuda, T, h):
    """pf_layernorm_fwd / pf_layernorm_bwd against torch fp32 (the fused one-pass backward for
    h = 256 * {1, 2, 4}, the two-kernel path for h = 768), with residual, dg, db and dsum."""
    import torch

    from paper_2602_05754_b200 import _native

    lib = _native.device()
    gen = torch.Generator().manual_seed(T + h)
    x = torch.randn(T, h, generator=gen).to(torch.bfloat16).cuda()
    g = (1 + 0.1 * torch.randn(h, generator=gen)).to(torch.bfloat16).cuda()
    b = (0.1 * torch.randn(h, generator=gen)).to(torch.bfloat16).cuda()
    dy = torch.randn(T, h, generator=gen).to(torch.bfloat16).cuda()
    res = torch.randn(T, h, generator=gen).to(torch.bfloat16).cuda()
    y = torch.empty_like(x)
    mean = torch.empty(T, device=cuda)
    rstd = torch.empty(T, device=cuda)
    dx = torch.empty_like(x)
    dg, db, dsum = (torch.full((h,), 0.25, device=cuda) for _ in range(3))
    st = torch.cuda.current_stream().cuda_stream
    _native.check(lib.pf_layernorm_fwd(x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
                                       rstd.data_ptr(), T, h, 1e-6, st), "ln fwd")
    _native.check(lib.pf_layernorm_bwd(x.data_ptr(), g.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dy.data_ptr(),
                                       res.data_ptr(), dx.data_ptr(), dg.data_ptr(), db.data_ptr(), dsum.data_ptr(),
                                       T, h, st), "ln bwd")
    torch.cuda.synchronize()
    xf = x.float().requires_grad_(True)
    gf = g.float().requires_grad_(True)
    bf = b.float().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xf, (h,), gf, bf, eps=1e-6)
    yr.backward(dy.float())
    assert (y.float() - yr).abs().max().item() <= 2e-2 * yr.abs().max().item()
    assert torch.allclose(mean, x.float().mean(1), atol=1e-4)
    ref_dx = xf.grad + res.float()
    assert (dx.float() - ref_dx).abs().max().item() <= 1e-2 * ref_dx.abs().max().item()
    assert torch.allclose(dg - 0.25, gf.grad, atol=2e-2 * gf.grad.abs().max().item())
    assert torch.allclose(db - 0.25, bf.grad, atol=1e-3 * bf.grad.abs().max().item() + 1e-3)
    # dsum sums the stored bf16 dx (fp32 atomics: order-dependent rounding only)
    assert torch.allclose(dsum - 0.25, dx.float().sum(0), atol=1e-3 * T ** 0.5, rtol=1e-4)
