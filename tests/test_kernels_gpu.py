"""K4/K5/K6/K7 device kernels vs a plain PyTorch fp32 reference or the golden oracle vectors."""
import ctypes
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def lib():
    from paper_2602_05754_b200 import _native

    return _native.device()


def chk(rc, what=""):
    assert rc == 0, f"{what}: {rc} {lib().pf_engine_last_error().decode()}"


def sp():
    import torch

    return torch.cuda.current_stream().cuda_stream


def bf(x):
    import torch

    return x.to(torch.bfloat16)


@pytest.mark.parametrize("T,h", [(256, 1024), (512, 2048), (136, 256), (200, 4096), (201, 4096), (72, 5120), (73, 5120), (64, 768)])
def test_rmsnorm_fwd_bwd(cuda, T, h):
    """Register-row forward and the fused backward (dx + dg in one pass) for the LLaMA widths
    (h = 4096 / 5120: the row-block kernels, odd T covers their tail rows); h = 768 takes the
    generic kernels."""
    import torch

    g = torch.Generator().manual_seed(1)
    x = bf(torch.randn(T, h, generator=g)).cuda()
    w = bf(1 + 0.1 * torch.randn(h, generator=g)).cuda()
    dy = bf(torch.randn(T, h, generator=g)).cuda()
    res = bf(torch.randn(T, h, generator=g)).cuda()
    y = torch.empty_like(x)
    rstd = torch.empty(T, device=cuda)
    chk(lib().pf_rmsnorm_fwd(x.data_ptr(), w.data_ptr(), y.data_ptr(), rstd.data_ptr(), T, h, 1e-5, sp()))
    xf = x.float().requires_grad_(True)
    wf = w.float().requires_grad_(True)
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * wf
    torch.cuda.synchronize()
    assert (y.float() - ref).abs().max().item() < 2e-2 * ref.abs().max().item()
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.zeros(h, device=cuda)
    chk(lib().pf_rmsnorm_bwd(x.data_ptr(), w.data_ptr(), rstd.data_ptr(), dy.data_ptr(), res.data_ptr(), dx.data_ptr(),
                             dg.data_ptr(), T, h, sp()))
    torch.cuda.synchronize()
    exp = xf.grad + res.float()
    assert (dx.float() - exp).abs().max().item() < 2e-2 * exp.abs().max().item()
    assert torch.allclose(dg, wf.grad, rtol=1e-3, atol=1e-3 * wf.grad.abs().max().item())
    # dg accumulates into its buffer; dx does not depend on residual being absent
    dg2 = torch.zeros(h, device=cuda)
    dx2 = torch.empty_like(x)
    for _ in range(2):
        chk(lib().pf_rmsnorm_bwd(x.data_ptr(), w.data_ptr(), rstd.data_ptr(), dy.data_ptr(), None, dx2.data_ptr(),
                                 dg2.data_ptr(), T, h, sp()))
    torch.cuda.synchronize()
    assert torch.allclose(dg2, 2 * dg, rtol=1e-5, atol=1e-5 * dg.abs().max().item())
    assert torch.allclose(dx2.float(), xf.grad, rtol=2e-2, atol=2e-2 * xf.grad.abs().max().item())


def test_swiglu_fwd_bwd(cuda):
    import torch
    import torch.nn.functional as F

    T, ffn = 256, 512
    g = torch.Generator().manual_seed(2)
    gu = bf(torch.randn(T, 2 * ffn, generator=g)).cuda()
    da = bf(torch.randn(T, ffn, generator=g)).cuda()
    a = torch.empty(T, ffn, dtype=torch.bfloat16, device=cuda)
    chk(lib().pf_swiglu_fwd(gu.data_ptr(), a.data_ptr(), T, ffn, sp()))
    from llama_ref import gate_index

    gi = gate_index(ffn, cuda)
    guf = gu.float().requires_grad_(True)
    ref = F.silu(guf[:, gi]) * guf[:, gi + 128]
    ref.backward(da.float())
    dgu = torch.empty_like(gu)
    chk(lib().pf_swiglu_bwd(gu.data_ptr(), da.data_ptr(), dgu.data_ptr(), T, ffn, sp()))
    torch.cuda.synchronize()
    assert (a.float() - ref).abs().max().item() < 1e-2 * ref.abs().max().item() + 1e-2
    assert (dgu.float() - guf.grad).abs().max().item() < 1e-2 * guf.grad.abs().max().item() + 1e-2


def test_gemm_swiglu_epilogue_matches_unfused(cuda):
    """Pair-GEMM SwiGLU epilogue == GEMM (bf16 store) followed by swiglu_fwd, bit for bit."""
    import torch

    T, D, ffn = 512, 256, 768
    g = torch.Generator().manual_seed(9)
    h = bf(torch.randn(T, D, generator=g)).cuda()
    w = bf(torch.randn(2 * ffn, D, generator=g) * 0.1).cuda()
    gu = torch.empty(T, 2 * ffn, dtype=torch.bfloat16, device=cuda)
    a = torch.empty(T, ffn, dtype=torch.bfloat16, device=cuda)
    chk(lib().pf_gemm_swiglu(h.data_ptr(), h.stride(0), w.data_ptr(), w.stride(0), gu.data_ptr(), a.data_ptr(), T,
                             ffn, D, sp()))
    gu_ref = torch.empty_like(gu)
    chk(lib().pf_gemm_bf16(h.data_ptr(), 0, h.stride(0), w.data_ptr(), 0, w.stride(0), gu_ref.data_ptr(),
                           gu_ref.stride(0), T, 2 * ffn, D, 1.0, 0, 512, None, 0, sp()))
    a_ref = torch.empty_like(a)
    chk(lib().pf_swiglu_fwd(gu_ref.data_ptr(), a_ref.data_ptr(), T, ffn, sp()))
    torch.cuda.synchronize()
    assert torch.equal(gu, gu_ref)
    assert torch.equal(a, a_ref)


@pytest.mark.parametrize("T,S,nh,nkv,D,hd", [(4096, 2048, 32, 8, 2048, 64), (512, 128, 4, 4, 256, 64),
                                             (300, 100, 6, 1, 256, 64), (4096, 2048, 32, 8, 4096, 128),
                                             (2048, 2048, 40, 40, 5120, 128), (384, 128, 2, 1, 256, 128)])
def test_gemm_rope_epilogue_matches_unfused(cuda, T, S, nh, nkv, D, hd):
    """qkv projection with RoPE fused in the pair-GEMM epilogue == GEMM then rope_fwd, bit for bit
    (GQA widths; T = 300 leaves a partial row tile, S = 100 several sequences per microbatch;
    head_dim 128 at the LLaMA-8B (32/8) and LLaMA-13B (40/40 MHA) shapes)."""
    import torch

    N = (nh + 2 * nkv) * hd
    g = torch.Generator().manual_seed(T + nh)
    x = bf(torch.randn(T, D, generator=g)).cuda()
    w = bf(torch.randn(N, D, generator=g) * 0.1).cuda()
    qkv = torch.empty(T, N, dtype=torch.bfloat16, device=cuda)
    rc = lib().pf_gemm_rope(x.data_ptr(), D, w.data_ptr(), D, qkv.data_ptr(), T, S, nh, nkv, hd, D, 500000.0, sp())
    if N % 256:
        assert rc == 4  # the fused epilogue needs whole 256-column tiles (the stage then runs GEMM + rope)
        return
    chk(rc)
    ref = torch.empty_like(qkv)
    chk(lib().pf_gemm_bf16(x.data_ptr(), 0, D, w.data_ptr(), 0, D, ref.data_ptr(), N, T, N, D, 1.0, 0, 512, None, 0,
                           sp()))
    chk(lib().pf_rope_fwd(ref.data_ptr(), T, S, nh, nkv, hd, 500000.0, sp()))
    torch.cuda.synchronize()
    assert torch.equal(qkv, ref)


def test_gelu_kernels_every_bf16_input(cuda):
    """gelu_fwd / gelu_bwd (the packed A&S 7.1.26 forms the GEMM epilogues share) over all 65,536 bf16
    inputs vs fp64 erf GELU: every finite input within 2 bf16 ulp of the fp64 value rounded to bf16 or
    1e-6 absolute (the approximation's erf error is 1.5e-7 absolute; gelu' crosses zero at -0.75), and
    at most 1% of values differing from the rounded fp64 value at all."""
    import math

    import numpy as np
    import torch

    bits = torch.arange(65536, dtype=torch.int32).to(torch.int16).view(torch.bfloat16)
    x = bits[torch.isfinite(bits.float())].contiguous()
    n = x.numel() // 8 * 8
    x = x[:n].cuda()
    act = torch.empty_like(x)
    chk(lib().pf_gelu_fwd(x.data_ptr(), act.data_ptr(), n, sp()))
    ones = torch.ones_like(x)
    dx = torch.empty_like(x)
    chk(lib().pf_gelu_bwd(x.data_ptr(), ones.data_ptr(), dx.data_ptr(), n, sp()))
    torch.cuda.synchronize()
    v = x.double().cpu().numpy()
    erf = np.vectorize(math.erf)(v / math.sqrt(2.0))
    ref_f = 0.5 * v * (1.0 + erf)
    ref_g = 0.5 * (1.0 + erf) + v * np.exp(-0.5 * v * v) / math.sqrt(2.0 * math.pi)
    for got, ref in ((act, ref_f), (dx, ref_g)):
        g = got.double().cpu().numpy()
        r = torch.from_numpy(ref).to(torch.bfloat16).double().numpy()
        ulp = np.maximum(np.abs(r) * 2.0 ** -6, 1e-6)
        ok = np.isfinite(r)
        assert (np.abs(g - r)[ok] <= ulp[ok]).all()
        assert (g != r)[ok].mean() <= 0.01


@pytest.mark.parametrize("T,ffn,D", [(512, 768, 256), (3200, 4096, 1024)])
def test_gemm_gelu_epilogues_match_unfused(cuda, T, ffn, D):
    """ViT MLP: GELU fused in the pair-GEMM epilogues == GEMM then gelu_fwd / gelu_bwd, bit for bit
    (zero bias, so the unfused GEMM rounds the same value); with a bias, vs torch fp32; dpre in place."""
    import torch

    g = torch.Generator().manual_seed(T + ffn + D)
    x = bf(torch.randn(T, D, generator=g)).cuda()
    w1 = bf(torch.randn(ffn, D, generator=g) * 0.1).cuda()
    w2 = bf(torch.randn(D, ffn, generator=g) * 0.1).cuda()  # fc2 weight [out=D][in=ffn]
    dy = bf(torch.randn(T, D, generator=g)).cuda()
    zero = torch.zeros(ffn, dtype=torch.bfloat16, device=cuda)
    pre = torch.empty(T, ffn, dtype=torch.bfloat16, device=cuda)
    act = torch.empty_like(pre)
    chk(lib().pf_gemm_gelu(x.data_ptr(), D, w1.data_ptr(), D, zero.data_ptr(), pre.data_ptr(), act.data_ptr(), T, ffn,
                           D, sp()))
    pre_ref = torch.empty_like(pre)
    chk(lib().pf_gemm_bf16(x.data_ptr(), 0, D, w1.data_ptr(), 0, D, pre_ref.data_ptr(), ffn, T, ffn, D, 1.0, 0, 512,
                           None, 0, sp()))
    act_ref = torch.empty_like(pre)
    chk(lib().pf_gelu_fwd(pre_ref.data_ptr(), act_ref.data_ptr(), T * ffn, sp()))
    torch.cuda.synchronize()
    assert torch.equal(pre, pre_ref) and torch.equal(act, act_ref)
    # bias: fp32 reference
    b = bf(torch.randn(ffn, generator=g)).cuda()
    chk(lib().pf_gemm_gelu(x.data_ptr(), D, w1.data_ptr(), D, b.data_ptr(), pre.data_ptr(), act.data_ptr(), T, ffn, D,
                           sp()))
    torch.cuda.synchronize()
    p32 = x.float() @ w1.float().t() + b.float()
    assert (pre.float() - p32).abs().max().item() <= 2e-2 * p32.abs().max().item()
    a32 = torch.nn.functional.gelu(pre.float())
    assert (act.float() - a32).abs().max().item() <= 2e-2 * a32.abs().max().item()
    # backward: dpre = bf16(dy . W2) * gelu'(pre); out of place, then in place over a copy of pre
    dpre = torch.empty_like(pre)
    db = torch.full((ffn,), 0.5, device=cuda)
    chk(lib().pf_gemm_dgelu(dy.data_ptr(), D, w2.data_ptr(), ffn, pre.data_ptr(), dpre.data_ptr(), db.data_ptr(), T,
                            ffn, D, sp()))
    da = torch.empty_like(pre)
    chk(lib().pf_gemm_bf16(dy.data_ptr(), 0, D, w2.data_ptr(), 1, ffn, da.data_ptr(), ffn, T, ffn, D, 1.0, 0, 512,
                           None, 0, sp()))
    dpre_ref = torch.empty_like(pre)
    chk(lib().pf_gelu_bwd(pre.data_ptr(), da.data_ptr(), dpre_ref.data_ptr(), T * ffn, sp()))
    inplace = pre.clone()
    chk(lib().pf_gemm_dgelu(dy.data_ptr(), D, w2.data_ptr(), ffn, inplace.data_ptr(), inplace.data_ptr(), None, T, ffn,
                            D, sp()))
    torch.cuda.synchronize()
    assert torch.equal(dpre, dpre_ref)
    assert torch.equal(inplace, dpre_ref)
    colsum = dpre_ref.float().sum(0) + 0.5  # db accumulates into its buffer
    assert torch.allclose(db, colsum, rtol=1e-4, atol=1e-3 * colsum.abs().max().item())


@pytest.mark.parametrize("T,ffn,D", [(512, 768, 256), (4096, 2048, 1024)])
def test_gemm_dswiglu_epilogue_matches_unfused(cuda, T, ffn, D):
    """Pair-GEMM SwiGLU-backward epilogue == GEMM (bf16 d_act) followed by swiglu_bwd, bit for bit
    (stream-K sums the split K in another order, so that run is checked to bf16 tolerance)."""
    import torch

    g = torch.Generator().manual_seed(T + ffn)
    dy = bf(torch.randn(T, D, generator=g)).cuda()
    wd = bf(torch.randn(D, ffn, generator=g) * 0.1).cuda()
    gu = bf(torch.randn(T, 2 * ffn, generator=g)).cuda()
    dgus = []
    for mode in (0, 1):  # data-parallel tiles, then forced stream-K (fixup before the epilogue math)
        chk(lib().pf_gemm_set_streamk(mode))
        dgu = torch.empty_like(gu)
        chk(lib().pf_gemm_dswiglu(dy.data_ptr(), dy.stride(0), wd.data_ptr(), wd.stride(0), gu.data_ptr(),
                                  dgu.data_ptr(), T, ffn, D, sp()))
        dgus.append(dgu)
    chk(lib().pf_gemm_set_streamk(0))
    da = torch.empty(T, ffn, dtype=torch.bfloat16, device=cuda)
    chk(lib().pf_gemm_bf16(dy.data_ptr(), 0, dy.stride(0), wd.data_ptr(), 1, wd.stride(0), da.data_ptr(),
                           da.stride(0), T, ffn, D, 1.0, 0, 512, None, 0, sp()))
    dgu_ref = torch.empty_like(gu)
    chk(lib().pf_swiglu_bwd(gu.data_ptr(), da.data_ptr(), dgu_ref.data_ptr(), T, ffn, sp()))
    torch.cuda.synchronize()
    assert torch.equal(dgus[0], dgu_ref)
    assert (dgus[1].float() - dgu_ref.float()).abs().max().item() <= 1e-2 * dgu_ref.float().abs().max().item()


@pytest.mark.parametrize("B,S,nh,nkv,hd,theta", [(2, 64, 4, 2, 64, 500000.0), (2, 2048, 32, 8, 128, 500000.0),
                                                 (1, 2048, 40, 40, 128, 10000.0)])
def test_rope_matches_reference(cuda, B, S, nh, nkv, hd, theta):
    """rope_fwd vs the fp32 rotate-half restatement, head_dim 64 and 128 (LLaMA-8B / 13B shapes)."""
    import torch

    from llama_ref import rope

    T = B * S
    W = (nh + 2 * nkv) * hd
    g = torch.Generator().manual_seed(3)
    qkv = bf(torch.randn(T, W, generator=g)).cuda()
    ref = qkv.float().view(B, S, nh + 2 * nkv, hd).clone()
    ref[:, :, : nh + nkv] = rope(ref[:, :, : nh + nkv], S, theta)
    chk(lib().pf_rope_fwd(qkv.data_ptr(), T, S, nh, nkv, hd, theta, sp()))
    torch.cuda.synchronize()
    got = qkv.float().view_as(ref)
    # bf16 output: one rounding of the fp32 rotation (|x| <~ 5 -> ulp <= 2^-5)
    assert (got - ref).abs().max().item() < 2e-2
    assert torch.equal(got[:, :, nh + nkv:], ref[:, :, nh + nkv:])  # v heads untouched


@pytest.mark.parametrize("V", [4096, 1024, 1000, 128256, 32000, 8, 65544])
def test_cross_entropy_fused(cuda, V):
    import torch
    import torch.nn.functional as F

    T = 128
    g = torch.Generator().manual_seed(4)
    logits = bf(3 * torch.randn(T, V, generator=g)).cuda()
    tgt = torch.randint(0, V, (T,), generator=g).int().cuda()
    lf = logits.float().requires_grad_(True)
    loss = F.cross_entropy(lf, tgt.long())
    loss.backward()
    ls = torch.zeros(1, device=cuda)
    chk(lib().pf_cross_entropy(logits.data_ptr(), tgt.data_ptr(), ls.data_ptr(), T, V, 1.0 / T, 1.0 / T, sp()))
    torch.cuda.synchronize()
    assert abs(ls.item() - loss.item()) < 1e-3 * loss.item()
    assert (logits.float() - lf.grad).abs().max().item() < 2e-2 * lf.grad.abs().max().item()


def test_apf_update_vs_reference_golden(cuda):
    """K4 fp32 on device vs the reference's fp64 apf_update (freezectl.cpp:147-156)."""
    import torch

    with open(os.path.join(GOLD, "apf.json")) as f:
        cases = json.load(f)
    for case in cases:
        n = case["n"]
        d = np.array([float.fromhex(x) for x in case["deltas"]]).reshape(-1, n)
        e = torch.zeros(n, device=cuda)
        ea = torch.zeros(n, device=cuda)
        sc = torch.zeros(n, device=cuda)
        for row in d:
            dd = torch.tensor(row, dtype=torch.float32, device=cuda)
            chk(lib().pf_apf_update(e.data_ptr(), ea.data_ptr(), dd.data_ptr(), sc.data_ptr(), n, case["alpha"], sp()))
        torch.cuda.synchronize()
        ref_e = np.array([float.fromhex(x) for x in case["ema"]])
        ref_a = np.array([float.fromhex(x) for x in case["ema_abs"]])
        ref_s = np.array([float.fromhex(x) for x in case["scores"]])
        np.testing.assert_allclose(e.cpu().numpy(), ref_e, rtol=2e-5, atol=1e-12)
        np.testing.assert_allclose(ea.cpu().numpy(), ref_a, rtol=2e-5, atol=1e-12)
        np.testing.assert_allclose(sc.cpu().numpy(), ref_s, rtol=1e-4, atol=1e-6)


def _pair_band(tiles_m, tiles_n):
    """Rows of units per K5p band (kernels.cuh pair_band_rows)."""
    band = 32
    while -(-tiles_m // band) * tiles_n > 2048:
        band *= 2
    return band


def _unit_table(shapes):
    """pf_unit_matrix table for matrices laid out back to back (64-element aligned)."""
    dt = np.dtype([("elem_offset", "<i8"), ("rows", "<i4"), ("cols", "<i4"), ("unit_offset", "<i4"),
                   ("tiles_n", "<i4"), ("units", "<i4"), ("pair_offset", "<i4")])
    tab = np.zeros(len(shapes), dtype=dt)
    off = u = po = 0
    for i, (r, c) in enumerate(shapes):
        tn = (c + 127) // 128
        tm = (r + 127) // 128
        units = tm * tn
        tab[i] = (off, r, c, u, tn, units, po)
        off = (off + r * c + 63) // 64 * 64
        u += units
        po += ((units + max(-(-tm // _pair_band(tm, tn)) * tn, tm) + 1) // 2) * 2  # pair_list_capacity
    return tab, off, u


def rowpair_list_ref(frozen, tiles_m, tiles_n):
    """K5r restated: per unit row, its unfrozen local unit ids paired in order, an odd row ending (u, -1)."""
    out = []
    for mb in range(tiles_m):
        row = [mb * tiles_n + nb for nb in range(tiles_n) if not frozen[mb * tiles_n + nb]]
        if len(row) % 2:
            row.append(-1)
        out += row
    return out


def pair_list_ref(frozen, tiles_m, tiles_n):
    """K5p restated: (band, column) groups band by band, unfrozen local unit ids top to bottom,
    each group padded to an even count with -1."""
    band = _pair_band(tiles_m, tiles_n)
    out = []
    for b0 in range(0, tiles_m, band):
        for nb in range(tiles_n):
            grp = [mb * tiles_n + nb for mb in range(b0, min(tiles_m, b0 + band)) if not frozen[mb * tiles_n + nb]]
            out += grp + ([-1] if len(grp) % 2 else [])
    return out


def test_mask_to_unit_lists_matches_numpy(cuda):
    import torch

    from paper_2602_05754_b200 import pipefreeze as pf

    tab, _, U = _unit_table([(384, 256), (256, 640), (1000, 128), (128, 128)])
    words = pf.sample_masks(7, U, [0.55])[0]
    w = np.concatenate([words, np.zeros(1, dtype=np.uint64)])
    wd = torch.tensor(w.view(np.int64), device=cuda)
    td = torch.tensor(tab.view(np.uint8), device=cuda)
    lists = torch.full((U + 64,), -1, dtype=torch.int32, device=cuda)
    counts = torch.zeros(len(tab), dtype=torch.int32, device=cuda)
    chk(lib().pf_mask_to_unit_lists(wd.data_ptr(), td.data_ptr(), len(tab), lists.data_ptr(), counts.data_ptr(), sp()))
    torch.cuda.synchronize()
    frozen = pf.unpack_mask(words, U)
    L = lists.cpu().numpy()
    for i, ent in enumerate(tab):
        lo, n = int(ent["unit_offset"]), int(ent["units"])
        expect = [j for j in range(n) if not frozen[lo + j]]
        assert counts[i].item() == len(expect)
        assert L[lo:lo + len(expect)].tolist() == expect


@pytest.mark.parametrize("ratio", [0.0, 0.55, 0.8, 1.0])
def test_mask_to_pair_lists_matches_numpy(cuda, ratio):
    """K5p: banded, column-grouped, even-padded pair lists; a 1002-row matrix spans 32 bands
    (the LM head shape) and a 64-column one exercises many groups per band."""
    import torch

    from paper_2602_05754_b200 import pipefreeze as pf

    tab, _, U = _unit_table([(384, 256), (256, 640), (1000, 128), (128, 128), (128256, 256), (2048, 8192)])
    words = pf.sample_masks(7, U, [ratio])[0]
    w = np.concatenate([words, np.zeros(1, dtype=np.uint64)])
    wd = torch.tensor(w.view(np.int64), device=cuda)
    td = torch.tensor(tab.view(np.uint8), device=cuda)
    cap = int(tab["pair_offset"][-1]) + int(tab["units"][-1]) * 2 + 64
    pairs = torch.full((cap,), -7, dtype=torch.int32, device=cuda)
    counts = torch.zeros(len(tab), dtype=torch.int32, device=cuda)
    chk(lib().pf_mask_to_pair_lists(wd.data_ptr(), td.data_ptr(), len(tab), pairs.data_ptr(), counts.data_ptr(),
                                    sp()))
    torch.cuda.synchronize()
    frozen = pf.unpack_mask(words, U)
    P = pairs.cpu().numpy()
    for i, ent in enumerate(tab):
        lo, n, tn, po = int(ent["unit_offset"]), int(ent["units"]), int(ent["tiles_n"]), int(ent["pair_offset"])
        expect = pair_list_ref(frozen[lo:lo + n], n // tn, tn)
        assert counts[i].item() == len(expect) and len(expect) % 2 == 0
        assert P[po:po + len(expect)].tolist() == expect


@pytest.mark.parametrize("ratio", [0.0, 0.55, 0.8, 1.0])
def test_mask_to_rowpair_lists_matches_numpy(cuda, ratio):
    """K5r: row-major pairs of unfrozen units of one unit row; 64 and 112 column blocks span
    several ballots; the LM-head shape has 1002 rows."""
    import torch

    from paper_2602_05754_b200 import pipefreeze as pf

    tab, _, U = _unit_table([(384, 256), (256, 640), (1000, 128), (128, 128), (128256, 256), (2048, 8192),
                             (4096, 14336)])
    words = pf.sample_masks(11, U, [ratio])[0]
    w = np.concatenate([words, np.zeros(1, dtype=np.uint64)])
    wd = torch.tensor(w.view(np.int64), device=cuda)
    td = torch.tensor(tab.view(np.uint8), device=cuda)
    cap = int(tab["pair_offset"][-1]) + int(tab["units"][-1]) * 2 + 64
    lists = torch.full((cap,), -7, dtype=torch.int32, device=cuda)
    counts = torch.zeros(len(tab), dtype=torch.int32, device=cuda)
    chk(lib().pf_mask_to_rowpair_lists(wd.data_ptr(), td.data_ptr(), len(tab), lists.data_ptr(), counts.data_ptr(),
                                       sp()))
    torch.cuda.synchronize()
    frozen = pf.unpack_mask(words, U)
    L = lists.cpu().numpy()
    for i, ent in enumerate(tab):
        lo, n, tn, po = int(ent["unit_offset"]), int(ent["units"]), int(ent["tiles_n"]), int(ent["pair_offset"])
        expect = rowpair_list_ref(frozen[lo:lo + n], n // tn, tn)
        assert counts[i].item() * 2 == len(expect)
        assert L[po:po + len(expect)].tolist() == expect


def test_masked_sgd_units_and_fused_apf(cuda):
    """theta -= scale*G only on touched units (stamp == step); APF advances every unit."""
    import torch

    tab, nparam, U = _unit_table([(256, 384), (128, 256)])
    g = torch.Generator().manual_seed(9)
    master = torch.randn(nparam, generator=g).cuda()
    weights = master.to(torch.bfloat16)
    grad = torch.randn(nparam, generator=g).cuda()
    stamps = torch.zeros(U, dtype=torch.int32)
    touched = [0, 2, 3, 6, 7]
    stamps[touched] = 5
    stamps = stamps.cuda()
    ema = torch.zeros(nparam, device=cuda)
    ema_abs = torch.zeros(nparam, device=cuda)
    elig = torch.zeros(U, dtype=torch.int32, device=cuda)
    td = torch.tensor(tab.view(np.uint8), device=cuda)
    m0 = master.clone()
    scale = 0.01
    chk(lib().pf_masked_sgd_units(master.data_ptr(), weights.data_ptr(), grad.data_ptr(), stamps.data_ptr(), 5, scale,
                                  td.data_ptr(), len(tab), U, ema.data_ptr(), ema_abs.data_ptr(), 0.9, 0.5,
                                  elig.data_ptr(), sp()))
    torch.cuda.synchronize()
    # expected: numpy restatement of sandbox.cpp:250 per unit
    m_exp = m0.cpu().numpy().copy()
    e_exp = np.zeros(nparam, dtype=np.float32)
    gnp = grad.cpu().numpy()
    for ent in tab:
        for lu in range(int(ent["units"])):
            u = int(ent["unit_offset"]) + lu
            rb, cb = divmod(lu, int(ent["tiles_n"]))
            for r in range(rb * 128, min(int(ent["rows"]), rb * 128 + 128)):
                s = int(ent["elem_offset"]) + r * int(ent["cols"]) + cb * 128
                e = s + min(128, int(ent["cols"]) - cb * 128)
                if u in touched:
                    m_exp[s:e] -= scale * gnp[s:e]
                    e_exp[s:e] = 0.1 * (-scale * gnp[s:e])
    np.testing.assert_allclose(master.cpu().numpy(), m_exp, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(ema.cpu().numpy(), e_exp, rtol=1e-5, atol=1e-9)
    assert torch.equal(weights, master.to(torch.bfloat16))
    # untouched units: score = 1 (E_abs == 0) -> not eligible; touched: |E|/E_abs = 1 -> not eligible (thr 0.5)
    assert elig.sum().item() == 0
