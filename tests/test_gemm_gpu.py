"""K1/K2/K3 tcgen05 GEMM parity vs a torch fp32 reference of the same op (bf16 inputs)."""
import ctypes

import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2602_05754_b200 import _native

    return _native.device(), _native


def _run(A, a_mn, B, b_mn, C, M, N, K, epi=0, bn=256, alpha=1.0, stamps=None, stamp=0):
    import torch

    lib, nat = _lib()
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.pf_gemm_bf16(A.data_ptr(), int(a_mn), A.stride(0), B.data_ptr(), int(b_mn), B.stride(0),
                          C.data_ptr(), C.stride(0), M, N, K, alpha, epi, bn,
                          stamps.data_ptr() if stamps is not None else None, stamp, stream)
    nat.check(rc, "pf_gemm_bf16")
    torch.cuda.synchronize()


def _ref(A, a_mn, B, b_mn):
    a = (A.t() if a_mn else A).float()
    b = (B.t() if b_mn else B).float()
    return a @ b.t()


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("bn", [256, 128])
@pytest.mark.parametrize("M,N,K", [(256, 512, 320), (296, 392, 200), (128, 256, 64), (1024, 768, 1024)])
def test_gemm_store_bf16(cuda, a_mn, b_mn, bn, M, N, K):
    import torch

    g = torch.Generator(device="cpu").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn((K, M) if a_mn else (M, K), generator=g).to(torch.bfloat16).cuda()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g).to(torch.bfloat16).cuda()
    C = torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    _run(A, a_mn, B, b_mn, C, M, N, K, epi=0, bn=bn)
    ref = _ref(A, a_mn, B, b_mn)
    err = (C.float() - ref).abs().max().item()
    tol = 1e-2 * ref.abs().max().item() + 1e-2
    assert err <= tol, f"max err {err} > {tol}"


@pytest.mark.parametrize("epi", [1, 3])
def test_gemm_add_and_f32(cuda, epi):
    import torch

    M, N, K = 384, 512, 448
    g = torch.Generator(device="cpu").manual_seed(5)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(K, N, generator=g).to(torch.bfloat16).cuda()
    ref = _ref(A, 0, B, 1) * 0.5
    if epi == 1:
        C0 = torch.randn(M, N, generator=g).to(torch.bfloat16).cuda()
        C = C0.clone()
        _run(A, 0, B, 1, C, M, N, K, epi=1, alpha=0.5)
        ref = ref + C0.float()
        assert (C.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item() + 1e-2
    else:
        C = torch.zeros(M, N, dtype=torch.float32, device=cuda)
        _run(A, 0, B, 1, C, M, N, K, epi=3, alpha=0.5)
        assert (C - ref).abs().max().item() <= 1e-4 * ref.abs().max().item()


def test_gemm_dw_unit_list_accumulates(cuda):
    """dW over unit lists: first touch stores, later microbatches accumulate; untouched units keep stale data."""
    import torch

    lib, nat = _lib()
    T, O, I = 512, 384, 512  # dY [T, O], X [T, I] -> G [O, I], 3 x 4 units
    g = torch.Generator(device="cpu").manual_seed(11)
    G = torch.full((O, I), 7.0, dtype=torch.float32, device=cuda)
    stamps = torch.zeros(3 * 4, dtype=torch.int32, device=cuda)
    expect = torch.full((O, I), 7.0, dtype=torch.float64)
    lists = [[0, 5, 6, 11], [5, 1, 11], [2]]
    stream = torch.cuda.current_stream().cuda_stream
    seen = set()
    for units in lists:
        dY = torch.randn(T, O, generator=g).to(torch.bfloat16).cuda()
        X = torch.randn(T, I, generator=g).to(torch.bfloat16).cuda()
        ul = torch.tensor(units, dtype=torch.int32, device=cuda)
        cnt = torch.tensor([len(units)], dtype=torch.int32, device=cuda)
        rc = lib.pf_gemm_dw_units(dY.data_ptr(), 1, dY.stride(0), X.data_ptr(), 1, X.stride(0), G.data_ptr(),
                                  G.stride(0), O, I, T, 1.0, ul.data_ptr(), cnt.data_ptr(), 12,
                                  stamps.data_ptr(), 0, 42, stream)
        nat.check(rc, "pf_gemm_dw_units")
        full = dY.double().cpu().t() @ X.double().cpu()
        for u in units:
            r, c = divmod(u, 4)
            blk = full[r * 128:(r + 1) * 128, c * 128:(c + 1) * 128]
            if u in seen:
                expect[r * 128:(r + 1) * 128, c * 128:(c + 1) * 128] += blk
            else:
                expect[r * 128:(r + 1) * 128, c * 128:(c + 1) * 128] = blk
        seen |= set(units)
    torch.cuda.synchronize()
    err = (G.double().cpu() - expect).abs().max().item()
    assert err <= 1e-3 * expect.abs().max().item()
    st = stamps.cpu().tolist()
    for u in range(12):
        assert st[u] == (42 if u in {0, 5, 6, 11, 1, 2} else 0)


@pytest.mark.parametrize("T,O,I", [(512, 384, 512), (320, 1000, 392), (1024, 4608, 384), (256, 256, 4608)])
def test_gemm_dw_rowpairs_accumulates(cuda, T, O, I):
    """Row-pair dW (128 x 256 MMA over two units of one row, a single 128 x 128 for an odd row):
    first touch stores, later microbatches accumulate, untouched units keep stale data; O = 1000
    has a partial row block, I = 392 a partial column block."""
    import numpy as np
    import torch

    from test_kernels_gpu import rowpair_list_ref

    lib, nat = _lib()
    tm, tn = -(-O // 128), -(-I // 128)
    U = tm * tn
    g = torch.Generator(device="cpu").manual_seed(T + O + I + 1)
    rng = np.random.default_rng(O + 1)
    G = torch.full((O, I), 7.0, dtype=torch.float32, device=cuda)
    stamps = torch.zeros(U, dtype=torch.int32, device=cuda)
    expect = torch.full((O, I), 7.0, dtype=torch.float64)
    stream = torch.cuda.current_stream().cuda_stream
    seen = set()
    for frac in (0.3, 0.55, 0.9, 0.0):
        frozen = rng.random(U) < frac
        ents = rowpair_list_ref(frozen, tm, tn)
        units = [u for u in ents if u >= 0]
        dY = torch.randn(T, O, generator=g).to(torch.bfloat16).cuda()
        X = torch.randn(T, I, generator=g).to(torch.bfloat16).cuda()
        el = torch.tensor(ents + [0, 0], dtype=torch.int32, device=cuda)
        cnt = torch.tensor([len(ents) // 2], dtype=torch.int32, device=cuda)
        rc = lib.pf_gemm_dw_rowpairs(dY.data_ptr(), dY.stride(0), X.data_ptr(), X.stride(0), G.data_ptr(),
                                     G.stride(0), O, I, T, el.data_ptr(), cnt.data_ptr(), stamps.data_ptr(), 0, 42,
                                     stream)
        nat.check(rc, "pf_gemm_dw_rowpairs")
        full = dY.double().cpu().t() @ X.double().cpu()
        for u in units:
            r, c = divmod(u, tn)
            rs, cs = slice(r * 128, min(O, r * 128 + 128)), slice(c * 128, min(I, c * 128 + 128))
            expect[rs, cs] = expect[rs, cs] + full[rs, cs] if u in seen else full[rs, cs]
        seen |= set(units)
    torch.cuda.synchronize()
    err = (G.double().cpu() - expect).abs().max().item()
    assert err <= 1e-3 * expect.abs().max().item()
    st = stamps.cpu().tolist()
    for u in range(U):
        assert st[u] == (42 if u in seen else 0)


@pytest.mark.parametrize("T,O,I", [(512, 384, 512), (320, 1000, 256), (1024, 4608, 384)])
def test_gemm_dw_pairs_accumulates(cuda, T, O, I):
    """CTA-pair dW over K5p pair lists: first touch stores, later microbatches accumulate,
    -1 partners write nothing, untouched units keep stale data; O = 1000 has a partial row
    block, O = 4608 spans two 32-row bands."""
    import numpy as np
    import torch

    from test_kernels_gpu import pair_list_ref

    lib, nat = _lib()
    tm, tn = -(-O // 128), -(-I // 128)
    U = tm * tn
    g = torch.Generator(device="cpu").manual_seed(T + O + I)
    rng = np.random.default_rng(O)
    G = torch.full((O, I), 7.0, dtype=torch.float32, device=cuda)
    stamps = torch.zeros(U, dtype=torch.int32, device=cuda)
    expect = torch.full((O, I), 7.0, dtype=torch.float64)
    stream = torch.cuda.current_stream().cuda_stream
    seen = set()
    for frac in (0.3, 0.55, 0.9):
        frozen = rng.random(U) < frac
        plist = pair_list_ref(frozen, tm, tn)
        units = [u for u in plist if u >= 0]
        dY = torch.randn(T, O, generator=g).to(torch.bfloat16).cuda()
        X = torch.randn(T, I, generator=g).to(torch.bfloat16).cuda()
        pl = torch.tensor(plist + [0], dtype=torch.int32, device=cuda)
        cnt = torch.tensor([len(plist)], dtype=torch.int32, device=cuda)
        rc = lib.pf_gemm_dw_pairs(dY.data_ptr(), dY.stride(0), X.data_ptr(), X.stride(0), G.data_ptr(), G.stride(0),
                                  O, I, T, pl.data_ptr(), cnt.data_ptr(), stamps.data_ptr(), 0, 42, stream)
        nat.check(rc, "pf_gemm_dw_pairs")
        full = dY.double().cpu().t() @ X.double().cpu()
        for u in units:
            r, c = divmod(u, tn)
            rs, cs = slice(r * 128, min(O, r * 128 + 128)), slice(c * 128, min(I, c * 128 + 128))
            expect[rs, cs] = expect[rs, cs] + full[rs, cs] if u in seen else full[rs, cs]
        seen |= set(units)
    torch.cuda.synchronize()
    err = (G.double().cpu() - expect).abs().max().item()
    assert err <= 1e-3 * expect.abs().max().item()
    st = stamps.cpu().tolist()
    for u in range(U):
        assert st[u] == (42 if u in seen else 0)


@pytest.mark.parametrize("pad", [0, 4, 8])
@pytest.mark.parametrize("epi", [0, 1])
def test_gemm_cta_pair_strided_c(cuda, pad, epi):
    """C with row stride N + pad through the TMA-staged epilogue (pad 0, 8) equals the fp32 reference
    and leaves the padding columns alone; rows that are not 16-byte aligned (pad 4) are rejected
    with PF_ERR_INVALID before any launch."""
    import torch

    lib, nat = _lib()
    M, N, K = 512, 768, 256
    g = torch.Generator(device="cpu").manual_seed(pad * 10 + epi)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(N, K, generator=g).to(torch.bfloat16).cuda()
    base = torch.randn(M, N + pad, generator=g).to(torch.bfloat16).cuda()
    C = base.clone()
    rc = lib.pf_gemm_bf16(A.data_ptr(), 0, K, B.data_ptr(), 0, K, C.data_ptr(), N + pad, M, N, K, 1.0, epi, 512,
                          None, 0, torch.cuda.current_stream().cuda_stream)
    if pad % 8:
        assert rc == 4  # PF_ERR_INVALID
        return
    nat.check(rc, "pf_gemm_bf16")
    torch.cuda.synchronize()
    ref = _ref(A, 0, B, 0) + (base[:, :N].float() if epi == 1 else 0)
    assert (C[:, :N].float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item() + 1e-2
    assert torch.equal(C[:, N:], base[:, N:])  # padding columns untouched


@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("epi", [0, 1, 3])
@pytest.mark.parametrize("M,N,K", [(256, 512, 320), (512, 768, 1024), (296, 392, 200), (1024, 2048, 512)])
def test_gemm_cta_pair(cuda, b_mn, epi, M, N, K):
    """CTA-pair kernel (tcgen05.mma.cta_group::2, 256x256 tiles) through block_n=512."""
    import torch

    g = torch.Generator(device="cpu").manual_seed(M + N + K + epi)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g).to(torch.bfloat16).cuda()
    ref = _ref(A, 0, B, b_mn)
    if epi == 3:
        C = torch.zeros(M, N, dtype=torch.float32, device=cuda)
        _run(A, 0, B, b_mn, C, M, N, K, epi=3, bn=512)
        assert (C - ref).abs().max().item() <= 1e-4 * ref.abs().max().item()
        return
    C0 = torch.randn(M, N, generator=g).to(torch.bfloat16).cuda() if epi == 1 else torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
    C = C0.clone()
    _run(A, 0, B, b_mn, C, M, N, K, epi=epi, bn=512)
    if epi == 1:
        ref = ref + C0.float()
    assert (C.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item() + 1e-2


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("epi", [0, 1, 3])
@pytest.mark.parametrize("M,N,K", [(4096, 2048, 1024), (2048, 2560, 832), (4352, 2304, 512), (4096, 2048, 8192),
                                   (3200, 1024, 1024), (3200, 1024, 4096)])
def test_gemm_cta_pair_stream_k(cuda, mode, b_mn, epi, M, N, K):
    """Forced stream-K on tile counts just above the 74 clusters (and, mode 1 only, the 52-tile ViT
    N = 1024 shapes below one wave): mode 1 splits every tile, mode 2
    runs the full waves data-parallel and splits the last wave's tiles over all clusters (a tile
    then spans up to three clusters: its head adds every parked piece)."""
    lib, nat = _lib()
    nat.check(lib.pf_gemm_set_streamk(mode), "pf_gemm_set_streamk")
    try:
        _stream_k_case(cuda, b_mn, epi, M, N, K)
    finally:
        lib.pf_gemm_set_streamk(0)


def _stream_k_case(cuda, b_mn, epi, M, N, K):
    import torch

    g = torch.Generator(device="cpu").manual_seed(M * 3 + N + K + epi)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn((K, N) if b_mn else (N, K), generator=g).to(torch.bfloat16).cuda()
    ref = _ref(A, 0, B, b_mn)
    for _ in range(2):  # back-to-back launches reuse the workspace (epoch-tagged flags)
        if epi == 3:
            C = torch.zeros(M, N, dtype=torch.float32, device=cuda)
            _run(A, 0, B, b_mn, C, M, N, K, epi=3, bn=512)
            assert (C - ref).abs().max().item() <= 1e-4 * ref.abs().max().item()
            continue
        C0 = torch.randn(M, N, generator=g).to(torch.bfloat16).cuda() if epi == 1 else torch.zeros(M, N, dtype=torch.bfloat16, device=cuda)
        C = C0.clone()
        _run(A, 0, B, b_mn, C, M, N, K, epi=epi, bn=512)
        r = ref + C0.float() if epi == 1 else ref
        assert (C.float() - r).abs().max().item() <= 1e-2 * r.abs().max().item() + 1e-2


@pytest.mark.parametrize("T,O,I", [(512, 384, 512), (320, 1000, 392), (1024, 4608, 384), (256, 256, 4608)])
def test_gemm_dw_dense_accumulates(cuda, T, O, I):
    """Dense-cell dW (256 x 256 CTA-pair tiles over every unit, no list): the first touch of a unit in
    a step stores, later calls accumulate; odd unit-row / unit-column counts (O = 1000 -> 8 row
    blocks with a partial one, I = 392 / 384 -> 4 / 3 column blocks) exercise the edge tiles."""
    import numpy as np
    import torch

    lib, nat = _lib()
    tm, tn = -(-O // 128), -(-I // 128)
    U = tm * tn
    g = torch.Generator(device="cpu").manual_seed(T + O + I + 7)
    G = torch.full((O, I), 7.0, dtype=torch.float32, device=cuda)
    stamps = torch.zeros(U, dtype=torch.int32, device=cuda)
    stamps[: U // 2] = 42  # half the units already touched this step: those accumulate
    expect = G.double().cpu().clone()
    touched = np.zeros(U, dtype=bool)
    touched[: U // 2] = True
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        dY = torch.randn(T, O, generator=g).to(torch.bfloat16).cuda()
        X = torch.randn(T, I, generator=g).to(torch.bfloat16).cuda()
        nat.check(lib.pf_gemm_dw_dense(dY.data_ptr(), dY.stride(0), X.data_ptr(), X.stride(0), G.data_ptr(),
                                       G.stride(0), O, I, T, stamps.data_ptr(), 0, 42, stream), "pf_gemm_dw_dense")
        full = dY.double().cpu().t() @ X.double().cpu()
        for u in range(U):
            r, c = divmod(u, tn)
            rs, cs = slice(r * 128, min(O, r * 128 + 128)), slice(c * 128, min(I, c * 128 + 128))
            expect[rs, cs] = expect[rs, cs] + full[rs, cs] if touched[u] else full[rs, cs]
            touched[u] = True
    torch.cuda.synchronize()
    err = (G.double().cpu() - expect).abs().max().item()
    assert err <= 1e-3 * expect.abs().max().item(), err
    assert stamps.cpu().tolist() == [42] * U
