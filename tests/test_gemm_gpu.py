"""tcgen05 GEMM (csrc/kernels/gemm.cu) vs a plain PyTorch fp32 reference of
the same op, over every operand-major combination and epilogue."""
import pytest
import torch

import paper_2503_02356_b200.capi as capi

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 64), (296, 520, 200), (1024, 1536, 1024), (24, 40, 16), (256, 2000, 512), (8192, 1536, 4096)]


def _mk(rows, cols, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(rows, cols, generator=g, device="cuda") * 0.5).to(torch.bfloat16)


@pytest.fixture(params=[1, 2], ids=["single-cta", "cta-pair"])
def gemm_mode(request):
    capi.check(capi.lib().cf_debug_set_gemm_mode(request.param))
    yield request.param
    capi.check(capi.lib().cf_debug_set_gemm_mode(0))


@pytest.mark.parametrize("a_k", [1, 0])
@pytest.mark.parametrize("b_k", [1, 0])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_majors(ctx, gemm_mode, a_k, b_k, shape):
    M, N, K = shape
    A = _mk(M, K, 1) if a_k else _mk(K, M, 1)   # stored [M,K] or [K,M]
    B = _mk(N, K, 2) if b_k else _mk(K, N, 2)   # stored [N,K] or [K,N]
    Am = A.float() if a_k else A.float().t()
    Bm = B.float() if b_k else B.float().t()
    ref = Am @ Bm.t()
    ldc = (N + 7) // 8 * 8
    C = torch.zeros(M, ldc, device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    ctx.gemm(A.data_ptr(), a_k, A.shape[1], B.data_ptr(), b_k, B.shape[1], C.data_ptr(), ldc, M, N, K, capi.EPI_F32)
    ctx.synchronize()
    err = (C[:, :N] - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err   # fp32 accumulation of exact bf16 products


@pytest.mark.parametrize("epi", [capi.EPI_BF16, capi.EPI_F32_ACC, capi.EPI_F32_RES, capi.EPI_BF16_TANH,
                                 capi.EPI_BF16_TANHGRAD])
def test_gemm_epilogues(ctx, gemm_mode, epi):
    M, N, K = 384, 768, 320
    A = _mk(M, K, 3)
    B = _mk(K, N, 4)  # reference [in,out] weight layout (N-major B)
    ref = A.float() @ B.float()
    R32 = torch.randn(M, N, device="cuda")
    Rbf = (torch.rand(M, N, device="cuda") * 0.9).to(torch.bfloat16)
    if epi in (capi.EPI_BF16, capi.EPI_BF16_TANH, capi.EPI_BF16_TANHGRAD):
        C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    else:
        C = R32.clone() if epi == capi.EPI_F32_ACC else torch.zeros(M, N, device="cuda")
    r_ptr = R32.data_ptr() if epi == capi.EPI_F32_RES else (Rbf.data_ptr() if epi == capi.EPI_BF16_TANHGRAD else 0)
    torch.cuda.synchronize()
    ctx.gemm(A.data_ptr(), 1, K, B.data_ptr(), 0, N, C.data_ptr(), N, M, N, K, epi, r_ptr, N)
    ctx.synchronize()
    expect = {capi.EPI_BF16: ref, capi.EPI_F32_ACC: ref + R32, capi.EPI_F32_RES: ref + R32,
              capi.EPI_BF16_TANH: torch.tanh(ref),
              capi.EPI_BF16_TANHGRAD: ref * (1 - Rbf.float() ** 2)}[epi]
    err = (C.float() - expect).abs().max().item() / expect.abs().max().item()
    assert err < (1e-2 if C.dtype == torch.bfloat16 else 1e-5), err


def test_gemm_residual_aliases_output(ctx, gemm_mode):
    """x += O @ Wo with the residual read and written in place (EPI_F32_RES)."""
    M, N, K = 257, 512, 512
    A = _mk(M, K, 5)
    B = _mk(K, N, 6)
    X = torch.randn(M, N, device="cuda")
    ref = X + A.float() @ B.float()
    torch.cuda.synchronize()
    ctx.gemm(A.data_ptr(), 1, K, B.data_ptr(), 0, N, X.data_ptr(), N, M, N, K, capi.EPI_F32_RES, X.data_ptr(), N)
    ctx.synchronize()
    assert (X - ref).abs().max().item() / ref.abs().max().item() < 1e-5


@pytest.mark.parametrize("shape,mode", [((384, 512, 320), 2), ((2048, 2048, 512), 0), ((8192, 22016, 4096), 0)],
                         ids=["small-forced-pair", "auto", "c2-gate-up"])
def test_gemm_swiglu_epilogue(ctx, shape, mode):
    """EPI_BF16_SWIGLU: gate|up written exactly as EPI_BF16 writes them, plus
    h = silu(gate) * up of the rounded values in the same epilogue."""
    M, N, K = shape
    F = N // 2
    capi.check(capi.lib().cf_debug_set_gemm_mode(mode))
    try:
        A = _mk(M, K, 7)
        B = _mk(K, N, 8)
        C0 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        C1 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        H = torch.zeros(M, F, device="cuda", dtype=torch.bfloat16)
        torch.cuda.synchronize()
        ctx.gemm(A.data_ptr(), 1, K, B.data_ptr(), 0, N, C0.data_ptr(), N, M, N, K, capi.EPI_BF16)
        ctx.gemm(A.data_ptr(), 1, K, B.data_ptr(), 0, N, C1.data_ptr(), N, M, N, K, capi.EPI_BF16_SWIGLU,
                 H.data_ptr(), F)
        ctx.synchronize()
    finally:
        capi.check(capi.lib().cf_debug_set_gemm_mode(0))
    assert torch.equal(C0, C1)
    g, u = C0[:, :F].float(), C0[:, F:].float()
    ref = g * torch.sigmoid(g) * u
    err = (H.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err


@pytest.mark.parametrize("shape,mode", [((384, 768, 256), 2), ((8192, 6144, 4096), 0)], ids=["forced-pair", "c2-qkv"])
def test_gemm_rope_epilogue(ctx, shape, mode):
    """EPI_BF16_ROPE: rotate-half RoPE on the q and k heads of the bf16-rounded
    q|k|v GEMM output, v untouched, k / v copied to the KV-cache rows."""
    M, N, K = shape
    col_k, col_v = (256, 512) if N == 768 else (4096, 5120)
    kvw = N - col_v
    capi.check(capi.lib().cf_debug_set_gemm_mode(mode))
    try:
        A = _mk(M, K, 12)
        B = _mk(K, N, 13)
        pos = torch.arange(M, device="cuda", dtype=torch.float64) + 7
        f = 10000.0 ** (-2.0 * torch.arange(64, device="cuda", dtype=torch.float64) / 128)
        ang = pos[:, None] * f[None, :]
        tab = torch.stack([torch.cos(ang), torch.sin(ang)], -1).float().contiguous()  # [M][64] (cos, sin)
        C0 = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        C1 = torch.zeros_like(C0)
        kc = torch.zeros(M, kvw, device="cuda", dtype=torch.bfloat16)
        vc = torch.zeros_like(kc)
        torch.cuda.synchronize()
        ctx.gemm(A.data_ptr(), 1, K, B.data_ptr(), 0, N, C0.data_ptr(), N, M, N, K, capi.EPI_BF16)
        capi.check(capi.lib().cf_op_gemm_rope(ctx.h, capi.C.c_void_p(A.data_ptr()), capi.C.c_int64(K),
                                              capi.C.c_void_p(B.data_ptr()), capi.C.c_int64(N),
                                              capi.C.c_void_p(C1.data_ptr()), capi.C.c_int64(M), capi.C.c_int64(N),
                                              capi.C.c_int64(K), capi.C.c_void_p(tab.data_ptr()),
                                              capi.C.c_int64(col_k), capi.C.c_int64(col_v),
                                              capi.C.c_void_p(kc.data_ptr()), capi.C.c_void_p(vc.data_ptr()),
                                              capi.C.c_int64(kvw)))
        ctx.synchronize()
    finally:
        capi.check(capi.lib().cf_debug_set_gemm_mode(0))
    x = C0.float()
    ref = x.clone()
    cs, sn = tab[..., 0], tab[..., 1]
    for h0 in range(0, col_v, 128):
        a, b = x[:, h0:h0 + 64], x[:, h0 + 64:h0 + 128]
        ref[:, h0:h0 + 64] = a * cs - b * sn
        ref[:, h0 + 64:h0 + 128] = b * cs + a * sn
    err = (C1.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-2, err
    assert torch.equal(C1[:, col_v:], C0[:, col_v:])
    assert torch.equal(kc, C1[:, col_k:col_v]) and torch.equal(vc, C1[:, col_v:])


@pytest.mark.parametrize("shape", [(8192, 32000, 4096), (300, 97, 64), (1000, 9000, 256), (130, 152064, 128),
                                   (77, 520, 96)], ids=["c2", "odd-v", "v9000", "qwen-vocab", "small"])
def test_fused_lm_head_ce(ctx, gemm_mode, shape):
    """LM head + cross-entropy fused into the head GEMM (EPI_CE_STATS partials
    + ce_finish, EPI_CE_GRAD dlogits from the LSE) vs torch fp32 on the same
    bf16 operands: LSE / row loss to 1e-5 relative, dlogits to bf16 rounding
    (toy_model.hpp:320-331, :369-388)."""
    T, V, d = shape
    ldh = (V + 7) // 8 * 8
    x = _mk(T, d, 5) * 0.3
    W = torch.zeros(d, ldh, device="cuda", dtype=torch.bfloat16)
    W[:, :V] = _mk(d, V, 6) * 0.3
    g = torch.Generator(device="cuda").manual_seed(7)
    tgt = torch.randint(0, V, (T,), generator=g, device="cuda", dtype=torch.int32)
    tgt[::5] = -1  # rows without a target
    logits = x.float() @ W[:, :V].float()
    lse_ref = torch.logsumexp(logits, dim=1)
    has = tgt >= 0
    loss_ref = torch.where(has, lse_ref - logits.gather(1, tgt.clamp(min=0).long()[:, None])[:, 0],
                           torch.zeros_like(lse_ref))
    inv = 1.0 / 12345.0
    p = torch.softmax(logits, dim=1)
    p[has, tgt[has].long()] -= 1.0
    dl_ref = torch.where(has[:, None], p * inv, torch.zeros_like(p))
    lse = torch.zeros(T, device="cuda")
    loss = torch.zeros(T, device="cuda")
    dl = torch.full((T, ldh), 7.0, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    ctx.lm_head_ce(x.data_ptr(), W.data_ptr(), ldh, T, V, d, tgt.data_ptr(), inv, lse.data_ptr(), loss.data_ptr(),
                   dl.data_ptr())
    ctx.synchronize()
    assert ((lse - lse_ref).abs() / lse_ref.abs().clamp(min=1)).max().item() < 1e-5
    assert ((loss - loss_ref).abs() / loss_ref.abs().clamp(min=1)).max().item() < 1e-5
    err = (dl[:, :V].float() - dl_ref).abs().max().item() / dl_ref.abs().max().item()
    assert err < 1e-2, err  # bf16 storage of the gradient
    assert (dl[~has, :V] == 0).all()
