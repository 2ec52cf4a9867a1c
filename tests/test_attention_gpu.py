"""Chunked attention kernels (packed segments + KV prefix + GQA) vs a plain
PyTorch fp32 reference of the same op (reference semantics:
toy_model.hpp:263-302 forward, :436-486 backward)."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(q, k, v, segs, H, KVH, dh):
    """fp32 reference: O [T, H*dh], LSE [H, T] for the listed segments."""
    T = q.shape[0]
    O = torch.zeros(T, H * dh, device="cuda")
    L = torch.zeros(H, T, device="cuda")
    per = H // KVH
    for qs, ln, kv0, pre in segs:
        qq = q[qs:qs + ln].float().view(ln, H, dh)
        kk = k[kv0:kv0 + pre + ln].float().view(pre + ln, KVH, dh)
        vv = v[kv0:kv0 + pre + ln].float().view(pre + ln, KVH, dh)
        kk = kk.repeat_interleave(per, dim=1)
        vv = vv.repeat_interleave(per, dim=1)
        s = torch.einsum("qhd,khd->hqk", qq, kk) / math.sqrt(dh)
        qi = torch.arange(ln, device="cuda")[:, None]
        kj = torch.arange(pre + ln, device="cuda")[None, :]
        s = s.masked_fill(kj > pre + qi, float("-inf"))
        L[:, qs:qs + ln] = torch.logsumexp(s, dim=-1)
        p = torch.softmax(s, dim=-1)
        O[qs:qs + ln] = torch.einsum("hqk,khd->qhd", p, vv).reshape(ln, H * dh)
    return O, L


CASES = {
    "dependent-prefix": dict(H=4, KVH=2, dh=128, T=200, R=500, segs=[(0, 200, 0, 300)]),
    "packed-standalone": dict(H=4, KVH=1, dh=128, T=485, R=485,
                              segs=[(0, 50, 0, 0), (50, 128, 50, 0), (178, 300, 178, 0), (478, 7, 478, 0)]),
    "long-prefix": dict(H=2, KVH=2, dh=128, T=256, R=4096 + 256, segs=[(0, 256, 0, 4096)]),
    "dh64": dict(H=4, KVH=2, dh=64, T=300, R=300, segs=[(0, 100, 0, 0), (100, 200, 100, 0)]),
}


def _inputs(c, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    H, KVH, dh, T, R = c["H"], c["KVH"], c["dh"], c["T"], c["R"]
    q = (torch.randn(T, H * dh, generator=g, device="cuda")).to(torch.bfloat16)
    k = (torch.randn(R, KVH * dh, generator=g, device="cuda")).to(torch.bfloat16)
    v = (torch.randn(R, KVH * dh, generator=g, device="cuda")).to(torch.bfloat16)
    return q, k, v


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("impl", [0, 1, 3])
def test_attention_forward(ctx, name, impl):
    c = CASES[name]
    if impl in (1, 3) and c["dh"] != 128 or (impl == 3 and (c["H"] // c["KVH"]) % 2):
        pytest.skip("tcgen05 path is head_dim 128")
    H, KVH, dh, T, R = c["H"], c["KVH"], c["dh"], c["T"], c["R"]
    q, k, v = _inputs(c)
    o = torch.zeros(T, H * dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(H, T, device="cuda")
    torch.cuda.synchronize()
    ctx.attention(impl, False, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, R, o.data_ptr(),
                  lse.data_ptr(), 0, 0, 0, 0, 0, c["segs"], T, H, KVH, dh)
    O, L = _ref(q, k, v, c["segs"], H, KVH, dh)
    covered = torch.zeros(T, dtype=torch.bool, device="cuda")
    for qs, ln, _, _ in c["segs"]:
        covered[qs:qs + ln] = True
    err = (o.float() - O)[covered].abs().max().item()
    assert err < 2e-2, err
    assert (lse - L)[:, covered].abs().max().item() < 2e-3


@pytest.mark.parametrize("name", ["dependent-prefix", "packed-standalone", "long-prefix", "dh64"])
@pytest.mark.parametrize("impl", [0, 1, 2])
def test_attention_backward(ctx, name, impl):
    c = CASES[name]
    if impl in (1, 2) and c["dh"] != 128:
        pytest.skip("tcgen05 path is head_dim 128")
    H, KVH, dh, T, R = c["H"], c["KVH"], c["dh"], c["T"], c["R"]
    q, k, v = _inputs(c, 1)
    g = torch.Generator(device="cuda").manual_seed(7)
    dout = torch.randn(T, H * dh, generator=g, device="cuda").to(torch.bfloat16)
    o = torch.zeros(T, H * dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(H, T, device="cuda")
    dq = torch.zeros(T, H * dh, device="cuda", dtype=torch.bfloat16)
    dk = torch.zeros(R, KVH * dh, device="cuda")
    dv = torch.zeros(R, KVH * dh, device="cuda")
    torch.cuda.synchronize()
    ctx.attention(0, False, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, R, o.data_ptr(),
                  lse.data_ptr(), 0, 0, 0, 0, 0, c["segs"], T, H, KVH, dh)
    ctx.attention(impl, True, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, R, o.data_ptr(),
                  lse.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), KVH * dh,
                  c["segs"], T, H, KVH, dh)
    qf, kf, vf = (x.float().requires_grad_(True) for x in (q, k, v))
    O, _ = _ref(qf, kf, vf, c["segs"], H, KVH, dh)
    O.backward(dout.float())
    for got, ref in ((dq.float(), qf.grad), (dk, kf.grad), (dv, vf.grad)):
        err = (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-6)
        assert err < 3e-2, err
