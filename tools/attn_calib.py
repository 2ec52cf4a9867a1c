"""Calibration: our tcgen05 attention vs torch SDPA (cuDNN / flash backends,
library kernels) on the same causal self-attention shape, so the attention
roofline fractions have a B200 library figure beside them.  Shape: one
sequence of T tokens, 32 q heads, 8 kv heads, head_dim 128, causal."""
import sys
import time

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
import paper_2503_02356_b200 as cf  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
H, KVH, dh = 32, 8, 128
pairs = T * (T + 1) / 2
fl_f, fl_b = 4 * H * dh * pairs, 8 * H * dh * pairs


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


ctx = cf.Context(0)
q = (torch.randn(T, H * dh, device="cuda") * 0.5).to(torch.bfloat16)
k = (torch.randn(T, KVH * dh, device="cuda") * 0.5).to(torch.bfloat16)
v = torch.randn(T, KVH * dh, device="cuda").to(torch.bfloat16)
dout = torch.randn(T, H * dh, device="cuda").to(torch.bfloat16)
o = torch.zeros(T, H * dh, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(H, T, device="cuda")
dq = torch.zeros_like(o)
dk = torch.zeros(T, KVH * dh, device="cuda")
dv = torch.zeros(T, KVH * dh, device="cuda")
segs = [(0, T, 0, 0)]


def ours(impl, bwd):
    ctx.attention(impl, bwd, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, T, o.data_ptr(),
                  lse.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), KVH * dh, segs, T, H,
                  KVH, dh)


ours(3, False)
tf = timeit(lambda: ours(3, False))
tb = timeit(lambda: ours(1, True))
print(f"ours   T={T}: fwd {tf*1e3:7.2f} ms {fl_f/tf/1e12:7.1f} TF | bwd {tb*1e3:7.2f} ms {fl_b/tb/1e12:7.1f} TF "
      f"(algorithmic 4/8*H*dh per pair)", flush=True)

import os  # noqa: E402

if os.environ.get("NO_SDPA"):
    sys.exit(0)
qs = q.view(1, T, H, dh).transpose(1, 2).contiguous().requires_grad_()
ks = k.view(1, T, KVH, dh).transpose(1, 2).contiguous().requires_grad_()
vs = v.view(1, T, KVH, dh).transpose(1, 2).contiguous().requires_grad_()
do = dout.view(1, T, H, dh).transpose(1, 2).contiguous()
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            kk, vv = ks, vs
            gqa = True
            out = F.scaled_dot_product_attention(qs, kk, vv, is_causal=True, enable_gqa=gqa)
            tfw = timeit(lambda: F.scaled_dot_product_attention(qs, kk, vv, is_causal=True, enable_gqa=gqa))

            def fb():
                out = F.scaled_dot_product_attention(qs, kk, vv, is_causal=True, enable_gqa=gqa)
                out.backward(do)

            tfb = timeit(fb)
            tbw = tfb - tfw
        print(f"{name:6s} T={T}: fwd {tfw*1e3:7.2f} ms {fl_f/tfw/1e12:7.1f} TF | bwd {tbw*1e3:7.2f} ms "
              f"{fl_b/tbw/1e12:7.1f} TF", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name:6s}: unavailable ({type(e).__name__}: {str(e)[:120]})", flush=True)
