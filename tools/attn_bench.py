"""Times the attention kernels at the C2 long-chunk shape (T=8192 queries of
one dependent chunk with a 32,768-token KV prefix, 32 q heads, 8 kv heads,
head_dim 128) through cf_op_attention; prints algorithmic TFLOP/s."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2503_02356_b200 as cf  # noqa: E402

T, P, H, KVH, dh = 8192, 32768, 32, 8, 128
R = P + T
ctx = cf.Context(0)
q = (torch.randn(T, H * dh, device="cuda") * 0.5).to(torch.bfloat16)
k = (torch.randn(R, KVH * dh, device="cuda") * 0.5).to(torch.bfloat16)
v = torch.randn(R, KVH * dh, device="cuda").to(torch.bfloat16)
dout = torch.randn(T, H * dh, device="cuda").to(torch.bfloat16)
o = torch.zeros(T, H * dh, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(H, T, device="cuda")
dq = torch.zeros_like(o)
dk = torch.zeros(R, KVH * dh, device="cuda")
dv = torch.zeros(R, KVH * dh, device="cuda")
segs = [(0, T, 0, P)]
pairs = T * P + T * (T + 1) / 2
torch.cuda.synchronize()


def run(impl, bwd):
    ctx.attention(impl, bwd, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, R, o.data_ptr(),
                  lse.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), KVH * dh, segs, T, H,
                  KVH, dh)


for name, impl, bwd, fl in (("fwd tcgen05 ping-pong", 3, False, 4), ("fwd tcgen05", 1, False, 4),
                            ("fwd mma.sync", 0, False, 4),
                            ("bwd tcgen05 pipelined", 1, True, 8), ("bwd tcgen05 v1", 2, True, 8),
                            ("bwd mma.sync", 0, True, 8)):
    run(1, False)
    run(impl, bwd)
    t0 = time.perf_counter()
    n = 3
    for _ in range(n):
        run(impl, bwd)
    dt = (time.perf_counter() - t0) / n
    print(f"{name:24s} {dt * 1e3:8.2f} ms  {fl * H * dh * pairs / dt / 1e12:7.1f} TFLOP/s (algorithmic)", flush=True)
