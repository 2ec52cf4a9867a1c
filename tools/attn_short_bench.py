"""Times the attention kernels on the C2 short-chunk shape: chunk 0 of the C2
block's packed short sequences (~8K queries in ~35 segments, 32 q heads,
8 kv heads, head_dim 128), through cf_op_attention; algorithmic TFLOP/s."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_02356_b200 as cf  # noqa: E402
from paper_2503_02356_b200 import capi  # noqa: E402

H, KVH, dh = 32, 8, 128
short = capi.synthesize(999, 1, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)
plan = cf.Plan.build(short, 8192, 1)
ch, sg, _, _ = plan.export()
c0 = ch[int(sys.argv[1]) if len(sys.argv) > 1 else 0]  # chunk index (FFD order: 0 holds the longest shorts)
lens = [int(x["length"]) for x in sg[c0["seg_offset"]:c0["seg_offset"] + c0["seg_count"]]]
segs, q0 = [], 0
for L in lens:
    segs.append((q0, L, q0, 0))
    q0 += L
T = R = q0
pairs = sum(L * (L + 1) / 2 for L in lens)
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
print(f"T={T} segments={len(lens)} mean={np.mean(lens):.0f} pairs={pairs:.3e}")


def run(impl, bwd):
    ctx.attention(impl, bwd, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, R, o.data_ptr(),
                  lse.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), KVH * dh, segs, T, H,
                  KVH, dh)


for name, impl, bwd, fl in (("fwd tcgen05 ping-pong", 3, False, 4), ("fwd tcgen05", 1, False, 4), 
                            ("fwd mma.sync", 0, False, 4), ("bwd tcgen05", 1, True, 8), ("bwd mma.sync", 0, True, 8)):
    run(1, False)
    run(impl, bwd)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 20
    for _ in range(n):
        run(impl, bwd)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{name:24s} {dt * 1e6:8.1f} us  {fl * H * dh * pairs / dt / 1e12:7.1f} TFLOP/s (algorithmic)", flush=True)
