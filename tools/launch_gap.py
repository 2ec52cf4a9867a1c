"""Back-to-back launch cadence vs kernel duration: times N dependent launches
of one GEMM shape on the library stream with CUDA events; run the same
script under ncu (gpu__time_duration) to get the kernel's own duration.
The difference is the per-launch gap (launch latency + prologue/tail not
overlapped) that programmatic dependent launch could hide.
Usage: python tools/launch_gap.py M N K [n]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2503_02356_b200 as cf  # noqa: E402
from paper_2503_02356_b200 import capi  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 200
ctx = cf.Context(0)
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
args = (A.data_ptr(), 1, K, B.data_ptr(), 0, N, C.data_ptr(), N, M, N, K, capi.EPI_BF16)
for _ in range(5):
    ctx.gemm(*args)
ctx.synchronize()
s = torch.cuda.ExternalStream(ctx.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(n):
    ctx.gemm(*args)
e1.record(s)
e1.synchronize()
print(f"M={M} N={N} K={K}: {e0.elapsed_time(e1) / n * 1e3:8.2f} us per launch (back-to-back, {n} launches)")
