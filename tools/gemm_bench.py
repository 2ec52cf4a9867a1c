"""Times the tcgen05 GEMM at the C2 per-layer shapes (T = 8192 tokens of one
chunk, Llama-7B-shaped layer) through cf_op_gemm; TFLOP/s per shape."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2503_02356_b200 as cf  # noqa: E402
from paper_2503_02356_b200 import capi  # noqa: E402

T, d, kvw, ffn = 8192, 4096, 1024, 11008
ctx = cf.Context(0)
SH = [  # name, M, N, K, a_kmajor, b_kmajor, epi
    ("qkv fwd", T, d + 2 * kvw, d, 1, 0, capi.EPI_BF16),
    ("gate|up fwd", T, 2 * ffn, d, 1, 0, capi.EPI_BF16),
    ("down fwd +res", T, d, ffn, 1, 0, capi.EPI_F32_RES),
    ("o fwd +res", T, d, d, 1, 0, capi.EPI_F32_RES),
    ("o fwd bf16-out", T, d, d, 1, 0, capi.EPI_BF16),
    ("o fwd f32-out", T, d, d, 1, 0, capi.EPI_F32),
    ("down dgrad", T, ffn, d, 1, 1, capi.EPI_BF16),
    ("gate|up dgrad", T, d, 2 * ffn, 1, 1, capi.EPI_F32),
    ("gate|up wgrad", d, 2 * ffn, T, 0, 0, capi.EPI_F32_ACC),
    ("down wgrad", ffn, d, T, 0, 0, capi.EPI_F32_ACC),
    ("qkv wgrad", d, d + 2 * kvw, T, 0, 0, capi.EPI_F32_ACC),
    ("head fwd", T, 32000, d, 1, 0, capi.EPI_F32),
    ("head dgrad", T, d, 32000, 1, 1, capi.EPI_F32),
    ("head wgrad", d, 32000, T, 0, 0, capi.EPI_F32_ACC),
]
ONCE = os.environ.get("GEMM_BENCH_ONCE") == "1"
only = sys.argv[1] if len(sys.argv) > 1 else None
for name, M, N, K, ak, bk, epi in SH:
    if only and only not in name:
        continue
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16) if ak else torch.randn(K, M, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16) if bk else torch.randn(K, N, device="cuda").to(torch.bfloat16)
    f32 = epi in (capi.EPI_F32, capi.EPI_F32_ACC, capi.EPI_F32_RES)
    C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    R = torch.zeros(M, N, device="cuda") if epi == capi.EPI_F32_RES else None
    args = (A.data_ptr(), ak, A.shape[1], B.data_ptr(), bk, B.shape[1], C.data_ptr(), N, M, N, K, epi,
            R.data_ptr() if R is not None else 0, N)
    torch.cuda.synchronize()
    if ONCE:  # one launch per shape, for an ncu capture with known shapes
        ctx.gemm(*args)
        ctx.synchronize()
        io = (M * K + N * K) * 2 + M * N * (4 if f32 else 2) * (2 if epi in (capi.EPI_F32_ACC, capi.EPI_F32_RES) else 1)
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "algorithmic_bytes": io}), flush=True)
        continue
    for _ in range(2):
        ctx.gemm(*args)
    ctx.synchronize()
    s = torch.cuda.ExternalStream(ctx.stream)
    # SUSTAIN=seconds: back-to-back launches for that long (power-capped
    # rate, as the sustained peak in MEASURED_PEAKS.json), else 10 launches
    sustain = float(os.environ.get("SUSTAIN", "0"))
    n = max(10, int(sustain * 1e3 / max(1e-3, 2 * M * N * K / 1.2e12))) if sustain else 10

    def timed(fn, stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / n

    ms = timed(lambda: ctx.gemm(*args), s)
    # cuBLAS on the same operand majors (bf16 in, bf16 out), for reference
    a_op = A if ak else A.t()
    b_op = B.t() if bk else B
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    torch.matmul(a_op, b_op, out=out)
    torch.cuda.synchronize()
    ms_cb = timed(lambda: torch.matmul(a_op, b_op, out=out), torch.cuda.current_stream())
    print(f"{name:16s} M={M:6d} N={N:6d} K={K:6d}  {ms:7.3f} ms  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s"
          f"   cuBLAS {ms_cb:7.3f} ms {2 * M * N * K / ms_cb / 1e9:7.1f} TFLOP/s  ratio {ms_cb / ms:5.3f}", flush=True)
