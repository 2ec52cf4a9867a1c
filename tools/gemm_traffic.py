"""Maps the GEMM launches of an ncu capture of one training step (layers 0-1
forward, then head + layer 31 backward: the engine.cu issue order) to their
shapes and writes per-launch DRAM traffic next to the algorithmic bytes
(A + B read once, C written once; +C read for accumulate/residual epilogues).
Usage: python tools/gemm_traffic.py gpurun_out/ncu_summary.json profiles/<round>_gemm_traffic.json"""
import json
import sys

T, d, kvw, ffn, V = 8192, 4096, 1024, 11008, 32000
BF16, F32, ACC, RES, SWIGLU = "bf16", "f32", "f32_acc", "f32_res", "bf16_swiglu"
FWD = [("qkv fwd +rope", T, d + 2 * kvw, d, BF16), ("o fwd +res", T, d, d, RES), ("gate|up fwd", T, 2 * ffn, d, SWIGLU),
       ("down fwd +res", T, d, ffn, RES)] * 2
# the backward starts with the fused-CE head: dlogits rebuilt from the LSE by
# a recompute of the head GEMM (EPI_CE_GRAD, bf16 out), then head wgrad/dgrad
# (round 2: the down + gate|up and o + q|k|v weight gradients run as one
# grouped launch each; their rows list both problems)
BWD = [("head ce-grad", T, V, d, BF16), ("head wgrad", d, V, T, ACC), ("head dgrad", T, d, V, F32),
       ("down dgrad", T, ffn, d, BF16), ("down+gate|up wgrad", [(ffn, d, T), (d, 2 * ffn, T)], None, None, ACC),
       ("gate|up dgrad", T, d, 2 * ffn, F32), ("o dgrad", T, d, d, BF16),
       ("o+qkv wgrad", [(d, d, T), (d, d + 2 * kvw, T)], None, None, ACC)]


def algorithmic(M, N, K, epi):
    c = {BF16: 2, F32: 4, ACC: 8, RES: 8, SWIGLU: 3}[epi]  # SWIGLU: gate|up + h (N/2 columns) in bf16
    if isinstance(M, list):  # grouped launch: the sum over its problems
        return sum(algorithmic(m, n, k, epi) for m, n, k in M)
    return 2 * (M * K + N * K) + c * M * N


def main():
    s = json.load(open(sys.argv[1]))
    rows = []
    for shapes, rep in ((FWD, "gemm_fwd.ncu-rep"), (BWD, "gemm_bwd.ncu-rep")):
        for (name, M, N, K, epi), l in zip(shapes, s[rep]):
            a = algorithmic(M, N, K, epi)
            rows.append({"shape": name, "M": M, "N": N, "K": K, "epilogue": epi, "kernel": l["kernel"],
                         "duration_us": l["duration"] * 1e6, "dram_bytes": l["dram_bytes"], "algorithmic_bytes": a,
                         "ratio": l["dram_bytes"] / a, "tensor_active_pct": l["tensor_active_pct"],
                         "sm_ghz": l["sm_clock"] / 1e9})
    n = len(rows)
    out = {"source": "ncu --set full --clock-control none, bench.py --workload short (one training step); "
                     "launches of layers 0-1 forward and head + layer 31 backward",
           "mean_dram_bytes_per_launch": sum(r["dram_bytes"] for r in rows) / n,
           "mean_algorithmic_bytes_per_launch": sum(r["algorithmic_bytes"] for r in rows) / n,
           "launches": rows}
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    for r in rows:
        print(f"{r['shape']:15s} {r['duration_us']:8.1f} us  dram {r['dram_bytes']/1e6:8.1f} MB  "
              f"alg {r['algorithmic_bytes']/1e6:8.1f} MB  x{r['ratio']:.2f}  tensor {r['tensor_active_pct']:.1f}%")
    print("mean dram / alg per launch (MB):", out["mean_dram_bytes_per_launch"] / 1e6,
          out["mean_algorithmic_bytes_per_launch"] / 1e6)


if __name__ == "__main__":
    main()
