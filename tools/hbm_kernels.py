"""ncu evidence for the non-contraction (HBM-bound) kernels at C2 widths.

  python tools/hbm_kernels.py run            # the profiled workload
  python tools/hbm_kernels.py parse raw.csv out.json

Workload: the C2 layer shape (d 4096, 32/8 heads, ffn 11008, vocab 32000)
with 2 layers, one 8,192-token standalone chunk and one 16,384-token
sequence split into a 2-chunk dependent group at chunk 8192 — every chunk is
T = 8192 rows, the C2 chunk size, so each launch's algorithmic bytes follow
from its kernel name alone.  Profile it with

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --kernel-name regex:'rmsnorm|gain_reduce|swiglu|ce_|embed|kv_store|dkv_to|rope|to_bf16|sum_f64' \
      --csv --page raw --log-file raw.csv python tools/hbm_kernels.py run

`achieved` = algorithmic bytes / ncu duration (cold-cache, serialised: a
lower bound on the in-step rate); `traffic` = dram read + write bytes.
"""
import csv
import io
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

T, D, KVW, FFN, V, H = 8192, 4096, 1024, 11008, 32000, 32

# algorithmic bytes per launch at T rows (what the kernel must read + write)
ALG = {
    "rmsnorm_row_kernel": (T * D * (4 + 2), "x fp32 in, normed bf16 out"),
    "rmsnorm_bwd_rows_kernel": (T * D * (4 + 4 + 4 + 4 + 2),
                                "x, dy, residual-grad fp32 in; dx fp32 + bf16(dx) out"),
    "gain_reduce_cols_kernel": (None, "per-CTA gain partials (parts x d fp32) in, d out"),
    "swiglu_bwd_kernel": (T * FFN * (4 + 2 + 4), "gate|up + dh bf16 in, dgate|dup bf16 out"),
    "ce_rows_kernel": (T * V * (4 + 2), "fp32 logits in, bf16 dlogits out"),
    "ce_kernel": (T * V * (4 + 2), "fp32 logits in, bf16 dlogits out"),
    "embed_kernel": (T * D * (2 + 4), "bf16 rows gathered, fp32 residual out"),
    "embed_bwd_kernel": (None, "dx fp32 in, embedding-gradient rows RMW"),
    "kv_store_kernel": (T * KVW * 2 * (2 + 2), "K, V bf16 copied into the group cache"),
    "dkv_to_dqkv_vec_kernel": (T * KVW * 2 * (4 + 2), "dK|dV fp32 in, bf16 (RoPE-rotated dK) out"),
    "dkv_to_dqkv_kernel": (T * KVW * 2 * (4 + 2), "dK|dV fp32 in, bf16 out"),
    "rope_table_kernel": (T * (D // H // 2) * 8, "cos/sin table out"),
    "to_bf16_kernel": (T * D * (4 + 2), "fp32 in, bf16 out"),
    "sum_f64_kernel": (T * 4, "row losses in"),
}


def run():
    import paper_2503_02356_b200 as cf
    ctx = cf.Context(0)
    model = cf.Model(ctx, cf.model_cfg(arch=1, vocab=V, d=D, heads=H, kv_heads=8, layers=2, ffn=FFN, seed=1))
    lengths = np.array([8192, 16384], np.int64)
    tokens = cf.gen_tokens(lengths, V, 3)
    plan = cf.Plan.build(lengths, 8192, 1)
    r = model.run_plan(plan, lengths, tokens)
    print(json.dumps({"loss": r.loss, "launches": r.gpu_launches}))


def parse(raw, out):
    text = open(raw).read()
    text = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.reader(io.StringIO(text)))
    head, units = rows[0], rows[1]
    idx = {k: i for i, k in enumerate(head)}
    scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6551.0)
    per = {}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].split("<")[0].split("::")[-1].strip()
        g = lambda m: float(r[idx[m]].replace(",", "")) * scale.get(units[idx[m]], 1.0)  # noqa: E731
        dur, rd, wr = g("gpu__time_duration.sum"), g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        per.setdefault(name, []).append((dur, rd + wr))
    res = {"workload": "C2 widths (d 4096, ffn 11008, V 32000), 2 layers, chunks of T = 8192 rows "
                       "(1 standalone + a 2-chunk dependent group); ncu cold-cache serialised launches",
           "peak_gbs": peak, "peak_kind": "measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs)", "kernels": {}}
    for name, v in sorted(per.items()):
        dur = float(np.median([x[0] for x in v]))
        traffic = float(np.median([x[1] for x in v]))
        alg, what = ALG.get(name, (None, ""))
        rec = {"launches": len(v), "median_us": dur * 1e6, "dram_bytes": traffic,
               "dram_gbs": traffic / dur / 1e9, "algorithmic_bytes": alg, "moves": what}
        if alg:
            rec["achieved_gbs"] = alg / dur / 1e9
            rec["frac_of_peak"] = alg / dur / 1e9 / peak
            rec["traffic_over_algorithmic"] = traffic / alg
        else:
            rec["frac_of_peak"] = traffic / dur / 1e9 / peak
        res["kernels"][name] = rec
    json.dump(res, open(out, "w"), indent=1)
    for k, v in res["kernels"].items():
        print(f"{k:28s} n={v['launches']:3d} {v['median_us']:9.1f} us  dram {v['dram_gbs']:7.0f} GB/s  "
              f"frac {v['frac_of_peak']:.2f}")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2], sys.argv[3])
