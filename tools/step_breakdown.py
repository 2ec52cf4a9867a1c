"""Per-op device time of one C2 step (cf_step_op_times, profiling on): every
forward / recompute / backward of every chunk, with the chunk's tokens and
attention pairs, summed by chunk type (standalone packed shorts vs the
dependent group of the 37,888-token sequence).  Writes JSON to stdout."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2503_02356_b200 as cf  # noqa: E402
from paper_2503_02356_b200 import capi  # noqa: E402


def main():
    ctx = cf.Context(0)
    model = cf.Model(ctx, cf.model_cfg(arch=cf.ARCH_LLAMA, **bench.MODEL))
    lengths = bench.block_lengths(1)
    tokens = cf.gen_tokens(lengths, bench.MODEL["vocab"], 1)
    plan = cf.Plan.build(lengths, bench.CHUNK, bench.K_RETAIN)
    st = cf.Step(model, plan, lengths, tokens)
    st.run()
    ctx.set_profiling(True)
    r = st.run()
    ctx.set_profiling(False)
    kinds, ids, ms = st.op_times()
    ch, sg, _, _ = plan.export()
    info = {}
    for c in ch:
        segs = sg[c["seg_offset"]:c["seg_offset"] + c["seg_count"]]
        pairs = sum(float(s["length"]) * float(s["start_token"]) + float(s["length"]) * (s["length"] + 1) / 2
                    for s in segs)
        info[int(c["chunk_id"])] = ("group" if c["kind"] == 1 else "standalone", int(c["total_tokens"]), pairs)
    agg, rows = {}, []
    names = {capi.PP_FORWARD: "forward", capi.PP_RECOMPUTE: "recompute", capi.PP_BACKWARD: "backward"}
    for k, i, t in zip(kinds, ids, ms):
        typ, tok, pairs = info[int(i)]
        key = f"{typ}/{names[int(k)]}"
        a = agg.setdefault(key, {"ops": 0, "ms": 0.0, "tokens": 0, "pairs": 0.0})
        a["ops"] += 1
        a["ms"] += float(t)
        a["tokens"] += tok
        a["pairs"] += pairs
        rows.append({"chunk": int(i), "type": typ, "op": names[int(k)], "tokens": tok, "pairs": pairs, "ms": float(t)})
    total = float(np.sum(ms))
    out = {"step_ms_sum_of_ops": total, "model_tflops": r.model_flops / (total / 1e3) / 1e12,
           "by_type": {k: dict(v, share=v["ms"] / total) for k, v in sorted(agg.items())},
           "class_ms": {"gemm": r.gemm_ms, "attention_fwd": r.attn_ms, "attention_bwd": r.attn_bwd_ms},
           "ops": rows}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
