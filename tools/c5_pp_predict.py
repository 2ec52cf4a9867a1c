"""Config C5 (BASELINE.json): Qwen2.5-32B-shaped, PP=4 x DP=2 chunk-aware 1F1B,
chunk 16K — simulator-in-the-loop prediction from MEASURED stage costs
(SURVEY §8f-1), because every gpurun call gets exactly one B200.

1. Measure on one B200, per chunk, the device time of every forward /
   recompute / backward of one pipeline stage's worth of layers (16 of 64)
   on the real C5 chunk plan (cf_step_op_times): a 16-layer model with the
   LM head (= the last stage, the heaviest) and a 1-layer model, so that
   per-layer and head costs separate:
       layer(c) = (t16(c) - t1(c)) / 15,  head(c) = t1(c) - layer(c).
2. Stage costs: stage 0 = 16 layers (+ embedding, ~0), stages 1-2 = 16
   layers, stage 3 = 16 layers + head.  The reference simulator applies one
   cost per chunk to every stage, so the prediction uses the last-stage cost
   (upper bound on the makespan) and, for comparison, the middle-stage cost.
3. DP=2: the 2-block global plan is split by the LPT unit partition
   (cf_plan_partition); each replica's sub-plan is simulated with the
   product's cf_pp_simulate (bit-exact with pipeline.hpp) on those costs.
   Step time = slowest replica's makespan + the stage-gradient all-reduce
   estimate (2 ranks, fp32, NVLink ~ 700 GB/s bus bandwidth).

4. Memory per stage (round 2): every stage's op stream is replayed under
   the executor's rules (cf_pp_stage_memory) for tape budgets 0..4
   (cf_run_opts.stage_tape_budget); stage peak = static (weights bf16 +
   fp32 grads of its layers, + embedding on stage 0, + final norm / head on
   the last) + peak tape tokens x measured tape bytes/token + kept stage-input
   tokens x d x 4 + the dependent group's KV state + the measured transient
   working set.  The chosen budget is the fastest (cf_pp_simulate_budget:
   checkpointed chunks pay their forward again) whose worst stage fits
   170 GB; the pipeline-aware tuner (cf_tune_grid_search_pp) re-picks
   (chunk size, K) with the in-flight tapes counted.

Writes one JSON object (stdout)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2503_02356_b200 as cf  # noqa: E402
from paper_2503_02356_b200 import capi  # noqa: E402

QWEN = dict(vocab=152064, d=5120, heads=40, kv_heads=8, ffn=27648, seed=1)
LAYERS, STAGES, DP, CHUNK, K = 64, 4, 2, 16384, 1


def block(seed):
    short = capi.synthesize(999, seed, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)
    return np.concatenate([short, [37888]]).astype(np.int64)


def measure(ctx, layers, plan, lengths, tokens, ids):
    m = cf.Model(ctx, cf.model_cfg(arch=cf.ARCH_LLAMA, layers=layers, **QWEN))
    st = cf.Step(m, plan, lengths, tokens, ids)
    st.run()  # warm-up
    ctx.set_profiling(True)
    r = st.run()
    ctx.set_profiling(False)
    kinds, cids, ms = st.op_times()
    st.close()
    m.close()
    return r, kinds, cids, ms


def main():
    ctx = cf.Context(0)
    blocks = [block(b + 1) for b in range(DP)]
    lengths = np.concatenate(blocks)
    ids = np.arange(len(lengths), dtype=np.int64)
    tokens = np.concatenate([cf.gen_tokens(bl, QWEN["vocab"], b + 1) for b, bl in enumerate(blocks)])
    gplan = cf.Plan.build(lengths, CHUNK, K, ids)
    replicas = [gplan.partition(DP, r) for r in range(DP)]
    out = {"workload": "C5: Qwen2.5-32B-shaped (d 5120, 64 L, 40 H, GQA-8, ffn 27648, V 152064), PP=4 x DP=2, "
                       "chunk 16384, K=1, two 1,000-seq long-tail blocks",
           "method": "per-chunk stage costs measured on one B200 (16-layer and 1-layer models on replica 0's "
                     "sub-plan), chunk-aware 1F1B timed by cf_pp_simulate (bit-exact with pipeline.hpp)"}
    # measure on replica 0's sub-plan (its chunks are representative of both)
    r16, k16, c16, t16 = measure(ctx, 16, replicas[0], lengths, tokens, ids)
    r1, k1, c1, t1 = measure(ctx, 1, replicas[0], lengths, tokens, ids)
    assert np.array_equal(k16, k1) and np.array_equal(c16, c1)
    layer = (t16 - t1) / 15.0
    head = t1 - layer
    fw, bw = {}, {}
    for kind, cid, lay, hd in zip(k16, c16, layer, head):
        if kind == capi.PP_FORWARD:
            fw[int(cid)] = (lay, hd)
        elif kind == capi.PP_BACKWARD:
            bw[int(cid)] = (lay, hd)
    out["measured"] = {"stage16_step_s": float(t16.sum() / 1e3), "one_layer_step_s": float(t1.sum() / 1e3),
                       "peak_hbm_gb_16_layers": r16.peak_hbm_bytes / 1e9,
                       "static_gb_16_layers": r16.static_hbm_bytes / 1e9,
                       "activations_gb_16_layers": r16.act_hbm_bytes / 1e9,
                       "kv_state_gb_16_layers": r16.kv_hbm_bytes / 1e9,
                       "model_tflops_16_layers": r16.model_flops / (t16.sum() / 1e3) / 1e12}
    per_stage = LAYERS // STAGES
    grad_bytes = 4 * (per_stage * (QWEN["d"] * (QWEN["d"] + 2 * 1024) + QWEN["d"] ** 2 + 3 * QWEN["d"] * QWEN["ffn"])
                      + QWEN["d"] * QWEN["vocab"])
    allreduce_ms = 2 * (DP - 1) / DP * grad_bytes / 700e9 * 1e3
    res = {}
    for label, with_head in (("last_stage_cost", True), ("middle_stage_cost", False)):
        spans, bubbles, occ = [], [], []
        for rp in replicas:
            ch = rp.export()[0]
            # costs of this replica's chunks: measured where replica 0 has the chunk, else by token count
            f = np.zeros(len(ch))
            b = np.zeros(len(ch))
            ref_tok = {int(c["chunk_id"]): int(c["total_tokens"]) for c in replicas[0].export()[0]}
            per_tok_f = np.mean([(v[0] * per_stage + (v[1] if with_head else 0)) / ref_tok[c] for c, v in fw.items()])
            per_tok_b = np.mean([(v[0] * per_stage + (v[1] if with_head else 0)) / ref_tok[c] for c, v in bw.items()])
            for i, c in enumerate(ch):
                cid = int(c["chunk_id"])
                if cid in fw and cid in bw:
                    f[i] = fw[cid][0] * per_stage + (fw[cid][1] if with_head else 0)
                    b[i] = bw[cid][0] * per_stage + (bw[cid][1] if with_head else 0)
                else:
                    f[i] = per_tok_f * int(c["total_tokens"])
                    b[i] = per_tok_b * int(c["total_tokens"])
            ops, _, _, pr = capi.pp_simulate(rp, STAGES, K, fwd_cost=f, bwd_cost=b)
            if with_head and rp is replicas[0]:  # predicted timeline, chrome-trace (1 unit = 1 ms here)
                with open("gpurun_out/c5_pp_trace.json", "w") as fh:
                    fh.write(capi.pp_export_trace(ops, True))
            spans.append(pr.makespan)
            bubbles.append(pr.bubble_ratio)
            occ.append(pr.occupancy_bubble)
        step_ms = max(spans) + allreduce_ms
        res[label] = {"makespan_ms_per_replica": spans, "bubble_ratio": bubbles,
                      "bubble_ratio_recompute_as_busy": occ, "allreduce_ms_est": allreduce_ms,
                      "step_ms": step_ms, "tokens_per_s_8gpu": float(lengths.sum()) / (step_ms / 1e3)}
    # whole-sequence 1F1B on the same replica for the paper's comparison
    seqs = sorted({int(s["sequence_id"]) for s in replicas[0].export()[1]})
    r0_lengths = lengths[seqs]
    _, _, _, p1 = capi.pp_simulate_1f1b(r0_lengths, STAGES, {"alpha": 1.0, "beta": 1.05e-5})
    out["prediction"] = res
    out["reference_1f1b_whole_sequence_bubble_cost_model"] = p1.bubble_ratio
    # simulator-in-the-loop: fit the reference CostModel
    # fwd = gamma + alpha*len + beta*(len^2 + len*prefix) to the measured
    # last-stage forward times, backward_multiplier = mean(bwd / fwd), then
    # grid_search (tuner.hpp:39) over (chunk_size, K) with those costs and a
    # per-stage memory model measured on the same 16-layer stage
    ch0 = replicas[0].export()[0]
    seg0 = replicas[0].export()[1]
    pre = {}
    for c in ch0:
        if c["kind"] == 1:
            s0 = seg0[c["seg_offset"]]
            pre[int(c["chunk_id"])] = int(s0["start_token"])
    X, y, ratio = [], [], []
    for c in ch0:
        cid = int(c["chunk_id"])
        if cid not in fw or cid not in bw:
            continue
        ln, p_ = float(c["total_tokens"]), float(pre.get(cid, 0))
        f_ms = fw[cid][0] * per_stage + fw[cid][1]
        b_ms = bw[cid][0] * per_stage + bw[cid][1]
        X.append([1.0, ln, ln * ln + ln * p_])
        y.append(f_ms)
        ratio.append(b_ms / f_ms)
    coef, *_ = np.linalg.lstsq(np.array(X), np.array(y), rcond=None)
    gamma, alpha, beta = (max(0.0, float(v)) for v in coef)
    bmult = float(np.mean(ratio))
    fit = {"gamma_ms": gamma, "alpha_ms_per_token": alpha, "beta_ms_per_token2": beta,
           "backward_multiplier": bmult, "chunks_fitted": len(y),
           "max_rel_residual": float(np.max(np.abs(np.array(X) @ np.array([gamma, alpha, beta]) - np.array(y))
                                        / np.array(y)))}
    GIB = float(1 << 30)
    stage_static = r16.static_hbm_bytes / GIB
    per_tok = r16.act_hbm_bytes / GIB / CHUNK  # K=1 retained tape of one 16K chunk
    per_ctx = 16 * 1024 * 12 / GIB             # K/V bf16 + dK/dV fp32 per context token, 16 layers
    mem = (stage_static, per_tok, per_ctx, 1.0)
    table, bc, bk, ev, report = capi.tune_grid_search(
        lengths[:len(blocks[0])], [4096, 8192, 16384, 32768], [1, 2, 4], STAGES,
        {"gamma": gamma, "alpha": alpha, "beta": beta, "backward_multiplier": bmult, "hop_latency": 0.0},
        mem, 165.0, 1000, 1, 0)
    out["cost_model_fit"] = fit
    out["tuner"] = {"memory_model": dict(zip(("base_gib", "per_chunk_token_gib", "per_context_token_gib",
                                              "gqa_ratio"), mem)),
                    "budget_gib": 165.0, "best_chunk_size": bc, "best_k": bk, "evaluations": ev,
                    "report": report}
    out["tokens_global"] = int(lengths.sum())
    out["memory"] = stage_memory(ctx, replicas, lengths, tokens, ids, fw, bw, per_stage, allreduce_ms, fit)
    print(json.dumps(out, default=lambda o: o.item() if hasattr(o, "item") else str(o)), flush=True)


def tape_bytes_per_token(layers, head):
    """alloc_tape(T, retain=true) of the executor, per token (engine.cu)."""
    d, H, kvw, ffn = QWEN["d"], QWEN["heads"], 1024, QWEN["ffn"]
    qkv_w, gu_w, dh = d + 2 * kvw, 2 * ffn, d // H
    per_layer = d * 4 + qkv_w * 2 + d * 2 + H * 4 + d * 4 + gu_w * 2 + d * 2 + d * 2 + ffn * 2
    return layers * per_layer + d * 4 + (dh // 2) * 8 + (4 + d * 2 if head else 0)


def stage_static_bytes(stage):
    d, kvw, ffn, V = QWEN["d"], 1024, QWEN["ffn"], QWEN["vocab"]
    per_layer = d * (d + 2 * kvw) + d * d + d * 2 * ffn + ffn * d + 2 * d
    n = (LAYERS // STAGES) * per_layer
    if stage == 0:
        n += V * d
    if stage == STAGES - 1:
        n += d + d * ((V + 7) // 8 * 8)
    return 6 * n  # bf16 weights + fp32 gradients


def stage_memory(ctx, replicas, lengths, tokens, ids, fw, bw, per_stage, allreduce_ms, fit):
    GB = 1e9
    # measured: one retained 16K tape of a 16-layer stage with the head, and
    # the transient working set beyond static + tapes + KV state
    m = cf.Model(ctx, cf.model_cfg(arch=cf.ARCH_LLAMA, layers=per_stage, **QWEN))
    one = np.array([CHUNK], np.int64)
    st = cf.Step(m, cf.Plan.build(one, CHUNK, 1), one, cf.gen_tokens(one, QWEN["vocab"], 9))
    st.run()
    r = st.run()
    st.close()
    m.close()
    tape_tok_measured = r.act_hbm_bytes / CHUNK
    transient = r.peak_hbm_bytes - r.static_hbm_bytes - r.act_hbm_bytes - r.kv_hbm_bytes
    kv_per_ctx_token = per_stage * 1024 * (2 * 2 + 2 * 4)  # K, V bf16 + dK|dV fp32
    out = {"tape_bytes_per_token_analytic": tape_bytes_per_token(per_stage, True),
           "tape_bytes_per_token_measured": tape_tok_measured,
           "transient_gb_measured": transient / GB,
           "static_gb": [stage_static_bytes(s) / GB for s in range(STAGES)],
           "static_gb_measured_16_layers_with_head": r.static_hbm_bytes / GB,
           "budget_gb": 170.0, "per_budget": {}}
    best = None
    ch0 = replicas[0].export()[0]
    tok0 = {int(c["chunk_id"]): float(c["total_tokens"]) for c in ch0}
    per_tok = (np.mean([(v[0] * per_stage + v[1]) / tok0[c] for c, v in fw.items()]),
               np.mean([(v[0] * per_stage + v[1]) / tok0[c] for c, v in bw.items()]))
    for budget in range(0, 5):
        worst, spans, stages_gb = 0.0, [], []
        for rp in replicas:
            mem = capi.pp_stage_memory(rp, STAGES, K, budget)
            segs = rp.export()[1]
            chs = rp.export()[0]
            group_len = max([int(segs[c["seg_offset"]]["start_token"] + segs[c["seg_offset"]]["length"])
                             for c in chs if c["kind"] == 1] or [0])
            per = []
            for s in range(STAGES):
                tape_tok = tape_bytes_per_token(per_stage, s == STAGES - 1)
                b = (stage_static_bytes(s) + mem["peak_tape_tokens"][s] * tape_tok +
                     mem["peak_kept_tokens"][s] * QWEN["d"] * 4 + group_len * kv_per_ctx_token + transient)
                per.append(b / GB)
            stages_gb.append(per)
            worst = max(worst, max(per))
            ch = rp.export()[0]
            f = np.array([fw.get(int(c["chunk_id"]), (0, 0))[0] * per_stage + fw.get(int(c["chunk_id"]), (0, 0))[1]
                          for c in ch])
            b_ = np.array([bw.get(int(c["chunk_id"]), (0, 0))[0] * per_stage + bw.get(int(c["chunk_id"]), (0, 0))[1]
                           for c in ch])
            miss = f == 0
            if miss.any():  # chunks only replica 1 has: replica 0's mean cost per token
                tok = ch["total_tokens"].astype(np.float64)
                f[miss] = per_tok[0] * tok[miss]
                b_[miss] = per_tok[1] * tok[miss]
            _, _, _, pr = capi.pp_simulate(rp, STAGES, K, fwd_cost=f, bwd_cost=b_, tape_budget=budget)
            spans.append(pr.makespan)
        step_ms = max(spans) + allreduce_ms
        rec = {"stage_peak_gb_per_replica": stages_gb, "worst_stage_gb": worst, "makespan_ms": spans,
               "step_ms": step_ms, "tokens_per_s_8gpu": float(lengths.sum()) / (step_ms / 1e3),
               "fits": bool(worst <= 170.0)}
        out["per_budget"][str(budget)] = rec
        if rec["fits"] and (best is None or step_ms < out["per_budget"][str(best)]["step_ms"]):
            best = budget
    out["chosen_budget"] = best
    # pipeline-aware tuner with the same per-stage memory model
    lay = tape_bytes_per_token(per_stage, True) / float(1 << 30)
    mem = (max(stage_static_bytes(s) for s in range(STAGES)) / float(1 << 30) + transient / float(1 << 30), lay,
           kv_per_ctx_token / float(1 << 30), 1.0)
    # the CostModel fitted to this run's measured stage costs (main())
    table, bc, bk, ev, report = capi.tune_grid_search_pp(
        lengths[:1000], [4096, 8192, 16384], [1, 2], STAGES,
        {"gamma": fit["gamma_ms"], "alpha": fit["alpha_ms_per_token"], "beta": fit["beta_ms_per_token2"],
         "backward_multiplier": fit["backward_multiplier"], "hop_latency": 0.0},
        mem, QWEN["d"] * 4 / float(1 << 30), best or 0, 170.0 / 1.073741824, 1000, 1, 0)
    out["tuner_pp"] = {"tape_budget": best or 0, "best_chunk_size": bc, "best_k": bk, "evaluations": ev,
                       "report": report, "memory_model": mem}
    return out


if __name__ == "__main__":
    main()
