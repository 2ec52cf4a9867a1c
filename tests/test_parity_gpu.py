"""End-to-end parity of the CUDA chunk path (through the C-ABI) against the
CPU oracle on the same bf16-rounded weights and the same batches.

Tolerances (compare_gradients metric, toy_model.hpp:681-718), stated for a
bf16-storage / fp32-accumulate path against an fp64 oracle:
  loss relative error <= 2e-3, per-tensor gradient max-norm error <= 3e-2.
Integer-exact / bitwise checks: recompute-loss equality, K-independence of
gradients, KV-completeness counters.
"""
import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi
from oracle.oracle import model_cfg as ocfg

pytestmark = pytest.mark.gpu

LOSS_TOL = 2e-3
GRAD_TOL = 3e-2


def _cfgs(arch, vocab, d, heads, kvh, layers, ffn=0, seed=7):
    return (cf.model_cfg(arch=arch, vocab=vocab, d=d, heads=heads, kv_heads=kvh, layers=layers, ffn=ffn, seed=seed),
            ocfg(arch=arch, vocab=vocab, d=d, heads=heads, kv_heads=kvh, layers=layers, ffn=ffn, seed=seed))


def _per_tensor_err(model, grads_gpu, grads_ref):
    out, off = [], 0
    for i in range(model.num_tensors()):
        name, r, c = model.tensor_info(i)
        a = grads_gpu[off:off + r * c]
        b = grads_ref[off:off + r * c]
        off += r * c
        mag = max(np.abs(a).max(), np.abs(b).max(), 1e-12)
        out.append((name, float(np.abs(a - b).max() / mag)))
    return out


CASES = [
    # arch, vocab, d, heads, kv_heads, layers, ffn, lengths, chunk, k
    ("toy-small", 0, 64, 64, 4, 2, 2, 0, [8, 8, 16, 40, 70], 32, 1),
    ("toy-k2", 0, 64, 64, 4, 2, 2, 0, [5, 12, 31, 130, 64, 9], 32, 2),
    ("toy-dh128", 0, 96, 256, 2, 1, 2, 0, [100, 300, 77], 128, 1),
    ("llama-small", 1, 96, 128, 4, 2, 2, 256, [8, 30, 64, 150, 33], 64, 1),
    ("llama-gqa", 1, 120, 256, 2, 1, 2, 512, [200, 90, 333], 128, 2),
    # head_dim 128 with 64-token chunks: 128-key tiles of early chunks reach
    # KV-cache rows that later chunks have not written yet
    ("llama-dh128-cs64", 1, 96, 256, 2, 1, 2, 512, [8, 30, 64, 150, 33, 100], 64, 1),
    ("llama-dh128-cs96-k2", 1, 96, 256, 2, 1, 2, 512, [300, 20, 97, 5], 96, 2),
    ("llama-dh128-mha-cs200", 1, 64, 256, 2, 2, 1, 384, [450, 64, 199], 200, 1),
    # cross-entropy forms: register-resident rows (V % 4 == 0, V <= 32768,
    # incl. the C2 vocabulary) and the strided kernel (odd V)
    ("toy-v32000", 0, 32000, 64, 4, 2, 1, 0, [40, 70, 20], 64, 1),
    ("toy-v9000", 0, 9000, 64, 4, 2, 1, 0, [33, 64], 64, 1),
    ("toy-v97", 0, 97, 64, 4, 2, 1, 0, [40, 70, 20], 64, 1),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_run_plan_matches_oracle(ctx, oracle, case):
    _, arch, V, d, H, KVH, L, ffn, lengths, cs, k = case
    gcfg, c = _cfgs(arch, V, d, H, KVH, L, ffn)
    lengths = np.array(lengths, np.int64)
    tokens = cf.gen_tokens(lengths, V, 11)
    model = cf.Model(ctx, gcfg)
    plan = cf.Plan.build(lengths, cs, k)
    r = model.run_plan(plan, lengths, tokens)
    params = model.params_flat()
    grads = model.grads_flat()
    ol, og, oi = oracle.run_plan(c, lengths, tokens, cs, k, params=params)
    assert r.recompute_loss_mismatches == 0
    assert r.kv_completeness_violations == 0
    assert r.recompute_forward_count == oi[1]
    assert r.peak_retained_tokens == oi[0]
    assert abs(r.loss - ol) / abs(ol) <= LOSS_TOL, (r.loss, ol)
    errs = _per_tensor_err(model, grads, og)
    worst = max(errs, key=lambda e: e[1])
    assert worst[1] <= GRAD_TOL, worst
    model.close()


@pytest.mark.parametrize("kvh", [1, 2], ids=["gqa", "mha-rope-epilogue"])
def test_run_plan_matches_oracle_forced_pair_gemms(ctx, oracle, kvh):
    """CTA-pair GEMMs at toy sizes (cf_debug_set_gemm_mode(2)), so the fused
    gate|up + SwiGLU epilogue and the pair epilogues run under the oracle,
    including a recomputed forward (sequence of 3 chunks, K = 1).  With
    kv_width 256 the q|k|v GEMM also carries RoPE and the KV-cache copy."""
    gcfg, c = _cfgs(1, 96, 256, 2, kvh, 2, 384)
    lengths = np.array([700, 130, 301, 64], np.int64)
    tokens = cf.gen_tokens(lengths, 96, 13)
    capi.check(capi.lib().cf_debug_set_gemm_mode(2))
    try:
        model = cf.Model(ctx, gcfg)
        plan = cf.Plan.build(lengths, 256, 1)
        r = model.run_plan(plan, lengths, tokens)
        params, grads = model.params_flat(), model.grads_flat()
    finally:
        capi.check(capi.lib().cf_debug_set_gemm_mode(0))
    ol, og, oi = oracle.run_plan(c, lengths, tokens, 256, 1, params=params)
    assert r.recompute_forward_count == oi[1] and oi[1] > 0
    assert r.recompute_loss_mismatches == 0
    assert abs(r.loss - ol) / abs(ol) <= LOSS_TOL, (r.loss, ol)
    worst = max(_per_tensor_err(model, grads, og), key=lambda e: e[1])
    assert worst[1] <= GRAD_TOL, worst
    model.close()


@pytest.mark.parametrize("arch", [0, 1])
def test_chunked_equals_unchunked_on_gpu(ctx, arch):
    """verify_equivalence on the GPU: chunked-with-state vs full sequences."""
    gcfg, _ = _cfgs(arch, 64, 64, 4, 2, 2, 128 if arch else 0)
    lengths = np.array([8, 8, 16, 32, 100, 45], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 3)
    model = cf.Model(ctx, gcfg)
    rep = cf.verify_equivalence(model, lengths, tokens, 16, 1, loss_tol=1e-4, grad_tol=1e-2)
    assert rep.passed, (rep.loss_rel_err, rep.max_grad_rel_err, rep.instrumentation)
    # the `chunkflow verify` report layout (plan_runner.hpp:352-365)
    txt = rep.to_text().splitlines()
    assert txt[0] == f"chunks: {rep.chunk_count}" and txt[-1] == "result: PASS"
    assert txt[2].startswith("embedding max_abs_diff=") and any(t.startswith("max_rel_err=") for t in txt)
    model.close()


def test_gradients_bitwise_identical_across_k(ctx):
    """test_plan_runner.cpp:98-115 on the GPU: K only changes what is
    retained vs recomputed; deterministic kernels make grads bitwise equal."""
    gcfg, _ = _cfgs(1, 64, 64, 4, 2, 2, 128)
    lengths = np.array([150, 20, 9], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 5)
    model = cf.Model(ctx, gcfg)
    base = None
    for k in (1, 2, 3, 8):
        r = model.run_plan(cf.Plan.build(lengths, 32, k), lengths, tokens)
        assert r.recompute_loss_mismatches == 0
        g = model.grads_flat()
        if base is None:
            base = (r.loss, g)
        else:
            assert r.loss == base[0]
            assert np.array_equal(g, base[1]), k
    model.close()


def test_corrupted_kv_grads_fail_verification(ctx):
    """Negative control (plan_runner.hpp:277-284): scaling incoming dK/dV by
    1.0000001 must break chunked == unchunked at a tight tolerance."""
    gcfg, _ = _cfgs(0, 64, 64, 4, 2, 2)
    lengths = np.array([200, 10], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 9)
    model = cf.Model(ctx, gcfg)
    good = model.run_plan(cf.Plan.build(lengths, 32, 1), lengths, tokens)
    g0 = model.grads_flat()
    bad = model.run_plan(cf.Plan.build(lengths, 32, 1), lengths, tokens, corrupt=True)
    g1 = model.grads_flat()
    assert good.loss == bad.loss
    assert not np.array_equal(g0, g1)
    model.close()


def test_init_matches_reference_bits(ctx, oracle):
    """Device SplitMix64 init == reference init_model stream (rounded to bf16)."""
    gcfg, c = _cfgs(0, 64, 64, 4, 2, 2)
    model = cf.Model(ctx, gcfg)
    # direct fp64 -> bf16 round-to-nearest-even (8 significant bits)
    m, e = np.frexp(oracle.init(c))
    ref = np.ldexp(np.rint(m * 256.0), e - 8)
    assert np.array_equal(model.params_flat(), ref)
    model.close()


def test_single_chunk_plan_bitwise_equals_full_run(ctx):
    """test_plan_runner.cpp:53-70 on the GPU: a one-chunk plan of one
    sequence runs exactly the kernels of the full-sequence run."""
    for arch, ffn in ((0, 0), (1, 256)):
        gcfg, _ = _cfgs(arch, 64, 128, 4, 2, 2, ffn)
        lengths = np.array([200], np.int64)
        tokens = cf.gen_tokens(lengths, 64, 21)
        model = cf.Model(ctx, gcfg)
        r = model.run_plan(cf.Plan.build(lengths, 256, 1), lengths, tokens)
        g0 = model.grads_flat()
        f = model.backward_full(lengths, tokens)
        g1 = model.grads_flat()
        assert r.loss == f.loss
        assert np.array_equal(g0, g1)
        model.close()


def test_random_plans_instrumentation_matches_static(ctx):
    """test_plan_runner.cpp:117-146 / acceptance.cpp:210-244 on the GPU: over
    20 seeded random batches, chunk sizes and K, the executor's measured peak
    of retained tokens and its recompute count equal the static plan's, every
    recomputed forward reproduces its first-pass loss bitwise and every KV
    read finds a complete prefix."""
    gcfg, _ = _cfgs(1, 64, 128, 4, 2, 2, 256)
    model = cf.Model(ctx, gcfg)
    rng = np.random.default_rng(17)
    for trial in range(20):
        n = int(rng.integers(1, 7))
        lengths = rng.integers(1, 300, size=n).astype(np.int64)
        cs = int(rng.choice([16, 32, 48, 64, 100, 128]))
        k = int(rng.integers(1, 4))
        plan = cf.Plan.build(lengths, cs, k)
        _, _, ev, diag = plan.export()
        tokens = cf.gen_tokens(lengths, 64, trial)
        r = model.run_plan(plan, lengths, tokens)
        assert r.peak_retained_tokens == diag["peak_retained_tokens"], trial
        assert r.recompute_forward_count == int(ev["is_recompute"].sum()), trial
        assert r.recompute_loss_mismatches == 0 and r.kv_completeness_violations == 0, trial
        assert np.isfinite(r.loss)
    model.close()


def test_fused_epilogues_multi_wave_discard_forward(ctx):
    """Regression: with more output tiles than CTA pairs, a fused epilogue
    must not write into a buffer its own GEMM is still reading.  A discard
    forward keeps neither the normed input nor the SwiGLU output, so both used
    to share one scratch; the recomputed forward then disagreed with the first
    pass.  Forced CTA-pair GEMMs; ffn = 4 d, so SwiGLU rows written by the
    first wave of gate|up tiles (16 M-blocks x 32 N-tiles, every wave spans
    all M-blocks) land on normed-input rows later waves still read."""
    gcfg, _ = _cfgs(1, 64, 1024, 8, 8, 1, 4096)
    lengths = np.array([10000, 300, 77], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 19)
    capi.check(capi.lib().cf_debug_set_gemm_mode(2))
    try:
        model = cf.Model(ctx, gcfg)
        r = model.run_plan(cf.Plan.build(lengths, 4096, 1), lengths, tokens)
        g_chunked = model.grads_flat()
        f = model.backward_full(lengths, tokens)
        g_full = model.grads_flat()
    finally:
        capi.check(capi.lib().cf_debug_set_gemm_mode(0))
    assert r.recompute_forward_count >= 1
    assert r.recompute_loss_mismatches == 0
    assert abs(r.loss - f.loss) / abs(f.loss) < 1e-4, (r.loss, f.loss)
    off = 0
    for i in range(model.num_tensors()):
        _, rr, cc = model.tensor_info(i)
        a, b = g_chunked[off:off + rr * cc], g_full[off:off + rr * cc]
        off += rr * cc
        assert np.abs(a - b).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-12) < 1e-2, model.tensor_info(i)[0]
    model.close()


def _report(tag, rows):
    import json
    import os
    out = os.environ.get("CF_PARITY_REPORT")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps({"case": tag, **rows}) + "\n")


def test_c1_exact_config_matches_oracle(ctx, oracle):
    """BASELINE config 1 exactly: toy arch, vocab 256, d 256,
    4 heads / 2 KV heads (head_dim 64), 2 layers, model seed 1, the C1
    canonical batch (synthesize(eval_table5, 32, seed 3) + a 2,048-token
    sequence, tokens SplitMix64(5)), chunk 512, K = 2: 26 chunks, 54 events,
    peak retained 1024, recompute 1024 tokens (plan_runner.hpp:368-395 run
    on the GPU against the fp64 oracle on the GPU's bf16-rounded weights).
    K = 1 must give bitwise the same gradients."""
    from oracle.oracle import c1_batch, c1_cfg
    lengths, tokens = c1_batch(oracle)
    oc = c1_cfg()
    gcfg = cf.model_cfg(arch=0, vocab=256, d=256, heads=4, kv_heads=2, layers=2, seed=1)
    model = cf.Model(ctx, gcfg)
    plan = cf.Plan.build(lengths, 512, 2)
    ch, _, ev, diag = plan.export()
    assert (len(ch), len(ev), diag["peak_retained_tokens"], diag["recompute_token_count"]) == (26, 54, 1024, 1024)
    r = model.run_plan(plan, lengths, tokens)
    params, grads = model.params_flat(), model.grads_flat()
    ol, og, oi = oracle.run_plan(oc, lengths, tokens, 512, 2, params=params)
    assert r.peak_retained_tokens == oi[0] == 1024
    assert r.recompute_forward_count == oi[1] == 2
    assert r.recompute_loss_mismatches == 0 and r.kv_completeness_violations == 0
    rel = abs(r.loss - ol) / abs(ol)
    errs = _per_tensor_err(model, grads, og)
    worst = max(errs, key=lambda e: e[1])
    _report("c1_exact", {"loss_gpu": r.loss, "loss_oracle": ol, "loss_rel": rel, "golden_loss_unrounded": 5.5455568137389548,
                         "per_tensor": errs})
    assert rel <= LOSS_TOL, (r.loss, ol)
    assert worst[1] <= GRAD_TOL, worst
    # K-independence (test_plan_runner.cpp:98-115) on the C1 workload
    r1 = model.run_plan(cf.Plan.build(lengths, 512, 1), lengths, tokens)
    assert r1.loss == r.loss and r1.recompute_loss_mismatches == 0
    assert np.array_equal(model.grads_flat(), grads)
    model.close()


def test_production_width_llama_slice_matches_oracle(ctx):
    """Production widths against the fp64 oracle (VERDICT r1 'what's weak'
    #1): the C2 layer shape — d 4096, 32 heads / 8 KV heads (GQA 4), SwiGLU
    ffn 11008, vocab 32000, RMSNorm, RoPE — with 2 layers.  A 3,400-token
    sequence split into a 4-chunk dependent group at chunk 1024 (K = 1: three
    recomputed forwards, prefix K/V reads, dK/dV accumulation) plus four
    short sequences packed into one chunk.  Default GEMM mode, so the CTA-pair
    kernel with the fused RoPE + KV-copy and SwiGLU epilogues runs multi-wave
    (e.g. gate|up 1024 x 22016: 344 tiles over 74 CTA pairs).  Compared with
    the vectorised fp64 oracle (oracle/llama_np.py, pinned to cf_oracle.cpp)
    of the unchunked batch — the verify_equivalence comparison
    (plan_runner.hpp:368-395) — on the GPU's bf16-rounded weights."""
    from oracle import llama_np
    from oracle.oracle import model_cfg as mcfg
    dims = dict(vocab=32000, d=4096, heads=32, kv_heads=8, layers=2, ffn=11008, seed=1)
    gcfg = cf.model_cfg(arch=1, **dims)
    lengths = np.array([3400, 600, 250, 120, 40], np.int64)
    tokens = cf.gen_tokens(lengths, dims["vocab"], 23)
    model = cf.Model(ctx, gcfg)
    plan = cf.Plan.build(lengths, 1024, 1)
    ch, _, _, _ = plan.export()
    assert [int(x) for x in ch["kind"]].count(1) == 4
    r = model.run_plan(plan, lengths, tokens)
    assert r.recompute_forward_count == 3 and r.recompute_loss_mismatches == 0
    assert r.kv_completeness_violations == 0
    grads = model.grads_flat()
    # K = 2 retains one more chunk: bitwise identical gradients
    r2 = model.run_plan(cf.Plan.build(lengths, 1024, 2), lengths, tokens)
    assert r2.loss == r.loss and r2.recompute_forward_count == 2
    assert np.array_equal(model.grads_flat(), grads)
    params = model.params_flat()
    model.close()
    ol, og = llama_np.backward_full(mcfg(arch=1, **dims), params, lengths, tokens)
    del params
    rel = abs(r.loss - ol) / abs(ol)
    shapes = llama_np.Shapes(mcfg(arch=1, **dims))
    errs, off = [], 0
    for name, rr, cc in shapes.tensors():
        a, b = grads[off:off + rr * cc], og[off:off + rr * cc]
        off += rr * cc
        errs.append((name, float(np.abs(a - b).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-12))))
    worst = max(errs, key=lambda e: e[1])
    _report("production_width_llama_2layer", {"loss_gpu": r.loss, "loss_oracle": ol, "loss_rel": rel,
                                              "per_tensor": errs})
    assert rel <= LOSS_TOL, (r.loss, ol)
    assert worst[1] <= GRAD_TOL, worst
