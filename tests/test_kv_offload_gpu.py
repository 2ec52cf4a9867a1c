"""KV offload (cf_run_opts.kv_offload; the offloading PAPER.md:417 leaves
for future work): a dependent group's K/V cache and fp32 dK/dV accumulators
live in pinned host memory, the device keeps two one-layer staging buffers,
and each layer's rows move on a copy stream around its attention.  The math
is untouched, so loss and every gradient must be BITWISE those of the
resident-state run, while the device KV footprint drops to 2/L of the state."""
import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi

pytestmark = pytest.mark.gpu

CASES = [
    # name, arch, vocab, d, heads, kv_heads, layers, ffn, lengths, chunk, k
    ("toy-dh64-k1", 0, 64, 128, 2, 1, 3, 0, [300, 20, 41, 170], 64, 1),
    ("llama-dh128-k1", 1, 96, 256, 2, 1, 4, 512, [900, 77, 500, 33], 128, 1),
    ("llama-dh128-k2-two-groups", 1, 96, 256, 2, 1, 3, 512, [700, 260, 640, 40], 128, 2),
    ("llama-gqa-dh64", 1, 96, 256, 4, 2, 2, 384, [333, 90, 200], 96, 1),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_offload_bitwise_equals_resident(ctx, case):
    _, arch, V, d, H, KVH, L, ffn, lengths, cs, k = case
    model = cf.Model(ctx, cf.model_cfg(arch=arch, vocab=V, d=d, heads=H, kv_heads=KVH, layers=L, ffn=ffn, seed=3))
    lengths = np.array(lengths, np.int64)
    tokens = cf.gen_tokens(lengths, V, 7)
    plan = cf.Plan.build(lengths, cs, k)
    ref = model.run_plan(plan, lengths, tokens)
    g_ref = model.grads_flat()
    for _ in range(2):  # twice: the cached pinned blocks are reused
        r = model.run_plan(plan, lengths, tokens, kv_offload=True)
        assert r.loss == ref.loss
        assert r.recompute_loss_mismatches == 0 and r.kv_completeness_violations == 0
        assert r.recompute_forward_count == ref.recompute_forward_count
        assert np.array_equal(model.grads_flat(), g_ref)
        # two one-layer staging buffers instead of L layers (with L = 2 the
        # staging IS the whole state, up to allocation rounding)
        assert r.kv_hbm_bytes <= ref.kv_hbm_bytes * min(1.0, 2.0 / L) * 1.01
    model.close()


def test_offload_forced_pair_gemms_and_prefix_epilogue(ctx):
    """CTA-pair GEMMs with the RoPE + KV-copy epilogue writing the staged
    cache rows (kv width 256) and a 4-chunk group with K = 1."""
    capi.check(capi.lib().cf_debug_set_gemm_mode(2))
    try:
        model = cf.Model(ctx, cf.model_cfg(arch=1, vocab=96, d=256, heads=2, kv_heads=2, layers=2, ffn=384, seed=5))
        lengths = np.array([1000, 130, 301, 64], np.int64)
        tokens = cf.gen_tokens(lengths, 96, 13)
        plan = cf.Plan.build(lengths, 256, 1)
        ref = model.run_plan(plan, lengths, tokens)
        g_ref = model.grads_flat()
        r = model.run_plan(plan, lengths, tokens, kv_offload=True)
        g = model.grads_flat()
    finally:
        capi.check(capi.lib().cf_debug_set_gemm_mode(0))
    assert r.loss == ref.loss and np.array_equal(g, g_ref)
    model.close()


def test_offload_with_pipeline_stages_and_tape_budget(ctx):
    """Offload composes with the chunk-aware 1F1B stage runner and its tape
    budget: bitwise equal to the unsplit resident run."""
    cfg = cf.model_cfg(arch=1, vocab=120, d=256, heads=2, kv_heads=1, layers=4, ffn=512, seed=7)
    lengths = np.array([40, 900, 77, 260, 500, 33], np.int64)
    tokens = cf.gen_tokens(lengths, 120, 11)
    plan = cf.Plan.build(lengths, 128, 1)
    full = cf.Model(ctx, cfg)
    st = cf.Step(full, plan, lengths, tokens)
    ref = st.run()
    ref_g = {full.tensor_info(i)[0]: full.get_grad(i) for i in range(full.num_tensors())}
    st.close()
    full.close()
    stages = [cf.Model(ctx, cfg, stage=s, num_stages=2) for s in range(2)]
    sp = cf.Step(stages[0], plan, lengths, tokens)
    r = sp.run_pp_local(stages, 1, tape_budget=2, kv_offload=True)
    assert r.loss == ref.loss and r.recompute_loss_mismatches == 0
    for m in stages:
        for i in range(m.num_tensors()):
            assert np.array_equal(m.get_grad(i), ref_g[m.tensor_info(i)[0]]), m.tensor_info(i)[0]
    sp.close()
    for m in stages:
        m.close()


def test_offload_device_kv_is_two_layers(ctx):
    """Device KV bytes: 2 staging layers instead of L layers of state."""
    L = 8
    model = cf.Model(ctx, cf.model_cfg(arch=1, vocab=64, d=256, heads=2, kv_heads=1, layers=L, ffn=512, seed=1))
    lengths = np.array([4096, 30], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 1)
    plan = cf.Plan.build(lengths, 1024, 1)
    a = model.run_plan(plan, lengths, tokens)
    b = model.run_plan(plan, lengths, tokens, kv_offload=True)
    assert a.loss == b.loss
    assert abs(b.kv_hbm_bytes / a.kv_hbm_bytes - 2.0 / L) < 0.01
    model.close()
