"""Pins the CPU oracle (oracle/cf_oracle.cpp) before it is trusted:
  * against the reference's own known answers (test_chunker.cpp,
    test_scheduler.cpp, test_plan_runner.cpp),
  * against the committed golden fixtures generated from the reference
    (tests/golden/make_golden.py),
  * bitwise against the reference itself when oracle/_ref is present.
"""
import json
import os

import numpy as np
import pytest

from oracle.oracle import c1_batch, c1_cfg, model_cfg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))
HAVE_REF = os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libcfref.so"))


def _plan_equal(lib, doc):
    ch, sg = lib.construct_chunks(doc["lengths"], doc["chunk_size"])
    ev, dg = lib.schedule_step(doc["lengths"], doc["chunk_size"], doc["k"])
    assert ch.tolist() == [tuple(x) for x in doc["chunks"]]
    assert sg.tolist() == [tuple(x) for x in doc["segments"]]
    assert ev.tolist() == [tuple(x) for x in doc["events"]]
    assert [int(x) for x in dg.tolist()] == doc["diag"]
    assert lib.listing(doc["lengths"], doc["chunk_size"], doc["k"]) == doc["listing"]


def test_oracle_worked_batches_match_golden(oracle):
    for key in ("worked_cs2_k1", "worked_cs4_k1", "ffd_beaten_cs10", "c1_plan"):
        _plan_equal(oracle, GOLD[key])


def test_oracle_random_plans_match_golden(oracle):
    for doc in GOLD["random"]:
        _plan_equal(oracle, doc)


def test_known_answers_from_reference_tests(oracle):
    # SplitLong (test_chunker.cpp:108-112): 37K @ 8K -> [8192 x4, 5120]
    ch, sg = oracle.construct_chunks([37 * 1024], 8 * 1024)
    assert [int(x) for x in ch["total_tokens"]] == [8192, 8192, 8192, 8192, 5120]
    assert [int(x) for x in sg["start_token"]] == [0, 8192, 16384, 24576, 32768]
    # a sequence of exactly chunk_size stays standalone (:182-187)
    ch, _ = oracle.construct_chunks([4], 4)
    assert ch["kind"].tolist() == [0]
    # FFD needs 3 bins, exhaustive packing finds 2 (:141-152)
    ch, _ = oracle.construct_chunks([5, 4, 4, 3, 2, 2], 10)
    assert len(ch) == 2
    # schedule_group(4,1) sequence (test_scheduler.cpp:54-67)
    ev, dg = oracle.schedule_group(4, 1, 10)
    kinds = [(int(e["kind"]), int(e["chunk_id"]), int(e["is_recompute"])) for e in ev]
    assert kinds == [(0, 1, 0), (0, 2, 0), (0, 3, 0), (1, 4, 0), (2, 4, 0), (1, 3, 1), (2, 3, 0), (1, 2, 1),
                     (2, 2, 0), (1, 1, 1), (2, 1, 0)]
    assert (int(dg["peak_retained_tokens"]), int(dg["recompute_token_count"])) == (10, 30)
    _, dg2 = oracle.schedule_group(4, 2, 10)
    assert (int(dg2["peak_retained_tokens"]), int(dg2["recompute_token_count"])) == (20, 20)
    # recompute law: n + max(0, n-k) forwards (:79-97)
    for n in range(1, 9):
        for k in range(1, 9):
            ev, _ = oracle.schedule_group(n, k)
            assert int((ev["kind"] != 2).sum()) == n + max(0, n - k)


def test_c1_plan_matches_survey_appendix(oracle):
    lengths, _ = c1_batch(oracle)
    assert lengths.tolist() == [294, 21, 225, 644, 644, 308, 64, 443, 24, 184, 783, 35, 648, 26, 601, 325, 672, 38,
                                259, 74, 132, 563, 173, 17, 30, 290, 151, 94, 257, 74, 36, 89, 2048]
    ch, sg = oracle.construct_chunks(lengths, 512)
    assert len(ch) == 26
    first = [sorted(int(s["sequence_id"]) for s in sg[c["seg_offset"]:c["seg_offset"] + c["seg_count"]])
             for c in ch[:8]]
    assert first == [[6, 7], [9, 15], [5, 22, 24], [0, 13, 17, 26], [20, 25, 31], [2, 8, 18], [19, 27, 28, 29],
                     [1, 11, 23, 30]]
    ev, dg = oracle.schedule_step(lengths, 512, 2)
    assert len(ev) == 54 and int(dg["peak_retained_tokens"]) == 1024 and int(dg["recompute_token_count"]) == 1024


def test_verify_defaults_bitwise(oracle):
    g = GOLD["verify_defaults"]
    cfg = model_cfg()
    assert np.array_equal(oracle.init(cfg), np.array(g["params"]))
    assert oracle.gen_tokens(g["lengths"], 32, 11).tolist() == g["tokens"]
    loss, grads, instr = oracle.run_plan(cfg, g["lengths"], g["tokens"], 16, 1)
    assert loss == g["loss"] == 3.476771351579374
    assert np.array_equal(grads, np.array(g["grads"]))
    assert instr.tolist() == g["instr"]
    lf, gf = oracle.backward_full(cfg, g["lengths"], g["tokens"])
    assert lf == g["loss_full"]
    assert np.array_equal(gf, np.array(g["grads_full"]))


def test_c1_run_plan_matches_reference_golden(oracle):
    """loss 5.5455568137389548, sums of grads."""
    lengths, tokens = c1_batch(oracle)
    g = GOLD["c1_run"]
    assert tokens[:16].tolist() == g["token_head"] and int(tokens.sum()) == g["token_sum"]
    loss, grads, instr = oracle.run_plan(c1_cfg(), lengths, tokens, 512, 2)
    assert loss == g["loss"]
    assert instr.tolist() == g["instr"]
    head = grads[-256 * 256:]
    assert head[:3].tolist() == g["head_grad_00_02"]
    assert abs(grads.sum() - g["grad_sum"]) < 1e-15
    assert abs(np.abs(grads).sum() - g["grad_abs_sum"]) < 1e-12


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_oracle_bitwise_vs_reference_random_models(oracle, reference):
    rng = np.random.default_rng(7)
    for trial in range(12):
        H = int(rng.choice([1, 2, 4]))
        KVH = int(rng.choice([h for h in (1, 2, 4) if H % h == 0]))
        d = H * int(rng.choice([2, 4, 8]))
        cfg = model_cfg(vocab=int(rng.integers(2, 40)), d=d, heads=H, kv_heads=KVH,
                        layers=int(rng.integers(1, 3)), seed=int(rng.integers(1, 99)))
        n = int(rng.integers(1, 6))
        lengths = rng.integers(2, 40, n)
        tokens = oracle.gen_tokens(lengths, cfg.vocab_size, trial)
        cs = int(rng.integers(2, 24))
        k = int(rng.integers(1, 4))
        lo, go, io = oracle.run_plan(cfg, lengths, tokens, cs, k)
        lr, gr, ir = reference.run_plan(cfg, lengths, tokens, cs, k)
        assert lo == lr and np.array_equal(go, gr) and io.tolist() == ir.tolist()
        lo, go = oracle.backward_full(cfg, lengths, tokens)
        lr, gr = reference.backward_full(cfg, lengths, tokens)
        assert lo == lr and np.array_equal(go, gr)
        lo, go, _ = oracle.run_plan(cfg, lengths, tokens, cs, k, corrupt=True)
        lr, gr, _ = reference.run_plan(cfg, lengths, tokens, cs, k, corrupt=True)
        assert np.array_equal(go, gr)


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_oracle_plans_bitwise_vs_reference_sweep(oracle, reference):
    rng = np.random.default_rng(11)
    for _ in range(400):
        n = int(rng.integers(1, 30))
        cs = int(rng.integers(1, 80))
        k = int(rng.integers(1, 6))
        lengths = rng.integers(1, 300, n)
        ids = rng.permutation(1000)[:n]
        a = oracle.construct_chunks(lengths, cs, ids)
        b = reference.construct_chunks(lengths, cs, ids)
        assert a[0].tolist() == b[0].tolist() and a[1].tolist() == b[1].tolist()
        ea, da = oracle.schedule_step(lengths, cs, k, ids)
        eb, db = reference.schedule_step(lengths, cs, k, ids)
        assert ea.tolist() == eb.tolist() and da.tolist() == db.tolist()


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_synthesize_matches_reference(oracle, reference):
    for seed in (1, 3, 99):
        assert np.array_equal(oracle.synthesize(500, seed, preset=1), reference.synthesize(500, seed, preset=1))
        a = oracle.synthesize(300, seed, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)
        b = reference.synthesize(300, seed, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)
        assert np.array_equal(a, b)


def test_llama_oracle_finite_differences(oracle):
    """The Llama extension has no reference: pin its analytic backward with
    central differences (toy_model.hpp:602-650 recipe, eps 1e-5)."""
    cfg = model_cfg(arch=1, vocab=11, d=8, heads=2, kv_heads=1, layers=2, ffn=12, seed=5, rope_theta=100.0)
    lengths = np.array([5, 9, 3])
    tokens = oracle.gen_tokens(lengths, 11, 4)
    params = oracle.init(cfg)
    rng = np.random.default_rng(0)
    params = params + rng.normal(0, 0.05, params.shape)  # move norm gains off 1
    loss, grads = oracle.backward_full(cfg, lengths, tokens, params=params)
    idx = rng.choice(len(params), 120, replace=False)
    eps = 1e-5
    for i in idx:
        p = params.copy()
        p[i] += eps
        lp = oracle.forward_full(cfg, lengths, tokens, params=p)
        p[i] -= 2 * eps
        lm = oracle.forward_full(cfg, lengths, tokens, params=p)
        fd = (lp - lm) / (2 * eps)
        assert abs(fd - grads[i]) <= 1e-6 + 1e-4 * abs(fd), (i, fd, grads[i])


def test_llama_oracle_chunked_equals_unchunked(oracle):
    cfg = model_cfg(arch=1, vocab=17, d=16, heads=4, kv_heads=2, layers=2, ffn=24, seed=3)
    lengths = np.array([40, 7, 19, 2])
    tokens = oracle.gen_tokens(lengths, 17, 8)
    lf, gf = oracle.backward_full(cfg, lengths, tokens)
    for cs, k in ((8, 1), (8, 3), (16, 2), (64, 1)):
        l, g, instr = oracle.run_plan(cfg, lengths, tokens, cs, k)
        assert abs(l - lf) <= 1e-12 * abs(lf)
        assert np.max(np.abs(g - gf)) <= 1e-9 * np.max(np.abs(gf))
        assert instr[2] == 0 and instr[3] == 0


def _per_tensor_rel(shapes, a, b):
    out, off = [], 0
    for name, r, c in shapes.tensors():
        x, y = a[off:off + r * c], b[off:off + r * c]
        off += r * c
        out.append((name, float(np.abs(x - y).max() / max(np.abs(x).max(), np.abs(y).max(), 1e-300))))
    return out


@pytest.mark.parametrize("arch,V,d,H,KVH,L,ffn,lengths", [
    (0, 32, 16, 4, 2, 2, 0, [8, 8, 16, 32]),           # CLI verify defaults' model
    (0, 256, 256, 4, 2, 2, 0, [294, 21, 225, 64]),     # C1 widths
    (1, 96, 64, 4, 2, 2, 128, [30, 64, 7, 2]),
    (1, 50, 128, 4, 1, 1, 96, [40, 3, 2]),            # GQA 4:1, head_dim 32
    (1, 40, 256, 2, 2, 2, 320, [70, 12]),             # MHA, head_dim 128
])
def test_vectorised_oracle_matches_cpp_oracle(oracle, arch, V, d, H, KVH, L, ffn, lengths):
    """oracle/llama_np.py (BLAS fp64 restatement used for production-width
    GPU parity) == cf_oracle.cpp backward_full / forward_full, per tensor, to
    1e-12 relative (the summation order differs, so not bitwise)."""
    from oracle import llama_np
    cfg = model_cfg(arch=arch, vocab=V, d=d, heads=H, kv_heads=KVH, layers=L, ffn=ffn, seed=7)
    lengths = np.array(lengths, np.int64)
    tokens = oracle.gen_tokens(lengths, V, 3)
    params = oracle.init(cfg)
    if arch == 1:  # move the norm gains off 1 so their gradients are exercised
        params = params + np.random.default_rng(1).normal(0, 0.02, params.shape)
    ol, og = oracle.backward_full(cfg, lengths, tokens, params=params)
    nl, ng = llama_np.backward_full(cfg, params, lengths, tokens)
    assert abs(nl - ol) <= 1e-12 * abs(ol)
    assert abs(llama_np.forward_full(cfg, params, lengths, tokens) - ol) <= 1e-12 * abs(ol)
    worst = max(_per_tensor_rel(llama_np.Shapes(cfg), ng, og), key=lambda e: e[1])
    assert worst[1] <= 1e-12, worst


def test_vectorised_oracle_c1_matches_reference_golden(oracle):
    """The vectorised oracle on the C1 canonical batch reproduces the
    reference's golden run_plan loss — chunked == unchunked
    holds in the reference at 9.9e-15."""
    from oracle import llama_np
    lengths, tokens = c1_batch(oracle)
    cfg = c1_cfg()
    loss, grads = llama_np.backward_full(cfg, oracle.init(cfg), lengths, tokens)
    g = GOLD["c1_run_plan"] if "c1_run_plan" in GOLD else None
    assert abs(loss - 5.5455568137389548) <= 1e-13 * 5.5455568137389548
    assert abs(grads.sum() - 0.0071303868983342488) <= 1e-9
    assert abs(np.abs(grads).sum() - 6.5459081754140787) <= 1e-11 * 6.5459081754140787
    del g


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_product_synthesize_and_sample_batch_match_reference(reference):
    """Product cf_synthesize / cf_sample_batch (csrc/host/plan.cpp) against
    the compiled reference synthesize / sample_batch (dataset.hpp:207-268):
    presets, explicit specs, epoch slices, the short last batch, past-epoch."""
    import ctypes as C
    from paper_2503_02356_b200 import capi
    for seed in (1, 3, 7, 99, 2**63 + 5):
        for preset, kw in ((1, {}), (2, {}), (0, dict(bounds=[1024], fracs=[1.0], max_length=1024)),
                           (0, dict(bounds=[64, 512, 4096, 32768], fracs=[0.5, 0.8, 0.99, 0.999], max_length=40000))):
            a = capi.synthesize(400, seed, preset=preset, **kw)
            b = reference.synthesize(400, seed, preset=preset, **kw)
            assert np.array_equal(a, b), (seed, preset)
    lengths = np.arange(1, 102, dtype=np.int64)
    for seed in (0, 5, 123456789):
        for gbs in (1, 7, 32, 101, 150):
            for step in range(0, 101 // gbs + 2):
                got = capi.sample_batch(len(lengths), gbs, step, seed)
                ids = np.zeros(gbs, np.int64)
                cnt = C.c_int64()
                reference._check(reference.lib.cfr_sample_batch(
                    lengths.ctypes.data_as(C.POINTER(C.c_int64)), C.c_int64(len(lengths)), C.c_int64(gbs),
                    C.c_int64(step), C.c_uint64(seed), ids.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(cnt)))
                assert np.array_equal(got, ids[:cnt.value]), (seed, gbs, step)
    # the reference's spec / argument errors (DistributionSpec::validate,
    # dataset.hpp:40-71; sample_batch :245-249) are errors here too
    bad = [dict(bounds=[1024], fracs=[1.0], max_length=2048), dict(bounds=[1024], fracs=[0.9], max_length=1024),
           dict(bounds=[1], fracs=[1.0], max_length=1), dict(bounds=[64, 32], fracs=[0.5, 1.0], max_length=64),
           dict(bounds=[64, 128], fracs=[0.5, 0.5], max_length=128), dict(bounds=[64], fracs=[0.0], max_length=64),
           dict(bounds=[1024], fracs=[1.0], max_length=512)]
    for kw in bad:
        with pytest.raises(ValueError):
            reference.synthesize(10, 1, preset=0, **kw)
        with pytest.raises(capi.CfError) as e:
            capi.synthesize(10, 1, preset=0, **kw)
        assert e.value.code == 1, kw
    for args in ((0, 4, 0, 1), (10, 0, 0, 1), (10, 4, -1, 1)):
        with pytest.raises(capi.CfError):
            capi.sample_batch(*args)
