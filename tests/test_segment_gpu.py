"""Operator-level parity: cf_segment_forward / cf_segment_backward
(detail::segment_forward / segment_backward, toy_model.hpp:206, :341).
Composing them over a split sequence the way run_plan does
(plan_runner.hpp:128-156, 306-321: prefixes from earlier segments' saved
K/V, incoming dK/dV from later segments' prefix gradients) must reproduce
run_plan on the same chunking bitwise, and the unchunked run within the
chunked == unchunked tolerance."""
import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi

pytestmark = pytest.mark.gpu

CASES = [  # arch, vocab, d, heads, kv_heads, layers, ffn
    ("toy", 0, 64, 64, 4, 2, 2, 0),
    ("llama", 1, 64, 128, 4, 2, 2, 256),
    ("llama-dh128", 1, 96, 256, 2, 1, 2, 512),
]


def _compose(model, tokens, bounds):
    n = len(tokens)
    targets = np.append(tokens[1:], -1).astype(np.int64)
    saved, tapes, loss_sum = [], [], 0.0
    for a, b in zip(bounds[:-1], bounds[1:]):
        pk = np.concatenate([s[0] for s in saved], axis=1) if saved else None
        pv = np.concatenate([s[1] for s in saved], axis=1) if saved else None
        ls, sk, sv, tape = model.segment_forward(tokens[a:b], targets[a:b], pk, pv, keep_tape=True)
        loss_sum += ls
        saved.append((sk, sv))
        tapes.append(tape)
    norm = float(n - 1)
    model.zero_grads()
    L, _, kvw = model.kv_shape(0)
    dk = np.zeros((L, n, kvw))
    dv = np.zeros((L, n, kvw))
    for i in reversed(range(len(tapes))):
        a, b = bounds[i], bounds[i + 1]
        pk = np.concatenate([s[0] for s in saved[:i]], axis=1) if i else None
        pv = np.concatenate([s[1] for s in saved[:i]], axis=1) if i else None
        dpk, dpv = model.segment_backward(tapes[i], norm, pk, pv, dk[:, a:b].copy(), dv[:, a:b].copy())
        dk[:, :a] += dpk
        dv[:, :a] += dpv
        tapes[i].close()
    return loss_sum / norm, model.grads_flat()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_segments_compose_to_run_plan(ctx, case):
    _, arch, V, d, H, KVH, L, ffn = case
    cfg = cf.model_cfg(arch=arch, vocab=V, d=d, heads=H, kv_heads=KVH, layers=L, ffn=ffn, seed=5)
    lengths = np.array([200], np.int64)
    tokens = cf.gen_tokens(lengths, V, 31)
    model = cf.Model(ctx, cfg)
    # run_plan with chunk 70, K = 3: chunks [0,70) [70,140) [140,200), all retained
    r = model.run_plan(cf.Plan.build(lengths, 70, 3), lengths, tokens)
    g_plan = model.grads_flat()
    loss, g_seg = _compose(model, tokens, [0, 70, 140, 200])
    assert loss == r.loss
    assert np.array_equal(g_seg, g_plan)
    # and the unchunked run, within the chunked == unchunked tolerance
    f = model.backward_full(lengths, tokens)
    g_full = model.grads_flat()
    assert abs(loss - f.loss) / abs(f.loss) < 1e-4
    off = 0
    for i in range(model.num_tensors()):
        _, rr, cc = model.tensor_info(i)
        a, b = g_seg[off:off + rr * cc], g_full[off:off + rr * cc]
        off += rr * cc
        assert np.abs(a - b).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-12) < 1e-2, i
    model.close()


def test_segment_forward_saved_kv_and_loss(ctx):
    """saved K/V of a segment equal the rows the same positions get when the
    whole sequence is one segment; loss_sum is unnormalized and skips -1."""
    cfg = cf.model_cfg(arch=1, vocab=64, d=128, heads=4, kv_heads=2, layers=2, ffn=256, seed=2)
    model = cf.Model(ctx, cfg)
    tokens = cf.gen_tokens(np.array([90], np.int64), 64, 4)
    targets = np.append(tokens[1:], -1).astype(np.int64)
    l_all, k_all, v_all, t = model.segment_forward(tokens, targets, keep_tape=False)
    assert t is None
    l1, k1, v1, _ = model.segment_forward(tokens[:50], targets[:50], keep_tape=False)
    l2, k2, v2, _ = model.segment_forward(tokens[50:], targets[50:], k1, v1, keep_tape=False)
    assert np.array_equal(k1, k_all[:, :50]) and np.array_equal(v1, v_all[:, :50])
    assert np.allclose(k2, k_all[:, 50:], rtol=0, atol=2e-2)  # different GEMM shapes -> bf16 rounding
    assert abs((l1 + l2) - l_all) / l_all < 1e-4
    no_targets = np.full(50, -1, np.int64)
    l0, _, _, _ = model.segment_forward(tokens[:50], no_targets, keep_tape=False)
    assert l0 == 0.0
    model.close()


def test_segment_errors(ctx):
    cfg = cf.model_cfg(arch=0, vocab=32, d=64, heads=4, kv_heads=2, layers=1, seed=1)
    model = cf.Model(ctx, cfg)
    tokens = np.arange(10, dtype=np.int32)
    targets = np.append(tokens[1:], -1).astype(np.int64)
    with pytest.raises(capi.CfError) as e:  # backward without a retained tape
        model.segment_backward(None, 9.0)
    assert e.value.code == 1 and "retained tape" in str(e.value)
    bad = tokens.copy()
    bad[3] = 99
    with pytest.raises(capi.CfError):  # out-of-vocabulary token
        model.segment_forward(bad, targets)
    _, sk, sv, tape = model.segment_forward(tokens, targets)
    with pytest.raises(capi.CfError):  # non-positive normalizer
        model.segment_backward(tape, 0.0)
    with pytest.raises(capi.CfError):  # prefix_len > 0 without prefix keys
        lib = capi.lib()
        capi.check(lib.cf_segment_forward(model.ctx.h, model.h, capi._p(tokens), capi.C.c_int64(10),
                                          capi._p(targets), None, None, capi.C.c_int64(4), 0, None, None, None,
                                          None))
    tape.close()
    model.close()


def test_cpp_facade_segment_ops(tmp_path):
    """Reference-style C++ caller of detail::segment_forward/backward
    (include/chunkflow_b200.hpp) reproduces run_plan exactly."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2503_02356_b200")
    exe = tmp_path / "segment_facade_test"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "segment_facade_test.cpp"), f"-L{lib}", "-lchunkflow_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    assert "loss_diff=0 grad_diff=0" in out, out
