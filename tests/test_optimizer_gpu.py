"""Fused AdamW (csrc/kernels/optim.cu) against a numpy
restatement of torch.optim.AdamW in float32 on the same gradients, over
several training steps (each step: chunked run_plan on the GPU -> grads ->
one fused update of fp32 master, moments and bf16 working weights), with
global-norm clipping and decoupled weight decay (not on RMSNorm gains)."""
import numpy as np
import pytest

import paper_2503_02356_b200 as cf

pytestmark = pytest.mark.gpu


def _bf16(x):
    m, e = np.frexp(np.asarray(x, np.float64))
    return np.ldexp(np.rint(m * 256.0), e - 8)


def test_adamw_matches_numpy_over_steps(ctx):
    cfg = cf.model_cfg(arch=1, vocab=96, d=128, heads=4, kv_heads=2, layers=2, ffn=256, seed=4)
    lengths = np.array([150, 40, 9, 70], np.int64)
    tokens = cf.gen_tokens(lengths, 96, 2)
    plan = cf.Plan.build(lengths, 64, 1)
    model = cf.Model(ctx, cfg)
    model.adamw_init()
    n = model.num_tensors()
    names = [model.tensor_info(i)[0] for i in range(n)]
    master = [model.get_master(i).astype(np.float32) for i in range(n)]
    for i in range(n):  # master starts as the working weights
        assert np.array_equal(master[i], model.get_param(i).astype(np.float32))
    m = [np.zeros_like(w) for w in master]
    v = [np.zeros_like(w) for w in master]
    lr, b1, b2, eps, wd, clip = 3e-3, 0.9, 0.95, 1e-8, 0.1, 0.5
    losses = []
    for t in range(1, 5):
        r = model.run_plan(plan, lengths, tokens)
        losses.append(r.loss)
        grads = [model.get_grad(i).astype(np.float32) for i in range(n)]
        norm = np.sqrt(sum(float((g.astype(np.float64) ** 2).sum()) for g in grads))
        got_norm = model.adamw_step(lr, b1, b2, eps, wd, clip)
        assert abs(got_norm - norm) <= 1e-5 * norm
        coef = np.float32(min(1.0, clip / (norm + 1e-6)))
        step_size = np.float32(lr / (1 - b1 ** t))
        sqrt_bc2 = np.float32(np.sqrt(1 - b2 ** t))
        for i in range(n):
            g = grads[i] * coef
            if "norm" not in names[i]:
                master[i] = master[i] - np.float32(lr * wd) * master[i]
            m[i] = np.float32(b1) * m[i] + np.float32(1 - b1) * g
            v[i] = np.float32(b2) * v[i] + np.float32(1 - b2) * g * g
            master[i] = master[i] - step_size * m[i] / (np.sqrt(v[i]) / sqrt_bc2 + np.float32(eps))
        for i in range(n):
            got = model.get_master(i)
            ref = master[i].astype(np.float64)
            err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-12)
            assert err < 2e-6, (t, names[i], err)
            w = model.get_param(i)
            if "norm" in names[i]:
                assert np.array_equal(w, got)            # fp32 gains are the master
            else:
                assert np.array_equal(w, _bf16(got)), names[i]  # bf16 working copy of the master
            master[i] = got.astype(np.float32)  # track the GPU's rounding from here on
    assert losses[-1] < losses[0]  # it trains
    model.close()


def test_adamw_requires_init_and_validates(ctx):
    model = cf.Model(ctx, cf.model_cfg(arch=0, vocab=32, d=64, heads=4, kv_heads=2, layers=1, seed=1))
    with pytest.raises(cf.capi.CfError):
        model.adamw_step(1e-3)
    model.adamw_init()
    with pytest.raises(cf.capi.CfError):
        model.adamw_step(1e-3, beta1=1.5)
    model.close()
