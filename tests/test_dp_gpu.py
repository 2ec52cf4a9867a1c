"""The NCCL data-parallel path inside the library (dlopen'd NCCL, comm init
from a launcher-broadcast unique id, fp32 gradient + loss all-reduce on the
context stream), exercised on one GPU with a 1-rank communicator: the result
must equal the run without a DP group bitwise.  Multi-rank partitioning is
covered on CPU by tests/test_dp_gloo.py."""
import numpy as np
import pytest

import paper_2503_02356_b200 as cf

pytestmark = pytest.mark.gpu


def test_single_rank_nccl_allreduce_is_identity():
    cfg = cf.model_cfg(arch=cf.ARCH_LLAMA, vocab=64, d=128, heads=2, kv_heads=1, layers=2, ffn=256, seed=3)
    lengths = np.array([200, 30, 77], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 2)
    plan = cf.Plan.build(lengths, 64, 1)
    a = cf.Context(0)
    ma = cf.Model(a, cfg)
    ra = ma.run_plan(plan, lengths, tokens)
    ga = ma.grads_flat()
    b = cf.Context(0)
    b.init_dp(0, 1, cf.Context.nccl_unique_id())
    mb = cf.Model(b, cfg)
    rb = mb.run_plan(plan.partition(1, 0), lengths, tokens)
    gb = mb.grads_flat()
    assert ra.loss == rb.loss
    assert np.array_equal(ga, gb)
