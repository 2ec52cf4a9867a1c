"""Run-time validation of plans the executor is handed: a plan
loaded from chunk_plan.json (cf_plan_from_chunk_json) may describe dependent
chunks whose structure the per-group KV cache cannot honour.  The reference
raises ValidationError lazily from assemble_prefix (plan_runner.hpp:128-156,
"KV prefix does not cover the segment start ..."); the B200 executor checks
the same structure up front in cf_step_prepare and must never touch memory
outside the group's cache.  Also the normalizer-override semantics of
plan_runner.hpp:87-91 (batch_normalizer only without an override)."""
import json

import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi

pytestmark = pytest.mark.gpu


def _model(ctx):
    return cf.Model(ctx, cf.model_cfg(arch=1, vocab=64, d=64, heads=4, kv_heads=2, layers=1, ffn=128, seed=3))


def _doc(lengths, cs):
    return json.loads(cf.Plan.build(np.array(lengths, np.int64), cs, 1).chunk_json())


def _run(model, doc, lengths, k=1):
    lengths = np.array(lengths, np.int64)
    plan = cf.Plan.from_chunk_json(json.dumps(doc), k)
    return model.run_plan(plan, lengths, cf.gen_tokens(lengths, 64, 1))


def _dep(doc, gid):
    return [c for c in doc["chunks"] if c.get("group") == gid]


def test_reference_plan_round_trip_runs(ctx):
    model = _model(ctx)
    r = _run(model, _doc([70, 20, 9], 32), [70, 20, 9])
    assert np.isfinite(r.loss) and r.kv_completeness_violations == 0
    model.close()


def test_gap_in_group_is_rejected(ctx):
    model = _model(ctx)
    doc = _doc([70, 20, 9], 32)
    _dep(doc, 0)[1]["segments"][0]["start"] += 1  # member 1 no longer starts where member 0 ends
    _dep(doc, 0)[1]["segments"][0]["length"] -= 1
    _dep(doc, 0)[1]["total_tokens"] -= 1
    with pytest.raises(capi.CfError, match="KV prefix does not cover the segment start of sequence 0") as e:
        _run(model, doc, [70, 20, 9])
    assert e.value.code == 1
    model.close()


def test_multi_segment_dependent_chunk_is_rejected(ctx):
    model = _model(ctx)
    doc = _doc([70, 20, 9], 32)
    c = _dep(doc, 0)[2]  # last member: add a second segment (short sequence 2)
    c["segments"].append({"length": 9, "sequence": 2, "start": 0})
    c["total_tokens"] += 9
    doc["chunks"] = [x for x in doc["chunks"] if not (x["kind"] == "standalone" and
                                                    any(s["sequence"] == 2 for s in x["segments"]))]
    with pytest.raises(capi.CfError, match="exactly one segment") as e:
        _run(model, doc, [70, 20, 9])
    assert e.value.code == 1
    model.close()


def test_index_in_group_mismatch_is_rejected(ctx):
    model = _model(ctx)
    doc = _doc([70, 20, 9], 32)
    m = _dep(doc, 0)
    m[0]["index_in_group"], m[1]["index_in_group"] = 1, 0
    with pytest.raises(capi.CfError, match="index_in_group") as e:
        _run(model, doc, [70, 20, 9])
    assert e.value.code == 1
    model.close()


def test_group_spanning_two_sequences_is_rejected(ctx):
    model = _model(ctx)
    doc = _doc([70, 66, 9], 32)
    g0, g1 = _dep(doc, 0), _dep(doc, 1)
    # member 1 of group 0 taken from sequence 1 (same offsets): a forged group
    g0[1]["segments"][0]["sequence"] = g1[1]["segments"][0]["sequence"]
    with pytest.raises(capi.CfError, match="spans sequences") as e:
        _run(model, doc, [70, 66, 9])
    assert e.value.code == 1
    model.close()


def test_length_one_sequence_needs_a_normalizer_override(ctx):
    """batch_normalizer (toy_model.hpp:533-541) rejects a length-1 sequence,
    but run_plan only calls it without an override (plan_runner.hpp:89-91)."""
    model = _model(ctx)
    lengths = np.array([1, 30, 12], np.int64)
    tokens = cf.gen_tokens(lengths, 64, 4)
    plan = cf.Plan.build(lengths, 16, 1)
    with pytest.raises(capi.CfError, match="must have length >= 2") as e:
        model.run_plan(plan, lengths, tokens)
    assert e.value.code == 1
    r = model.run_plan(plan, lengths, tokens, normalizer=41.0)
    ref = model.run_plan(cf.Plan.build(lengths[1:], 16, 1), lengths[1:], tokens[1:], normalizer=41.0)
    # the length-1 sequence has no target: same loss as the batch without it
    assert abs(r.loss - ref.loss) <= 1e-6 * abs(ref.loss)
    model.close()
