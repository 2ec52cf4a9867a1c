"""Pipeline-parallel planning (product C++, host/pp.cpp through the C-ABI) is
bit-exact with the reference simulator (pipeline.hpp): per-stage op streams
(build_stage_order :178-210), dispatch times (run_dispatch :98-162),
makespan and bubble_ratio (:325-331), for the state-aware and the plain
1F1B schedules.  The reference runs from oracle/_ref (compiled in place)."""
import json
import os

import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi
from oracle.oracle import c1_batch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _product_trace(lengths, cs, k, stages, cost, backward_first=True):
    plan = cf.Plan.build(lengths, cs, k)
    c = dict(zip(("gamma", "alpha", "beta", "backward_multiplier", "hop_latency"), cost))
    ops, busy, busy_t, r = capi.pp_simulate(plan, stages, k, c, backward_first)
    return ops, busy, busy_t, r


def _compare(reference, lengths, cs, k, stages, cost=(0.0, 1.0, 0.0, 2.0, 0.0), backward_first=True):
    rops, rbusy, rbusy_t, rmk, rbb = reference.pp_trace(lengths, cs, k, stages, cost, 1, backward_first)
    ops, busy, busy_t, r = _product_trace(lengths, cs, k, stages, cost, backward_first)
    assert ops.shape == rops.shape[:2]
    assert np.array_equal(ops["kind"], rops[..., 0].astype(np.int64))
    assert np.array_equal(ops["chunk_id"], rops[..., 1].astype(np.int64))
    # bitwise: same additions in the same order
    assert np.array_equal(ops["start"], rops[..., 2]) and np.array_equal(ops["end"], rops[..., 3])
    assert np.array_equal(busy, rbusy) and np.array_equal(busy_t, rbusy_t)
    assert r.makespan == rmk and r.bubble_ratio == rbb
    return r


def test_worked_batch_golden():
    """test_pipeline.cpp:141-211 / SURVEY §6: 56 / 54 / 46 / 60 units."""
    sim = GOLD["simulator"]
    _, _, _, r = capi.pp_simulate_1f1b([1, 1, 2, 4], 4)
    assert (r.makespan, r.bubble_ratio) == tuple(sim["1f1b"])
    for key, cs, k in (("sa_k1", 2, 1), ("sa_k2", 2, 2), ("sa_cs4", 4, 1)):
        _, _, _, r = capi.pp_simulate(cf.Plan.build([1, 1, 2, 4], cs, k), 4, k)
        assert (r.makespan, r.bubble_ratio) == tuple(sim[key]), key
    assert round(100 * capi.pp_simulate(cf.Plan.build([1, 1, 2, 4], 2, 1), 4, 1)[3].bubble_ratio, 2) == 55.56


@pytest.mark.parametrize("stages", [1, 2, 3, 4, 6])
@pytest.mark.parametrize("cs,k", [(2, 1), (2, 2), (4, 1), (1, 1), (1, 3)])
def test_worked_batch_traces(reference, stages, cs, k):
    _compare(reference, [1, 1, 2, 4], cs, k, stages)
    _compare(reference, [1, 1, 2, 4], cs, k, stages, backward_first=False)
    _compare(reference, [1, 1, 2, 4], cs, k, stages, cost=(0.5, 1.0, 0.25, 1.5, 0.75))


def test_c1_batch_traces(reference, oracle):
    lengths, _ = c1_batch(oracle)
    for stages in (2, 4, 8):
        for k in (1, 2, 3):
            _compare(reference, lengths, 512, k, stages, cost=(0.0, 1.0, 1.05e-5, 2.0, 3.0))


def test_random_traces(reference):
    rng = np.random.default_rng(7)
    for _ in range(60):
        n = int(rng.integers(1, 40))
        cs = int(rng.integers(4, 300))
        lengths = rng.integers(1, 4 * cs, n)
        stages = int(rng.integers(1, 9))
        k = int(rng.integers(1, 5))
        cost = (float(rng.random()), float(rng.random()) + 0.1, float(rng.random()) * 1e-3,
                float(rng.random()) * 3 + 0.5, float(rng.random()) * 5)
        _compare(reference, lengths, cs, k, stages, cost, backward_first=bool(rng.integers(0, 2)))


def test_1f1b_random(reference):
    rng = np.random.default_rng(11)
    for _ in range(30):
        lengths = rng.integers(1, 500, int(rng.integers(1, 30)))
        stages = int(rng.integers(1, 9))
        cost = (0.0, 1.0, float(rng.random()) * 1e-3, 2.0, float(rng.random()))
        rops, rbusy, rbusy_t, rmk, rbb = reference.pp_trace(lengths, 1, 1, stages, cost, 0, False)
        ops, busy, busy_t, r = capi.pp_simulate_1f1b(
            lengths, stages, dict(zip(("gamma", "alpha", "beta", "backward_multiplier", "hop_latency"), cost)))
        assert np.array_equal(ops["kind"], rops[..., 0].astype(np.int64))
        assert np.array_equal(ops["chunk_id"], rops[..., 1].astype(np.int64))
        assert np.array_equal(ops["start"], rops[..., 2]) and np.array_equal(ops["end"], rops[..., 3])
        assert (r.makespan, r.bubble_ratio) == (rmk, rbb)


def test_measured_costs_override():
    """Simulator-in-the-loop: per-chunk measured costs replace the model."""
    plan = cf.Plan.build([1, 1, 2, 4], 2, 1)
    n = plan.counts()[0]
    fw = np.arange(1, n + 1, dtype=np.float64)
    _, _, _, r1 = capi.pp_simulate(plan, 2, 1, fwd_cost=fw, bwd_cost=2 * fw)
    _, _, _, r2 = capi.pp_simulate(plan, 2, 1, cost={"alpha": 0.0, "gamma": 1.0})
    assert r1.makespan > r2.makespan > 0
    ops, busy, busy_t, r = capi.pp_simulate(plan, 1, 1, fwd_cost=fw, bwd_cost=2 * fw)
    # one stage: no bubble except recompute time
    assert busy_t[0] == r.makespan and r.occupancy_bubble == 0.0


def test_stage_ops_cover_every_chunk():
    plan = cf.Plan.build([300, 40, 5000, 900, 77], 1024, 2)
    ch = plan.export()[0]
    ops, _, _, r = capi.pp_simulate(plan, 4, 2)
    for s in range(4):
        f = ops[s][ops[s]["kind"] == capi.PP_FORWARD]["chunk_id"]
        b = ops[s][ops[s]["kind"] == capi.PP_BACKWARD]["chunk_id"]
        assert sorted(f.tolist()) == sorted(ch["chunk_id"].tolist()) == sorted(b.tolist())
        assert f.tolist() == ch["chunk_id"].tolist()  # forwards in plan order


def test_validation_errors():
    plan = cf.Plan.build([1, 1, 2, 4], 2, 1)
    with pytest.raises(capi.CfError):
        capi.pp_simulate(plan, 0, 1)
    with pytest.raises(capi.CfError):
        capi.pp_simulate(plan, 2, 0)
    with pytest.raises(capi.CfError):
        capi.pp_simulate(plan, 2, 1, cost={"alpha": -1.0})
    with pytest.raises(capi.CfError):
        capi.pp_simulate(plan, 2, 1, cost={"backward_multiplier": 0.0})
    assert capi.pp_stage_layers(64, 3, 4) == (48, 64)
    assert capi.pp_stage_layers(2, 1, 2) == (1, 2)
    with pytest.raises(capi.CfError):
        capi.pp_stage_layers(2, 0, 3)


@pytest.mark.parametrize("chrome", [True, False])
def test_export_trace_matches_reference(reference, oracle, chrome):
    """export_trace (pipeline.hpp:353-396): table text byte-identical; chrome-
    trace documents equal value for value (floats compared exactly — the
    product prints the shortest round-trip digits, nlohmann's Grisu2 now and
    then a 17th digit of the same double)."""
    lengths, _ = c1_batch(oracle)

    def same(mine, ref):
        if chrome:
            assert json.loads(mine) == json.loads(ref)
        else:
            assert mine == ref

    cases = [([1, 1, 2, 4], 2, 1, 4, (0.0, 1.0, 0.0, 2.0, 0.0)), ([1, 1, 2, 4], 2, 2, 3, (0.25, 1.0, 0.1, 1.5, 0.5)),
             (lengths, 512, 2, 4, (0.0, 1.0, 1.05e-5, 2.0, 3.0))]
    for lens, cs, k, stages, cost in cases:
        c = dict(zip(("gamma", "alpha", "beta", "backward_multiplier", "hop_latency"), cost))
        ops, _, _, _ = capi.pp_simulate(cf.Plan.build(lens, cs, k), stages, k, c)
        same(capi.pp_export_trace(ops, chrome), reference.export_trace(lens, cs, k, stages, cost, 1, chrome))
    ops, _, _, _ = capi.pp_simulate_1f1b([1, 1, 2, 4], 4)
    assert capi.pp_export_trace(ops, chrome) == reference.export_trace([1, 1, 2, 4], 1, 1, 4, mode=0, chrome=chrome)
    for lens, cs, k, stages, cost in cases[:2]:  # integral / short decimals: bytes equal too
        c = dict(zip(("gamma", "alpha", "beta", "backward_multiplier", "hop_latency"), cost))
        ops2, _, _, _ = capi.pp_simulate(cf.Plan.build(lens, cs, k), stages, k, c)
        assert capi.pp_export_trace(ops2, chrome) == reference.export_trace(lens, cs, k, stages, cost, 1, chrome)
    if chrome:
        doc = json.loads(capi.pp_export_trace(ops, True))
        assert doc["traceEvents"][0] == {"dur": 1000, "name": "F chunk0", "ph": "X", "pid": 0, "tid": 0, "ts": 0}
        assert capi.pp_export_trace(np.zeros((0, 0), capi.PP_OP_DT), True) == '{\n  "traceEvents": []\n}\n'


def _tune_both(reference, lengths, css, ks, stages, cost, mem, budget, gbs, nb, seed):
    c = dict(zip(("gamma", "alpha", "beta", "backward_multiplier", "hop_latency"), cost))
    out = []
    for text in ("csv", "report"):
        table, bc, bk, ev, txt = capi.tune_grid_search(lengths, css, ks, stages, c, mem, budget, gbs, nb, seed,
                                                       text=text)
        assert txt == reference.tune(lengths, css, ks, stages, cost, mem, budget, gbs, nb, seed, csv=text == "csv")
        out.append((table, bc, bk, ev))
    return out[0]


def test_tuner_worked_batch(reference):
    """test_tuner.cpp: worked batch, 4 stages, budget grid {2,4} x {1,2}: best (2, 2); 54 / 46 / 60 / 60."""
    table, bc, bk, ev = _tune_both(reference, [1, 1, 2, 4], [2, 4], [1, 2], 4, (0.0, 1.0, 0.0, 2.0, 0.0),
                                   (0.0, 0.0, 0.0, 1.0), 1e9, 4, 1, 1)
    assert (bc, bk, ev) == (2, 2, 4)
    assert table["mean_time"].tolist() == [54.0, 46.0, 60.0, 60.0]
    # single stage forces k = 1; memory budget 5 with peak = k * cs
    table, bc, bk, ev = _tune_both(reference, [3, 5, 2, 7, 4, 6], [2, 4, 8], [1, 2, 4], 1,
                                   (1.0, 1.0, 0.0, 2.0, 0.0), (0.0, 1.0, 0.0, 1.0), 5.0, 6, 1, 1)
    assert (bc, bk) == (4, 1) and not table[(table["chunk_size"] == 8) & (table["k"] == 1)]["feasible"][0]
    # nothing feasible
    _, bc, bk, _ = _tune_both(reference, [1, 1, 2, 4], [2, 4], [1, 2], 4, (0.0, 1.0, 0.0, 2.0, 0.0),
                              (10.0, 0.0, 0.0, 1.0), 1.0, 4, 1, 1)
    assert (bc, bk) == (-1, -1)


def test_tuner_random_and_c1(reference, oracle):
    lengths, _ = c1_batch(oracle)
    _tune_both(reference, lengths, [256, 512, 1024], [1, 2, 4], 4, (0.5, 1.0, 1.05e-5, 2.0, 1.0),
               (34.87, 2.9e-3, 1.7e-5, 0.25), 60.0, 16, 3, 5)
    rng = np.random.default_rng(17)
    for _ in range(15):
        n = int(rng.integers(1, 60))
        lens = rng.integers(1, 3000, n)
        css = sorted(set(int(x) for x in rng.integers(16, 2048, int(rng.integers(1, 4)))))
        ks = sorted(set(int(x) for x in rng.integers(1, 5, int(rng.integers(1, 3)))))
        _tune_both(reference, lens, css, ks, int(rng.integers(1, 6)),
                   (float(rng.random()), 1.0, float(rng.random()) * 1e-4, 2.0, float(rng.random())),
                   (float(rng.random()) * 40, 1e-3, 1e-5, 1.0), float(rng.random()) * 60 + 1,
                   int(rng.integers(1, n + 3)), int(rng.integers(1, 5)), int(rng.integers(0, 100)))


def test_tuner_validation():
    for kw in (dict(chunk_sizes=[]), dict(budget_gib=0.0), dict(batches_to_sample=0)):
        args = dict(lengths=[1, 2, 3], chunk_sizes=[2], ks=[1], stages=2)
        args.update(kw)
        with pytest.raises(capi.CfError):
            capi.tune_grid_search(**args)


def test_stage_memory_replay_budget_bounds():
    """cf_pp_stage_memory replays each stage's 1F1B op stream with the
    executor's tape rules: without a budget stage s of an all-standalone plan
    holds min(P - s, M) tapes at its warm-up peak; with a budget B no stage
    holds more than B, and the first-stage checkpoints keep no input."""
    lengths = np.array([500, 480, 470, 450, 430, 400, 900, 1500, 40, 30], np.int64)
    plan = cf.Plan.build(lengths, 512, 1)
    free = capi.pp_stage_memory(plan, 4, 1, 0)
    assert list(free["peak_tapes"]) == [4, 3, 2, 1] and free["checkpointed"].sum() == 0
    assert free["peak_kept_tokens"][0] == 0
    for b in (1, 2, 3):
        m = capi.pp_stage_memory(plan, 4, 1, b)
        assert (m["peak_tapes"] <= b).all() and m["peak_tapes"].max() == b
        assert (m["peak_tape_tokens"] <= free["peak_tape_tokens"]).all()
        assert m["checkpointed"][0] > 0 and m["peak_kept_tokens"][0] == 0
    # randomized: the bound holds for every plan, stage count and budget
    rng = np.random.default_rng(9)
    for _ in range(100):
        L = rng.integers(1, 400, size=int(rng.integers(1, 15))).astype(np.int64)
        cs, k, P, b = int(rng.integers(16, 256)), int(rng.integers(1, 4)), int(rng.integers(1, 6)), int(rng.integers(0, 4))
        m = capi.pp_stage_memory(cf.Plan.build(L, cs, k), P, k, b)
        if b:
            assert (m["peak_tapes"] <= b).all()
        assert (m["peak_tape_tokens"] <= m["peak_tapes"] * cs).all()


def test_tuner_pp_counts_in_flight_chunks():
    """grid_search_pp: one stage with no budget predicts at least the
    reference tuner's peak; four stages without a budget predict more (the
    1F1B warm-up holds 4 chunks on stage 0) and a tape budget brings the
    prediction back under the memory budget at the price of recompute time."""
    lengths = capi.synthesize(300, 5, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)
    lengths = np.concatenate([lengths, [9000, 12000]]).astype(np.int64)
    mem = (40.0, 0.004, 1e-4, 1.0)
    cost = {"alpha": 1.0, "beta": 1e-4}
    ref, _, _, _, _ = capi.tune_grid_search(lengths, [2048, 4096], [1, 2], 4, cost, mem, 1e9, 150, 2, 3)
    free, _, _, _, _ = capi.tune_grid_search_pp(lengths, [2048, 4096], [1, 2], 4, cost, mem, 0.0, 0, 1e9, 150, 2, 3)
    assert (free["predicted_peak_gib"] > ref["predicted_peak_gib"]).all()
    b2, _, _, _, _ = capi.tune_grid_search_pp(lengths, [2048, 4096], [1, 2], 4, cost, mem, 1e-5, 2, 1e9, 150, 2, 3)
    assert (b2["predicted_peak_gib"] < free["predicted_peak_gib"]).all()
    assert (b2["mean_time"] >= free["mean_time"]).all()
    # the reference timing when nothing is checkpointed: identical makespans
    one, _, _, _, _ = capi.tune_grid_search_pp(lengths, [2048], [1], 4, cost, mem, 0.0, 0, 1e9, 150, 2, 3)
    assert one["mean_time"][0] == ref["mean_time"][0]
