"""Product planning (C++ in libchunkflow_b200.so, through the C-ABI) is
bit-exact with the reference chunker/scheduler: golden fixtures, the oracle
on >10^3 random batches, and the full C2/C4 batch layouts."""
import json
import os

import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from oracle.oracle import c1_batch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def _product(lengths, cs, k, ids=None):
    p = cf.Plan.build(lengths, cs, k, ids)
    ch, sg, ev, dg = p.export()
    return p, ch, sg, ev, dg


def _check_doc(doc):
    p, ch, sg, ev, dg = _product(doc["lengths"], doc["chunk_size"], doc["k"])
    assert ch.tolist() == [tuple(x) for x in doc["chunks"]]
    assert sg.tolist() == [tuple(x) for x in doc["segments"]]
    assert ev.tolist() == [tuple(x) for x in doc["events"]]
    assert [int(x) for x in dg.tolist()] == doc["diag"]
    assert p.listing() == doc["listing"]


@pytest.mark.parametrize("key", ["worked_cs2_k1", "worked_cs4_k1", "ffd_beaten_cs10", "c1_plan"])
def test_golden_plans(key):
    _check_doc(GOLD[key])


def test_golden_random_plans():
    for doc in GOLD["random"]:
        _check_doc(doc)


def test_listing_text_exact():
    """test_scheduler.cpp:243-257."""
    p = cf.Plan.build([1, 1, 2, 4], 2, 1)
    assert p.listing() == ("F+ chunk=0 group=-\nB  chunk=0 group=-\nF+ chunk=1 group=-\nB  chunk=1 group=-\n"
                           "F- chunk=2 group=0\nF+ chunk=3 group=0\nB  chunk=3 group=0\n"
                           "F+ chunk=2 group=0 recompute\nB  chunk=2 group=0\n")
    assert p.groups() == {0: [2, 3]}


def test_random_batches_bitwise_vs_oracle(oracle):
    rng = np.random.default_rng(123)
    for trial in range(1500):
        n = int(rng.integers(1, 40))
        cs = int(rng.integers(1, 100))
        k = int(rng.integers(1, 6))
        hi = int(rng.choice([20, 200, 600]))
        lengths = rng.integers(1, hi, n)
        ids = rng.permutation(5000)[:n] if trial % 3 == 0 else None
        _, ch, sg, ev, dg = _product(lengths, cs, k, ids)
        och, osg = oracle.construct_chunks(lengths, cs, ids)
        oev, odg = oracle.schedule_step(lengths, cs, k, ids)
        assert ch.tolist() == och.tolist(), (lengths.tolist(), cs)
        assert sg.tolist() == osg.tolist()
        assert ev.tolist() == oev.tolist()
        assert dg.tolist() == odg.tolist()


def test_c2_layout_matches_reference_summary():
    s = GOLD["c2_plan_summary"]
    _, ch, sg, ev, dg = _product(s["lengths"], s["chunk_size"], s["k"])
    assert len(ch) == s["n_chunks"] == 33 and len(ev) == s["n_events"] == 70
    assert [int(x) for x in dg.tolist()] == s["diag"] == [8192, 32768, 0]
    h = lambda a, c: int(np.bitwise_xor.reduce((a.view(np.int64) * 1000003 + c).ravel()))  # noqa: E731
    assert h(ch, 7) == s["chunk_hash"] and h(sg, 11) == s["segment_hash"] and h(ev, 13) == s["event_hash"]


def test_c4_eight_blocks_match_oracle(oracle):
    """8 x 1,000-sequence blocks (C4): 269 chunks, 570 events (SURVEY Appx A)."""
    lengths, ids = [], []
    for blk in range(8):
        blen = list(oracle.synthesize(999, blk + 1, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)) + [37888]
        lengths += blen
    lengths = np.array(lengths, np.int64)
    _, ch, sg, ev, dg = _product(lengths, 8192, 1)
    assert len(ch) == 269 and len(ev) == 570
    och, osg = oracle.construct_chunks(lengths, 8192)
    oev, odg = oracle.schedule_step(lengths, 8192, 1)
    assert ch.tolist() == och.tolist() and sg.tolist() == osg.tolist() and ev.tolist() == oev.tolist()


def test_c1_plan(oracle):
    lengths, _ = c1_batch(oracle)
    _, ch, sg, ev, dg = _product(lengths, 512, 2)
    assert len(ch) == 26 and len(ev) == 54


def test_validation_errors_map_to_status_codes():
    with pytest.raises(cf.capi.CfError) as e:
        cf.Plan.build([4, 5], 0, 1)
    assert e.value.code == 1  # CF_EVALIDATION (chunk_size must be at least 1)
    with pytest.raises(cf.capi.CfError) as e:
        cf.Plan.build([4, 5], 4, 0)
    assert e.value.code == 1
    with pytest.raises(cf.capi.CfError):
        cf.Plan.group(0, 1)


def test_empty_and_edge_batches(oracle):
    for lengths, cs in (([], 4), ([1], 1), ([1, 1, 1], 1), ([7], 7), ([8], 7), ([100000], 8192)):
        _, ch, sg, ev, dg = _product(np.array(lengths, np.int64), cs, 1)
        och, osg = oracle.construct_chunks(np.array(lengths, np.int64), cs)
        assert ch.tolist() == och.tolist() and sg.tolist() == osg.tolist()


def test_gen_tokens_matches_oracle(oracle):
    lengths = np.array([8, 8, 16, 32, 1000])
    for vocab, seed in ((32, 11), (256, 5), (32000, 1), (7, 3)):
        assert np.array_equal(cf.gen_tokens(lengths, vocab, seed), oracle.gen_tokens(lengths, vocab, seed))
