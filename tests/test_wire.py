"""Wire formats and memory model (product C++ in libchunkflow_b200.so, host/
wire.cpp) against the reference compiled in place (oracle/_ref):

* chunk_plan.json / execution_plan.json text byte-identical to the reference's
  nlohmann dump (chunker.hpp:233-292, scheduler.hpp:300-328), and a plan read
  back from the reference's document schedules identically;
* dataset JSONL (dataset.hpp:112-176) parsed and re-written byte-identically,
  with the reference's error categories;
* calibrate / predict_peak / coefficients_to_json (memory_model.hpp) on the
  paper's Table 6 rows (test_memory_model.cpp:20-100) and random designs.
"""
import json

import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200 import capi
from oracle.oracle import c1_batch


def _upstream_dump(text):
    """The reference builds against nlohmann/json 3.11.3 (vendor/ is absent);
    the only copy in this image (cudnn_frontend's) carries a local patch that
    prints integer arrays on one line.  Upstream dump(2) — what the product
    emits — pretty-prints every array; Python's json.dumps with sorted keys
    and 2-space indent produces exactly that text for these documents."""
    return json.dumps(json.loads(text), indent=2, sort_keys=True, separators=(",", ": ")) + "\n"


def _batches():
    yield [1, 1, 2, 4], 2, 1
    yield [1, 1, 2, 4], 4, 2
    rng = np.random.default_rng(3)
    for _ in range(40):
        cs = int(rng.integers(4, 500))
        yield rng.integers(1, 3 * cs, int(rng.integers(1, 60))).tolist(), cs, int(rng.integers(1, 4))


def test_plan_json_bytes_match_reference(reference, oracle):
    cases = list(_batches())
    lengths, _ = c1_batch(oracle)
    cases.append((lengths.tolist(), 512, 2))
    for lengths, cs, k in cases:
        p = cf.Plan.build(lengths, cs, k)
        for mine, ref in ((p.chunk_json(), reference.plan_json(lengths, cs, k, 0)),
                          (p.exec_json(), reference.plan_json(lengths, cs, k, 1))):
            assert json.loads(mine) == json.loads(ref)  # same document
            assert mine == _upstream_dump(ref)          # upstream nlohmann dump(2) text


def test_schedule_from_reference_chunk_plan(reference):
    """`chunkflow pack` output fed to the B200 planner == `chunkflow schedule`."""
    for lengths, cs, k in _batches():
        doc = reference.plan_json(lengths, cs, k, 0)
        p = cf.Plan.from_chunk_json(doc, k)
        assert p.exec_json() == _upstream_dump(reference.schedule_json(doc, k))
        assert p.chunk_json() == _upstream_dump(doc)
        assert cf.Plan.from_chunk_json(_upstream_dump(doc), k).exec_json() == p.exec_json()
        # and it is the same plan the batch builds directly
        q = cf.Plan.build(lengths, cs, k)
        assert [x.tolist() for x in p.export()[:3]] == [x.tolist() for x in q.export()[:3]]


def test_malformed_chunk_plan_is_parse_error():
    for bad in ['{"chunks": []}', '{"chunk_size": 4, "chunks": [{"id": 0}]}', '{', '[1, 2']:
        with pytest.raises(capi.CfError) as e:
            cf.Plan.from_chunk_json(bad, 1)
        assert e.value.code == 6  # CF_EPARSE (chunkflow::ParseError)


def test_jsonl_roundtrip_matches_reference(reference):
    rng = np.random.default_rng(5)
    lines = []
    for i in range(30):
        n = int(rng.integers(1, 20))
        rec = {"length": n}
        if i % 3:
            rec["id"] = int(rng.integers(0, 10 ** 6)) * 31 + i
        if i % 2:
            rec["tokens"] = rng.integers(0, 50000, n).tolist()
        lines.append(json.dumps(rec, separators=(", ", ": ") if i % 4 == 0 else (",", ":")))
        if i % 7 == 0:
            lines.append("   ")
    text = "\n".join(lines) + "\n"
    ids, lengths, has, tok = capi.dataset_load_jsonl(text)
    assert len(ids) == 30
    per = [tok[o - n:o] if h else None for o, n, h in zip(np.cumsum(lengths * has), lengths, has)]
    assert all(p is None or len(p) == n for p, n in zip(per, lengths))
    out = "".join(capi.dataset_write_jsonl([i], [n], p) for i, n, p in zip(ids, lengths, per))
    assert out == reference.jsonl_roundtrip(text)


@pytest.mark.parametrize("bad,code", [
    ('{"length": 0}\n', 1), ('{"length": 3, "tokens": [1, 2]}\n', 1), ('{"id": 1, "length": 2}\n{"id": 1, "length": 3}\n', 1),
    ('{"length": "3"}\n', 6), ('[1]\n', 6), ('{"length": 3\n', 6), ('{"length": 2, "id": 1.5}\n', 6),
    ('{"length": 2, "tokens": 7}\n', 6)])
def test_jsonl_errors(reference, bad, code):
    with pytest.raises(capi.CfError) as e:
        capi.dataset_load_jsonl(bad)
    assert e.value.code == code
    with pytest.raises(ValueError) as r:
        reference.jsonl_roundtrip(bad)
    assert f"[{code}]" in str(r.value)


TABLE6 = "chunk_size,k,context_len,peak_gib\n" + "\n".join(
    f"{a},{b},{c},{d}" for a, b, c, d in [(2048, 1, 32768, 41.6), (2048, 1, 262144, 45.6), (4096, 1, 32768, 47.5),
                                          (4096, 1, 262144, 50.8), (8192, 1, 32768, 59.3), (8192, 1, 262144, 63.8)])


@pytest.mark.parametrize("gqa", [1.0, 0.25])
def test_memory_model_table6(reference, gqa):
    """test_memory_model.cpp:64-74: base 34.8717, 2.93666e-3, 1.71480e-5, resid 0.59524."""
    cs, k, ctx, pk = capi.mem_parse_csv(TABLE6)
    c, resid = capi.mem_calibrate(cs, k, ctx, pk, gqa)
    rc, rresid, rdoc = reference.calibrate(TABLE6, gqa)
    assert [c.base_gib, c.per_chunk_token_gib, c.per_context_token_gib, c.gqa_ratio] == rc.tolist()
    assert resid == rresid
    assert capi.mem_coeffs_json(c) == rdoc
    if gqa == 1.0:
        assert abs(c.base_gib - 34.8717) < 1e-3 and abs(c.per_chunk_token_gib - 2.93666e-3) < 1e-7
        assert abs(c.per_context_token_gib - 1.71480e-5) < 1e-9 and abs(resid - 0.59524) < 1e-4
    assert abs(capi.mem_predict(c, 2048, 1, 32768) - 41.6) < 1.0


def test_memory_model_random_designs(reference):
    rng = np.random.default_rng(9)
    for _ in range(50):
        n = int(rng.integers(3, 12))
        rows = [(int(rng.integers(1, 9)) * 1024, int(rng.integers(1, 5)), int(rng.integers(1, 300)) * 1024,
                 float(rng.random() * 100)) for _ in range(n)]
        csv = "\n".join(f"{a}, {b}, {c}, {d!r}" for a, b, c, d in rows)
        gqa = float(rng.choice([1.0, 0.25, 0.125]))
        try:
            rc, rresid, rdoc = reference.calibrate(csv, gqa)
        except ValueError:
            with pytest.raises(capi.CfError):
                capi.mem_calibrate(*capi.mem_parse_csv(csv), gqa)
            continue
        c, resid = capi.mem_calibrate(*capi.mem_parse_csv(csv), gqa)
        assert [c.base_gib, c.per_chunk_token_gib, c.per_context_token_gib, c.gqa_ratio] == rc.tolist()
        assert resid == rresid
        assert capi.mem_coeffs_json(c) == rdoc


def test_memory_model_degenerate():
    for rows in ([(2048, 1, 32768, 41.6), (4096, 1, 32768, 47.5)],
                 [(2048, 1, 32768, 41.6), (2048, 1, 262144, 45.6), (2048, 1, 65536, 42.0)]):
        with pytest.raises(capi.CfError) as e:
            capi.mem_calibrate(*zip(*rows))
        assert e.value.code == 1
    with pytest.raises(capi.CfError) as e:
        capi.mem_parse_csv("1,2,x,4\n")
    assert e.value.code == 6
