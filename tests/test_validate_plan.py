"""validate_plan over caller-built ExecutionPlans through the C-ABI
(cf_plan_validate_events) — the malformed-plan cases of the reference's
test_scheduler.cpp:165-240 — with the violation texts pinned verbatim
against the compiled reference (oracle/_ref, cfr_validate_events)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2503_02356_b200 as cf
from paper_2503_02356_b200.capi import EVENT_DT

HAVE_REF = os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libcfref.so"))


def _ref_validate(reference, events, chunk_size, k, groups, chunk_tokens):
    P = C.POINTER(C.c_int64)
    ev = np.ascontiguousarray(events, EVENT_DT)
    gid = np.array(sorted(groups) or [0], np.int64)
    off = np.zeros(len(groups) + 1, np.int64)
    mem = []
    for i, g in enumerate(sorted(groups)):
        mem += groups[g]
        off[i + 1] = len(mem)
    mem = np.array(mem or [0], np.int64)
    tc = np.array(list(chunk_tokens) or [0], np.int64)
    tn = np.array(list(chunk_tokens.values()) or [0], np.int64)
    peak, rec, n = C.c_int64(), C.c_int64(), C.c_size_t()
    buf = C.create_string_buffer(1 << 16)
    reference._check(reference.lib.cfr_validate_events(
        C.c_int64(chunk_size), C.c_int64(k), ev.ctypes.data_as(C.c_void_p), C.c_int64(len(ev)), gid.ctypes.data_as(P),
        off.ctypes.data_as(P), mem.ctypes.data_as(P), C.c_int64(len(groups)), tc.ctypes.data_as(P),
        tn.ctypes.data_as(P), C.c_int64(len(chunk_tokens)), C.byref(peak), C.byref(rec), buf, C.c_size_t(1 << 16),
        C.byref(n)))
    return peak.value, rec.value, [v for v in buf.value.decode().split("\n") if v]


def _check(reference, events, chunk_size, k=1, groups=None, chunk_tokens=None):
    groups, chunk_tokens = groups or {}, chunk_tokens or {}
    p = cf.Plan.validate_events(events, chunk_size, k, groups, chunk_tokens)
    dg = p.export()[3]
    got = (int(dg["peak_retained_tokens"]), int(dg["recompute_token_count"]), p.violations())
    if reference is not None:
        assert got == _ref_validate(reference, events, chunk_size, k, groups, chunk_tokens)
    return got


@pytest.fixture(scope="module")
def ref():
    if not HAVE_REF:
        return None
    from oracle.oracle import Reference
    return Reference()


def _group(n, k, cs=4):
    p = cf.Plan.group(n, k, cs)
    return p.export()[2], p.groups()


def test_flags_backward_without_retain_forward(ref):
    ev = np.zeros(1, EVENT_DT)
    ev[0]["kind"], ev[0]["chunk_id"], ev[0]["group_id"], ev[0]["index_in_group"] = 2, 0, -1, -1
    _, _, v = _check(ref, ev, 4)
    assert v and "without a live retain-forward" in v[0]


def test_flags_double_backward(ref):
    ev, groups = _group(1, 1)
    ev = np.concatenate([ev, ev[:1], ev[1:2]])  # re-retain, second backward
    _, _, v = _check(ref, ev, 4, 1, groups)
    assert any("more than once" in x for x in v)


def test_flags_group_order_violations(ref):
    ev, groups = _group(2, 2)
    asc = ev.copy()
    asc[[2, 3]] = asc[[3, 2]]  # backwards ascending instead of descending
    _, _, v = _check(ref, asc, 4, 2, groups)
    assert any("out of descending group order" in x for x in v)
    rev = ev.copy()
    rev[[0, 1]] = rev[[1, 0]]  # first-pass forwards out of ascending order
    _, _, v = _check(ref, rev, 4, 2, groups)
    assert any("out of ascending group order" in x for x in v)


def test_flags_missing_backward(ref):
    ev, groups = _group(1, 1)
    _, _, v = _check(ref, ev[:-1], 4, 1, groups)
    assert any("never backwarded" in x for x in v)


def test_k_bound_holds_on_random_batches(ref):
    """test_scheduler.cpp:224-239: schedule_step plans replayed through the
    caller-built-plan entry are violation-free, within k * chunk_size, and
    report the same diagnostics as the scheduler's own validation."""
    rng = np.random.default_rng(11)
    for _ in range(40):
        cs = int(2 + rng.integers(14))
        k = int(1 + rng.integers(4))
        lengths = (1 + rng.integers(70, size=int(1 + rng.integers(12)))).astype(np.int64)
        plan = cf.Plan.build(lengths, cs, k)
        ch, _, ev, dg = plan.export()
        tokens = {int(c["chunk_id"]): int(c["total_tokens"]) for c in ch}
        peak, rec, v = _check(ref, ev, cs, k, plan.groups(), tokens)
        assert v == [] and peak <= k * cs
        assert (peak, rec) == (int(dg["peak_retained_tokens"]), int(dg["recompute_token_count"]))


def test_listing_of_a_caller_plan():
    ev, groups = _group(2, 1, 2)
    p = cf.Plan.validate_events(ev, 2, 1, groups)
    assert p.listing() == cf.Plan.group(2, 1, 2).listing()


def test_bad_event_kind_is_a_validation_error():
    ev = np.zeros(1, EVENT_DT)
    ev[0]["kind"] = 7
    with pytest.raises(cf.capi.CfError) as e:
        cf.Plan.validate_events(ev, 4)
    assert e.value.code == 1
