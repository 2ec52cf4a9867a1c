"""ctypes binding of libchunkflow_b200.so (include/chunkflow_b200.h).

The shared library is the product: every compute call below goes to the
sm_100a kernels inside it.  There is no fallback — if the library is missing
the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CF_LIB selects another build of the library (A/B kernel measurements)
LIB_PATH = os.environ.get("CF_LIB") or os.path.join(_HERE, "libchunkflow_b200.so")

CHUNK_DT = np.dtype([(k, np.int64) for k in
                     ("chunk_id", "kind", "group_id", "index_in_group",
                      "total_tokens", "seg_offset", "seg_count")])
SEG_DT = np.dtype([(k, np.int64) for k in ("sequence_id", "start_token", "length")])
EVENT_DT = np.dtype([(k, np.int64) for k in
                     ("kind", "chunk_id", "group_id", "index_in_group",
                      "is_recompute", "save_kv", "read_kv_prefix",
                      "accumulate_kv_grad")])
DIAG_DT = np.dtype([(k, np.int64) for k in
                    ("peak_retained_tokens", "recompute_token_count",
                     "num_violations")])

PP_OP_DT = np.dtype([("kind", np.int64), ("chunk_id", np.int64), ("start", np.float64), ("end", np.float64)])
PP_FORWARD, PP_RECOMPUTE, PP_BACKWARD = 0, 1, 2

ARCH_TOY, ARCH_LLAMA = 0, 1
EPI_BF16, EPI_F32, EPI_F32_ACC, EPI_F32_RES, EPI_BF16_TANH, EPI_BF16_TANHGRAD, EPI_BF16_SWIGLU = range(7)


class ModelCfg(C.Structure):
    _fields_ = [("arch", C.c_int32), ("reserved", C.c_int32),
                ("vocab_size", C.c_int64), ("d_model", C.c_int64),
                ("num_heads", C.c_int64), ("num_kv_heads", C.c_int64),
                ("num_layers", C.c_int64), ("ffn_width", C.c_int64),
                ("seed", C.c_uint64), ("rope_theta", C.c_double),
                ("rms_eps", C.c_double)]


class RunOpts(C.Structure):
    _fields_ = [("corrupt_kv_grads", C.c_int32), ("accumulate_grads", C.c_int32),
                ("normalizer_override", C.c_double), ("stage_tape_budget", C.c_int64), ("kv_offload", C.c_int32),
                ("reserved2", C.c_int32)]


class PpCost(C.Structure):
    _fields_ = [("gamma", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("backward_multiplier", C.c_double), ("hop_latency", C.c_double)]


class PpResult(C.Structure):
    _fields_ = [("makespan", C.c_double), ("bubble_ratio", C.c_double),
                ("occupancy_bubble", C.c_double), ("ops_per_stage", C.c_int64)]


class MemCoeffs(C.Structure):
    _fields_ = [("base_gib", C.c_double), ("per_chunk_token_gib", C.c_double),
                ("per_context_token_gib", C.c_double), ("gqa_ratio", C.c_double)]


class AdamWCfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("max_grad_norm", C.c_double), ("decay_gains", C.c_int32),
                ("reserved", C.c_int32)]


class RunResult(C.Structure):
    _fields_ = [("loss", C.c_double), ("peak_retained_tokens", C.c_int64),
                ("recompute_forward_count", C.c_int64),
                ("recompute_loss_mismatches", C.c_int64),
                ("kv_completeness_violations", C.c_int64), ("tokens", C.c_int64),
                ("gpu_launches", C.c_int64), ("peak_hbm_bytes", C.c_int64),
                ("static_hbm_bytes", C.c_int64), ("act_hbm_bytes", C.c_int64),
                ("kv_hbm_bytes", C.c_int64), ("model_flops", C.c_double),
                ("hw_flops", C.c_double), ("gemm_ms", C.c_double), ("gemm_flops", C.c_double),
                ("gemm_launches", C.c_int64), ("attn_ms", C.c_double), ("attn_flops", C.c_double),
                ("attn_launches", C.c_int64), ("attn_bwd_ms", C.c_double), ("attn_bwd_flops", C.c_double),
                ("attn_bwd_launches", C.c_int64), ("other_launches", C.c_int64),
                ("peak_live_tapes", C.c_int64), ("checkpoint_recomputes", C.c_int64),
                ("attn_dep_ms", C.c_double), ("attn_dep_flops", C.c_double),
                ("attn_bwd_dep_ms", C.c_double), ("attn_bwd_dep_flops", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


# Every symbol include/chunkflow_b200.h declares (checked by the CPU tests).
EXPORTS = [
    "cf_last_error", "cf_version", "cf_plan_build", "cf_plan_build_group",
    "cf_plan_counts", "cf_plan_export", "cf_plan_export_groups",
    "cf_plan_violation", "cf_plan_listing", "cf_plan_partition",
    "cf_plan_rank_tokens", "cf_plan_destroy", "cf_pp_simulate", "cf_pp_simulate_1f1b", "cf_pp_stage_layers", "cf_gen_tokens", "cf_synthesize", "cf_sample_batch",
    "cf_ctx_create",
    "cf_ctx_destroy", "cf_ctx_stream", "cf_ctx_set_profiling", "cf_nccl_unique_id", "cf_ctx_init_dp",
    "cf_model_create", "cf_model_destroy", "cf_model_num_tensors",
    "cf_model_tensor_info", "cf_model_get_param", "cf_model_set_param",
    "cf_model_get_grad", "cf_model_zero_grads", "cf_model_grad_buffer",
    "cf_model_num_params", "cf_run_plan", "cf_step_prepare", "cf_step_run",
    "cf_step_destroy", "cf_backward_full", "cf_model_create_stage", "cf_ctx_init_pp", "cf_pp_step_run",
    "cf_pp_run_local", "cf_step_op_times", "cf_step_input_bytes", "cf_pp_local_create", "cf_pp_local_destroy", "cf_ctx_init_pp_local", "cf_plan_chunk_json", "cf_plan_exec_json", "cf_plan_from_chunk_json",
    "cf_dataset_load_jsonl", "cf_dataset_write_jsonl", "cf_mem_calibrate", "cf_mem_predict", "cf_mem_parse_csv",
    "cf_mem_coeffs_json", "cf_pp_export_trace", "cf_tune_grid_search", "cf_ctx_synchronize", "cf_op_gemm", "cf_op_attention", "cf_debug_set_gemm_mode", "cf_debug_set_attn_stress",
    "cf_segment_forward", "cf_segment_backward", "cf_segment_destroy", "cf_op_gemm_rope",
    "cf_plan_validate_events", "cf_op_lm_head_ce", "cf_pp_stage_memory", "cf_tune_grid_search_pp",
    "cf_pp_simulate_budget", "cf_model_adamw_init", "cf_model_adamw_step", "cf_model_get_master",
]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.cf_last_error.restype = C.c_char_p
        L.cf_version.restype = C.c_char_p
        L.cf_ctx_stream.restype = C.c_void_p
        L.cf_model_num_tensors.restype = C.c_int64
        L.cf_model_num_params.restype = C.c_int64
        vp = C.c_void_p
        for name in ("cf_plan_destroy", "cf_ctx_destroy", "cf_model_destroy", "cf_step_destroy",
                     "cf_pp_local_destroy", "cf_segment_destroy"):
            getattr(L, name).argtypes = [vp]
            getattr(L, name).restype = None
        L.cf_model_num_tensors.argtypes = [vp]
        L.cf_model_num_params.argtypes = [vp]
        L.cf_ctx_stream.argtypes = [vp]
        L.cf_op_gemm.argtypes = [vp, vp, C.c_int, C.c_int64, vp, C.c_int, C.c_int64, vp, C.c_int64,
                                 C.c_int64, C.c_int64, C.c_int64, C.c_int, vp, C.c_int64]
        L.cf_op_lm_head_ce.argtypes = [vp, vp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, vp, C.c_float, vp,
                                       vp, vp]
        _lib = L
    return _lib


class CfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[cf {code}] {msg}")
        self.code = code


def check(rc):
    if rc != 0:
        raise CfError(rc, lib().cf_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Plan:
    """A chunk plan + execution schedule (construct_chunks + schedule_step)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    @classmethod
    def build(cls, lengths, chunk_size, k, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        h = C.c_void_p()
        check(lib().cf_plan_build(_p(ids), _p(lengths), C.c_int64(len(lengths)),
                                  C.c_int64(chunk_size), C.c_int64(k), C.byref(h)))
        return cls(h)

    @classmethod
    def group(cls, n, k, chunk_size=1):
        h = C.c_void_p()
        check(lib().cf_plan_build_group(C.c_int64(n), C.c_int64(k), C.c_int64(chunk_size), C.byref(h)))
        return cls(h)

    def counts(self):
        v = [C.c_int64() for _ in range(4)]
        check(lib().cf_plan_counts(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def export(self):
        nc, ns, ne, ng = self.counts()
        ch = np.zeros(nc, CHUNK_DT)
        sg = np.zeros(ns, SEG_DT)
        ev = np.zeros(ne, EVENT_DT)
        dg = np.zeros(1, DIAG_DT)
        check(lib().cf_plan_export(self.h, _p(ch), _p(sg), _p(ev), _p(dg)))
        return ch, sg, ev, dg[0]

    def groups(self):
        nc, ns, ne, ng = self.counts()
        gid = np.zeros(max(ng, 1), np.int64)
        off = np.zeros(ng + 1, np.int64)
        check(lib().cf_plan_export_groups(self.h, None, _p(off), None))
        mem = np.zeros(max(int(off[-1]), 1), np.int64)
        check(lib().cf_plan_export_groups(self.h, _p(gid), _p(off), _p(mem)))
        return {int(gid[i]): [int(x) for x in mem[off[i]:off[i + 1]]] for i in range(ng)}

    def violations(self):
        n = int(self.export()[3]["num_violations"])
        out = []
        for i in range(n):
            buf = C.create_string_buffer(256)
            check(lib().cf_plan_violation(self.h, C.c_int64(i), buf, C.c_size_t(256)))
            out.append(buf.value.decode())
        return out

    def listing(self):
        n = C.c_size_t()
        check(lib().cf_plan_listing(self.h, None, C.c_size_t(0), C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().cf_plan_listing(self.h, buf, C.c_size_t(n.value + 1), None))
        return buf.value.decode()

    def chunk_json(self) -> str:
        """chunk_plan.json text of `chunkflow pack` (chunker.hpp:233)."""
        return _text(lambda buf, cap, n: lib().cf_plan_chunk_json(self.h, buf, cap, n))

    def exec_json(self) -> str:
        """execution_plan.json text of `chunkflow schedule` (scheduler.hpp:300)."""
        return _text(lambda buf, cap, n: lib().cf_plan_exec_json(self.h, buf, cap, n))

    @classmethod
    def from_chunk_json(cls, text: str, k: int):
        """chunk_plan_from_json + schedule_step (chunker.hpp:261)."""
        h = C.c_void_p()
        check(lib().cf_plan_from_chunk_json(text.encode(), C.c_int64(k), C.byref(h)))
        return cls(h)

    @classmethod
    def validate_events(cls, events, chunk_size, k=1, groups=None, chunk_tokens=None, chunk_plan=None):
        """validate_plan (scheduler.hpp:182) over a caller-built ExecutionPlan:
        `events` an EVENT_DT array, `groups` {group: [chunk ids in index order]},
        `chunk_tokens` {chunk: tokens}.  Diagnostics via export()[3] /
        violations() / listing().  With `chunk_plan` (a Plan.build result) the
        returned plan carries its chunks and can be run."""
        ev = np.ascontiguousarray(events, EVENT_DT)
        groups = groups or {}
        gid = np.array(sorted(groups), np.int64)
        off = np.zeros(len(gid) + 1, np.int64)
        mem = []
        for i, g in enumerate(gid):
            mem += list(groups[int(g)])
            off[i + 1] = len(mem)
        mem = np.array(mem or [0], np.int64)
        chunk_tokens = chunk_tokens or {}
        tc = np.array(list(chunk_tokens.keys()) or [0], np.int64)
        tn = np.array(list(chunk_tokens.values()) or [0], np.int64)
        h = C.c_void_p()
        check(lib().cf_plan_validate_events(C.c_int64(chunk_size), C.c_int64(k), _p(ev), C.c_int64(len(ev)),
                                            _p(gid if len(gid) else np.zeros(1, np.int64)), _p(off), _p(mem),
                                            C.c_int64(len(gid)), _p(tc), _p(tn), C.c_int64(len(chunk_tokens)),
                                            chunk_plan.h if chunk_plan is not None else None, C.byref(h)))
        return cls(h)

    def partition(self, world, rank):
        h = C.c_void_p()
        check(lib().cf_plan_partition(self.h, C.c_int64(world), C.c_int64(rank), C.byref(h)))
        return Plan(h)

    def rank_tokens(self, world):
        out = np.zeros(world, np.int64)
        check(lib().cf_plan_rank_tokens(self.h, C.c_int64(world), _p(out)))
        return out

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.cf_plan_destroy(self.h)
            self.h = C.c_void_p()


def _pp_cost(cost):
    if isinstance(cost, PpCost):
        return cost
    c = dict(gamma=0.0, alpha=1.0, beta=0.0, backward_multiplier=2.0, hop_latency=0.0)
    c.update(cost or {})
    return PpCost(**c)


def pp_simulate(plan: "Plan", stages, k, cost=None, backward_first=True, fwd_cost=None, bwd_cost=None,
                tape_budget=0):
    """simulate_state_aware_1f1b + bubble_ratio (pipeline.hpp:250-331);
    tape_budget > 0 times the executor's stage-input checkpointing
    (cf_pp_simulate_budget).  Returns (ops[stages, per] of PP_OP_DT, busy,
    busy_total, PpResult)."""
    c = _pp_cost(cost)
    r = PpResult()
    fw = None if fwd_cost is None else np.ascontiguousarray(fwd_cost, np.float64)
    bw = None if bwd_cost is None else np.ascontiguousarray(bwd_cost, np.float64)
    args = (plan.h, C.c_int64(stages), C.c_int64(k), C.byref(c), C.c_int(int(backward_first)),
            None if fw is None else _p(fw), None if bw is None else _p(bw))
    if tape_budget:
        args = args + (C.c_int64(tape_budget),)
        fn = lib().cf_pp_simulate_budget
    else:
        fn = lib().cf_pp_simulate
    check(fn(*args, None, None, None, C.byref(r)))
    ops = np.zeros((stages, r.ops_per_stage), PP_OP_DT)
    busy = np.zeros(stages, np.float64)
    busy_t = np.zeros(stages, np.float64)
    check(fn(*args, _p(ops), _p(busy), _p(busy_t), C.byref(r)))
    return ops, busy, busy_t, r


def pp_simulate_1f1b(lengths, stages, cost=None):
    """simulate_1f1b + bubble_ratio (pipeline.hpp:218-242, 325-331)."""
    lengths = np.ascontiguousarray(lengths, np.int64)
    c = _pp_cost(cost)
    r = PpResult()
    ops = np.zeros((stages, 2 * len(lengths)), PP_OP_DT)
    busy = np.zeros(stages, np.float64)
    busy_t = np.zeros(stages, np.float64)
    check(lib().cf_pp_simulate_1f1b(_p(lengths), C.c_int64(len(lengths)), C.c_int64(stages), C.byref(c),
                                    _p(ops), _p(busy), _p(busy_t), C.byref(r)))
    return ops, busy, busy_t, r


def pp_export_trace(ops, chrome=True) -> str:
    """export_trace (pipeline.hpp:353-396) of ops[stages, per] (PP_OP_DT)."""
    ops = np.ascontiguousarray(ops, PP_OP_DT)
    st, per = ops.shape
    return _text(lambda buf, cap, n: lib().cf_pp_export_trace(_p(ops), C.c_int64(st), C.c_int64(per),
                                                              C.c_int(0 if chrome else 1), buf, cap, n))


TUNE_ROW_DT = np.dtype([("chunk_size", np.int64), ("k", np.int64), ("mean_time", np.float64),
                        ("predicted_peak_gib", np.float64), ("feasible", np.int64)])


def tune_grid_search(lengths, chunk_sizes, ks, stages, cost=None, mem=None, budget_gib=80.0, global_batch_size=256,
                     batches_to_sample=4, seed=0, ids=None, text="report"):
    """grid_search (tuner.hpp:39): returns (table, best_cs, best_k, evaluations, text);
    text = "report" (tuner_report) or "csv" (tuner_table_csv)."""
    lengths = np.ascontiguousarray(lengths, np.int64)
    ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
    css = np.ascontiguousarray(chunk_sizes, np.int64)
    kk = np.ascontiguousarray(ks, np.int64)
    c = _pp_cost(cost)
    m = mem if isinstance(mem, MemCoeffs) else MemCoeffs(*(mem or (0.0, 0.0, 0.0, 1.0)))
    table = np.zeros(len(css) * len(kk), TUNE_ROW_DT)
    bc, bk, ev = C.c_int64(), C.c_int64(), C.c_int64()

    def call(buf, cap, n):
        return lib().cf_tune_grid_search(_p(ids), _p(lengths), C.c_int64(len(lengths)), _p(css), C.c_int64(len(css)),
                                         _p(kk), C.c_int64(len(kk)), C.c_int64(stages), C.byref(c), C.byref(m),
                                         C.c_double(budget_gib), C.c_int64(global_batch_size),
                                         C.c_int64(batches_to_sample), C.c_uint64(seed), _p(table), C.byref(bc),
                                         C.byref(bk), C.byref(ev), C.c_int(int(text == "csv")), buf, cap, n)
    txt = _text(call)
    return table, bc.value, bk.value, ev.value, txt


def tune_grid_search_pp(lengths, chunk_sizes, ks, stages, cost=None, mem=None, kept_token_gib=0.0, tape_budget=0,
                        budget_gib=80.0, global_batch_size=256, batches_to_sample=4, seed=0, ids=None,
                        text="report"):
    """Pipeline-aware grid_search (cf_tune_grid_search_pp): per-stage in-flight
    tapes under `tape_budget` decide feasibility.  Returns as tune_grid_search."""
    lengths = np.ascontiguousarray(lengths, np.int64)
    ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
    css = np.ascontiguousarray(chunk_sizes, np.int64)
    kk = np.ascontiguousarray(ks, np.int64)
    c = _pp_cost(cost)
    m = mem if isinstance(mem, MemCoeffs) else MemCoeffs(*(mem or (0.0, 0.0, 0.0, 1.0)))
    table = np.zeros(len(css) * len(kk), TUNE_ROW_DT)
    bc, bk, ev = C.c_int64(), C.c_int64(), C.c_int64()

    def call(buf, cap, n):
        return lib().cf_tune_grid_search_pp(
            _p(ids), _p(lengths), C.c_int64(len(lengths)), _p(css), C.c_int64(len(css)), _p(kk), C.c_int64(len(kk)),
            C.c_int64(stages), C.byref(c), C.byref(m), C.c_double(kept_token_gib), C.c_int64(tape_budget),
            C.c_double(budget_gib), C.c_int64(global_batch_size), C.c_int64(batches_to_sample), C.c_uint64(seed),
            _p(table), C.byref(bc), C.byref(bk), C.byref(ev), C.c_int(int(text == "csv")), buf, cap, n)
    txt = _text(call)
    return table, bc.value, bk.value, ev.value, txt


def pp_stage_memory(plan: "Plan", stages, k, tape_budget=0):
    """cf_pp_stage_memory: per-stage dict of peak tapes / tape tokens / kept
    input tokens / checkpointed forwards."""
    out = {f: np.zeros(stages, np.int64) for f in ("peak_tapes", "peak_tape_tokens", "peak_kept_tokens",
                                                  "checkpointed")}
    check(lib().cf_pp_stage_memory(plan.h, C.c_int64(stages), C.c_int64(k), C.c_int64(tape_budget),
                                   _p(out["peak_tapes"]), _p(out["peak_tape_tokens"]), _p(out["peak_kept_tokens"]),
                                   _p(out["checkpointed"])))
    return out


def pp_stage_layers(layers, stage, stages):
    b, e = C.c_int64(), C.c_int64()
    check(lib().cf_pp_stage_layers(C.c_int64(layers), C.c_int64(stage), C.c_int64(stages), C.byref(b), C.byref(e)))
    return b.value, e.value


def _text(call):
    n = C.c_size_t()
    check(call(None, C.c_size_t(0), C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(call(buf, C.c_size_t(n.value + 1), C.byref(n)))
    return buf.raw[:n.value].decode()


def dataset_load_jsonl(text: str):
    """load_lengths (dataset.hpp:112) -> (ids, lengths, has_tokens, tokens)."""
    raw = text.encode()
    n, nt = C.c_int64(), C.c_int64()
    check(lib().cf_dataset_load_jsonl(raw, C.byref(n), None, None, None, C.byref(nt), None))
    ids = np.zeros(n.value, np.int64)
    lengths = np.zeros(n.value, np.int64)
    has = np.zeros(n.value, np.int64)
    tok = np.zeros(max(1, nt.value), np.int32)
    check(lib().cf_dataset_load_jsonl(raw, C.byref(n), _p(ids), _p(lengths), _p(has), C.byref(nt), _p(tok)))
    return ids, lengths, has.astype(bool), tok[:nt.value]


def dataset_write_jsonl(ids, lengths, tokens=None) -> str:
    """write_records (dataset.hpp:169)."""
    ids = np.ascontiguousarray(ids, np.int64)
    lengths = np.ascontiguousarray(lengths, np.int64)
    tok = None if tokens is None else np.ascontiguousarray(tokens, np.int32)
    return _text(lambda buf, cap, n: lib().cf_dataset_write_jsonl(
        _p(ids), _p(lengths), None if tok is None else _p(tok), C.c_int64(len(ids)), buf, cap, n))


def mem_calibrate(chunk_size, k, context_len, peak_gib, gqa_ratio=1.0):
    """calibrate (memory_model.hpp:59) -> (MemCoeffs, max_residual_gib)."""
    cs = np.ascontiguousarray(chunk_size, np.int64)
    kk = np.ascontiguousarray(k, np.int64)
    ctx = np.ascontiguousarray(context_len, np.int64)
    pk = np.ascontiguousarray(peak_gib, np.float64)
    out, res = MemCoeffs(), C.c_double()
    check(lib().cf_mem_calibrate(_p(cs), _p(kk), _p(ctx), _p(pk), C.c_int64(len(cs)), C.c_double(gqa_ratio),
                                 C.byref(out), C.byref(res)))
    return out, res.value


def mem_predict(coeffs: MemCoeffs, chunk_size, k, context_len):
    out = C.c_double()
    check(lib().cf_mem_predict(C.byref(coeffs), C.c_int64(chunk_size), C.c_int64(k), C.c_int64(context_len),
                               C.byref(out)))
    return out.value


def mem_parse_csv(text: str):
    raw = text.encode()
    n = C.c_int64()
    check(lib().cf_mem_parse_csv(raw, C.byref(n), None, None, None, None))
    cs, kk, ctx = (np.zeros(n.value, np.int64) for _ in range(3))
    pk = np.zeros(n.value, np.float64)
    check(lib().cf_mem_parse_csv(raw, C.byref(n), _p(cs), _p(kk), _p(ctx), _p(pk)))
    return cs, kk, ctx, pk


def mem_coeffs_json(coeffs: MemCoeffs) -> str:
    return _text(lambda buf, cap, n: lib().cf_mem_coeffs_json(C.byref(coeffs), buf, cap, n))


def synthesize(count, seed, preset=1, bounds=(), fracs=(), max_length=0):
    b = np.ascontiguousarray(bounds, np.int64)
    f = np.ascontiguousarray(fracs, np.float64)
    out = np.zeros(count, np.int64)
    check(lib().cf_synthesize(_p(b), _p(f), C.c_int64(len(b)), C.c_int64(max_length), C.c_int64(preset),
                              C.c_int64(count), C.c_uint64(seed), _p(out)))
    return out


def sample_batch(n, global_batch, step, seed):
    out = np.zeros(global_batch, np.int64)
    cnt = C.c_int64()
    check(lib().cf_sample_batch(C.c_int64(n), C.c_int64(global_batch), C.c_int64(step), C.c_uint64(seed),
                                _p(out), C.byref(cnt)))
    return out[:cnt.value]


def gen_tokens(lengths, vocab, seed):
    lengths = np.ascontiguousarray(lengths, np.int64)
    out = np.zeros(int(lengths.sum()), np.int32)
    check(lib().cf_gen_tokens(_p(lengths), C.c_int64(len(lengths)), C.c_int64(vocab),
                              C.c_uint64(seed), _p(out)))
    return out


class Context:
    """One device context (stream + memory pool) on one GPU."""

    def __init__(self, device=0):
        self.h = C.c_void_p()
        check(lib().cf_ctx_create(C.c_int(device), C.byref(self.h)))

    @property
    def stream(self):
        return lib().cf_ctx_stream(self.h)

    def synchronize(self):
        check(lib().cf_ctx_synchronize(self.h))

    def set_profiling(self, on: bool):
        check(lib().cf_ctx_set_profiling(self.h, C.c_int(int(on))))

    def lm_head_ce(self, x, head, ldh, T, V, d, targets, inv_norm, lse, row_loss, dlogits=0):
        """cf_op_lm_head_ce on device pointers (ints)."""
        check(lib().cf_op_lm_head_ce(self.h, x, head, ldh, T, V, d, targets, inv_norm, lse, row_loss,
                                     dlogits or None))

    def init_dp(self, rank, world, uid: bytes | None):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid) if uid else None
        check(lib().cf_ctx_init_dp(self.h, C.c_int(rank), C.c_int(world), buf))

    def init_pp_local(self, pipe: "LocalPipe", stage):
        """Attach to an in-process pipeline (cf_ctx_init_pp_local)."""
        check(lib().cf_ctx_init_pp_local(self.h, pipe.h, C.c_int(stage)))

    def init_pp(self, rank, world, num_stages, uid: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(lib().cf_ctx_init_pp(self.h, C.c_int(rank), C.c_int(world), C.c_int(num_stages), buf))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().cf_nccl_unique_id(buf))
        return bytes(buf)

    def gemm(self, a, a_kmajor, lda, b, b_kmajor, ldb, c, ldc, m, n, k, epi, r=0, ldr=0):
        check(lib().cf_op_gemm(self.h, C.c_void_p(a), a_kmajor, lda, C.c_void_p(b), b_kmajor, ldb,
                               C.c_void_p(c), ldc, m, n, k, epi, C.c_void_p(r), ldr))

    def attention(self, impl, backward, q, q_stride, k, v, kv_stride, kv_rows, o, lse, dout, dq, dk, dv,
                  acc_stride, segs, T, H, KVH, dh):
        """Operator-level attention on device pointers; segs = [[q_start, len, kv_row0, prefix], ...]."""
        s = np.ascontiguousarray(np.asarray(segs, np.int32).reshape(-1, 4))
        vp = C.c_void_p
        check(lib().cf_op_attention(self.h, C.c_int(impl), C.c_int(int(backward)), vp(q), C.c_int64(q_stride),
                                    vp(k), vp(v), C.c_int64(kv_stride), C.c_int64(kv_rows), vp(o), vp(lse),
                                    vp(dout), vp(dq), vp(dk), vp(dv), C.c_int64(acc_stride), _p(s),
                                    C.c_int64(len(s)), C.c_int64(T), C.c_int64(H), C.c_int64(KVH),
                                    C.c_int64(dh)))

    def close(self):
        if self.h and self.h.value:
            lib().cf_ctx_destroy(self.h)
            self.h = C.c_void_p()


class LocalPipe:
    """In-process pipeline links (cf_pp_local): one context per stage, each
    driven by its own thread through Step.run_pp."""

    def __init__(self, num_stages):
        self.h = C.c_void_p()
        check(lib().cf_pp_local_create(C.c_int(num_stages), C.byref(self.h)))

    def close(self):
        if self.h and self.h.value:
            lib().cf_pp_local_destroy(self.h)
            self.h = C.c_void_p()


class Model:
    """Device model (ToyModelParams / Llama-shaped) with fp32 gradients."""

    def __init__(self, ctx: Context, cfg: ModelCfg, stage=None, num_stages=1):
        """Whole model, or (stage, num_stages) = one pipeline stage's slice."""
        self.ctx = ctx
        self.cfg = cfg
        self.h = C.c_void_p()
        self.stage, self.num_stages = (0, 1) if stage is None else (stage, num_stages)
        if stage is None:
            check(lib().cf_model_create(ctx.h, C.byref(cfg), C.byref(self.h)))
        else:
            check(lib().cf_model_create_stage(ctx.h, C.byref(cfg), C.c_int64(stage), C.c_int64(num_stages),
                                              C.byref(self.h)))

    def num_tensors(self):
        return lib().cf_model_num_tensors(self.h)

    def num_params(self):
        return lib().cf_model_num_params(self.h)

    def tensor_info(self, i):
        name = C.create_string_buffer(128)
        r, c = C.c_int64(), C.c_int64()
        check(lib().cf_model_tensor_info(self.h, C.c_int64(i), name, C.c_size_t(128), C.byref(r), C.byref(c)))
        return name.value.decode(), r.value, c.value

    def get_param(self, i):
        _, r, c = self.tensor_info(i)
        out = np.zeros((r, c), np.float64)
        check(lib().cf_model_get_param(self.h, C.c_int64(i), _p(out)))
        return out

    def set_param(self, i, value):
        v = np.ascontiguousarray(value, np.float64)
        check(lib().cf_model_set_param(self.h, C.c_int64(i), _p(v)))

    def get_grad(self, i):
        _, r, c = self.tensor_info(i)
        out = np.zeros((r, c), np.float64)
        check(lib().cf_model_get_grad(self.h, C.c_int64(i), _p(out)))
        return out

    def params_flat(self):
        return np.concatenate([self.get_param(i).ravel() for i in range(self.num_tensors())])

    def grads_flat(self):
        return np.concatenate([self.get_grad(i).ravel() for i in range(self.num_tensors())])

    def adamw_init(self):
        """fp32 master weights + zero moments (cf_model_adamw_init)."""
        check(lib().cf_model_adamw_init(self.h))

    def adamw_step(self, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, max_grad_norm=0.0,
                   decay_gains=False):
        """One fused AdamW step on the current gradients; returns the global
        gradient norm (before clipping)."""
        c = AdamWCfg(lr, beta1, beta2, eps, weight_decay, max_grad_norm, int(decay_gains), 0)
        norm = C.c_double()
        check(lib().cf_model_adamw_step(self.h, C.byref(c), C.byref(norm)))
        return norm.value

    def get_master(self, i):
        _, r, c = self.tensor_info(i)
        out = np.zeros((r, c), np.float64)
        check(lib().cf_model_get_master(self.h, C.c_int64(i), _p(out)))
        return out

    def grad_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        check(lib().cf_model_grad_buffer(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def run_plan(self, plan: Plan, lengths, tokens, ids=None, corrupt=False, normalizer=0.0,
                 accumulate=False, kv_offload=False) -> RunResult:
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        o = RunOpts(int(corrupt), int(accumulate), normalizer, 0, int(kv_offload))
        r = RunResult()
        check(lib().cf_run_plan(self.ctx.h, self.h, plan.h, _p(ids), _p(lengths), _p(tokens),
                                C.c_int64(len(lengths)), C.byref(o), C.byref(r)))
        return r

    def backward_full(self, lengths, tokens, ids=None, normalizer=0.0) -> RunResult:
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        r = RunResult()
        check(lib().cf_backward_full(self.ctx.h, self.h, _p(ids), _p(lengths), _p(tokens),
                                     C.c_int64(len(lengths)), C.c_double(normalizer), C.byref(r)))
        return r

    def kv_shape(self, rows):
        c = self.cfg
        return (int(c.num_layers), int(rows), int(c.num_kv_heads * (c.d_model // c.num_heads)))

    def segment_forward(self, tokens, targets, prefix_k=None, prefix_v=None, keep_tape=True):
        """detail::segment_forward (toy_model.hpp:206): one segment of one
        sequence after `prefix_k/v` ([L, prefix_len, kv_width] fp64).  Returns
        (loss_sum, saved_k, saved_v, tape); tape is None unless keep_tape."""
        tokens = np.ascontiguousarray(tokens, np.int32)
        targets = np.ascontiguousarray(targets, np.int64)
        n = len(tokens)
        if len(targets) != n:
            raise ValueError("tokens and targets differ in length")
        plen = 0 if prefix_k is None else int(np.shape(prefix_k)[1])
        pk = None if prefix_k is None else np.ascontiguousarray(prefix_k, np.float64)
        pv = None if prefix_v is None else np.ascontiguousarray(prefix_v, np.float64)
        sk = np.zeros(self.kv_shape(n))
        sv = np.zeros(self.kv_shape(n))
        loss = C.c_double()
        h = C.c_void_p()
        check(lib().cf_segment_forward(self.ctx.h, self.h, _p(tokens), C.c_int64(n), _p(targets),
                                       None if pk is None else _p(pk), None if pv is None else _p(pv),
                                       C.c_int64(plen), C.c_int(int(keep_tape)), C.byref(loss), _p(sk), _p(sv),
                                       C.byref(h)))
        return loss.value, sk, sv, (SegmentTape(h, plen, self) if h.value else None)

    def segment_backward(self, tape, normalizer, prefix_k=None, prefix_v=None, incoming_dk=None, incoming_dv=None,
                         d_prefix_k=None, d_prefix_v=None):
        """detail::segment_backward (toy_model.hpp:341): accumulates parameter
        gradients (the model's buffer) and the prefix K/V gradients into
        d_prefix_k/v (allocated as zeros when None; returned)."""
        h = tape.h if tape is not None else C.c_void_p()
        plen = tape.prefix_len if tape is not None else 0
        pk = None if prefix_k is None else np.ascontiguousarray(prefix_k, np.float64)
        pv = None if prefix_v is None else np.ascontiguousarray(prefix_v, np.float64)
        ik = None if incoming_dk is None else np.ascontiguousarray(incoming_dk, np.float64)
        iv = None if incoming_dv is None else np.ascontiguousarray(incoming_dv, np.float64)
        dpk = np.zeros(self.kv_shape(plen)) if d_prefix_k is None else d_prefix_k
        dpv = np.zeros(self.kv_shape(plen)) if d_prefix_v is None else d_prefix_v
        opt = lambda a: None if a is None else _p(a)  # noqa: E731
        check(lib().cf_segment_backward(self.ctx.h, self.h, h, opt(pk), opt(pv), _p(dpk), _p(dpv), opt(ik), opt(iv),
                                        C.c_double(normalizer)))
        return dpk, dpv

    def zero_grads(self):
        check(lib().cf_model_zero_grads(self.h))

    def close(self):
        if self.h and self.h.value:
            lib().cf_model_destroy(self.h)
            self.h = C.c_void_p()


class SegmentTape:
    """Retained activations of one segment_forward (cf_segment)."""

    def __init__(self, h, prefix_len, model):
        self.h = h
        self.prefix_len = prefix_len
        self.model = model  # the tape's device memory lives in the model's context

    def close(self):
        if self.h and self.h.value and self.model.h and self.model.h.value:
            lib().cf_segment_destroy(self.h)
        self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Step:
    """Prepared step (cf_step_prepare): inputs resident in HBM."""

    def __init__(self, model: Model, plan: Plan, lengths, tokens, ids=None):
        self.model = model
        self.plan = plan
        self.lengths = np.ascontiguousarray(lengths, np.int64)
        self.ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        self.tokens = np.ascontiguousarray(tokens, np.int32)
        self.h = C.c_void_p()
        check(lib().cf_step_prepare(model.ctx.h, model.h, plan.h, _p(self.ids), _p(self.lengths),
                                    _p(self.tokens), C.c_int64(len(self.lengths)), C.byref(self.h)))

    def run(self, corrupt=False, normalizer=0.0, accumulate=False, kv_offload=False) -> RunResult:
        o = RunOpts(int(corrupt), int(accumulate), normalizer, 0, int(kv_offload))
        r = RunResult()
        check(lib().cf_step_run(self.model.ctx.h, self.model.h, self.h, C.byref(o), C.byref(r)))
        return r

    def input_bytes(self):
        """Host -> device bytes of this step's inputs (cf_step_input_bytes)."""
        n = C.c_int64()
        check(lib().cf_step_input_bytes(self.h, C.byref(n)))
        return n.value

    def op_times(self):
        """(kinds, chunk_ids, ms) of every op of the last run (profiling on)."""
        n = C.c_int64()
        check(lib().cf_step_op_times(self.h, C.byref(n), None, None, None))
        kinds = np.zeros(n.value, np.int64)
        ids = np.zeros(n.value, np.int64)
        ms = np.zeros(n.value, np.float64)
        check(lib().cf_step_op_times(self.h, C.byref(n), _p(kinds), _p(ids), _p(ms)))
        return kinds, ids, ms

    def run_pp(self, k, corrupt=False, normalizer=0.0, accumulate=False, tape_budget=0, kv_offload=False) -> RunResult:
        """This rank's pipeline stage (cf_pp_step_run; needs Context.init_pp).
        tape_budget > 0: stage-input checkpointing beyond that many tapes."""
        o = RunOpts(int(corrupt), int(accumulate), normalizer, int(tape_budget), int(kv_offload))
        r = RunResult()
        check(lib().cf_pp_step_run(self.model.ctx.h, self.model.h, self.h, C.c_int64(k), C.byref(o), C.byref(r)))
        return r

    def run_pp_local(self, models, k, corrupt=False, normalizer=0.0, accumulate=False, tape_budget=0,
                     kv_offload=False) -> RunResult:
        """All pipeline stages on this device (cf_pp_run_local)."""
        arr = (C.c_void_p * len(models))(*[m.h.value for m in models])
        o = RunOpts(int(corrupt), int(accumulate), normalizer, int(tape_budget), int(kv_offload))
        r = RunResult()
        check(lib().cf_pp_run_local(self.model.ctx.h, arr, C.c_int64(len(models)), self.h, C.c_int64(k),
                                    C.byref(o), C.byref(r)))
        return r

    def close(self):
        if self.h and self.h.value:
            lib().cf_step_destroy(self.h)
            self.h = C.c_void_p()
