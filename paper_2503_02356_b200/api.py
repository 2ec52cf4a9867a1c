"""Reference-shaped Python API over the C-ABI.

Names and argument meaning follow the reference's chunkflow:: functions
(/root/reference/proj/include/chunkflow/): construct_chunks (chunker.hpp:177),
schedule_step (scheduler.hpp:132), validate_plan (:182), run_plan
(plan_runner.hpp:67), verify_equivalence (:368), compare_gradients
(toy_model.hpp:681).  Errors surface as CfError carrying the reference's
status code (CF_EVALIDATION for ValidationError, ...).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .capi import CfError, Context, Model, ModelCfg, Plan, RunResult  # noqa: F401


def model_cfg(arch=0, vocab=32, d=16, heads=4, kv_heads=2, layers=2, ffn=0, seed=7,
              rope_theta=10000.0, rms_eps=1e-5) -> ModelCfg:
    """ToyModelConfig defaults of the verify CLI (chunkflow_main.cpp:230-245)."""
    return ModelCfg(arch, 0, vocab, d, heads, kv_heads, layers, ffn, seed, rope_theta, rms_eps)


@dataclass
class ChunkSegment:
    sequence_id: int
    start_token: int
    length: int


@dataclass
class Chunk:
    chunk_id: int
    kind: str  # "standalone" | "dependent"
    segments: list
    group_id: int = -1
    index_in_group: int = -1
    total_tokens: int = 0


@dataclass
class ChunkPlan:
    chunk_size: int
    chunks: list
    groups: dict
    lengths: np.ndarray = field(repr=False, default=None)
    ids: np.ndarray = field(repr=False, default=None)


@dataclass
class ExecutionPlan:
    events: np.ndarray
    k: int
    chunk_size: int
    groups: dict
    handle: Plan = field(repr=False, default=None)


@dataclass
class PlanDiagnostics:
    peak_retained_tokens: int
    recompute_token_count: int
    violations: list


def construct_chunks(lengths, chunk_size, ids=None) -> ChunkPlan:
    lengths = np.ascontiguousarray(lengths, np.int64)
    ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
    p = Plan.build(lengths, chunk_size, 1, ids)
    ch, sg, _, _ = p.export()
    chunks = []
    for c in ch:
        segs = [ChunkSegment(int(s["sequence_id"]), int(s["start_token"]), int(s["length"]))
                for s in sg[c["seg_offset"]:c["seg_offset"] + c["seg_count"]]]
        chunks.append(Chunk(int(c["chunk_id"]), "standalone" if c["kind"] == 0 else "dependent", segs,
                            int(c["group_id"]), int(c["index_in_group"]), int(c["total_tokens"])))
    return ChunkPlan(int(chunk_size), chunks, p.groups(), lengths, ids)


def schedule_step(chunk_plan: ChunkPlan, k: int) -> ExecutionPlan:
    p = Plan.build(chunk_plan.lengths, chunk_plan.chunk_size, k, chunk_plan.ids)
    _, _, ev, _ = p.export()
    return ExecutionPlan(ev, int(k), chunk_plan.chunk_size, p.groups(), p)


def validate_plan(plan: ExecutionPlan) -> PlanDiagnostics:
    _, _, _, dg = plan.handle.export()
    return PlanDiagnostics(int(dg["peak_retained_tokens"]), int(dg["recompute_token_count"]),
                           plan.handle.violations())


def run_plan(model: Model, plan: ExecutionPlan, lengths, tokens, ids=None, corrupt_kv_grads=False,
             normalizer_override=0.0) -> RunResult:
    return model.run_plan(plan.handle, lengths, tokens, ids, corrupt_kv_grads, normalizer_override)


@dataclass
class GradComparison:
    rows: list
    loss_rel_err: float
    max_rel_err: float
    mean_rel_err: float

    def to_text(self) -> str:
        """GradComparison::to_text (toy_model.hpp:668-678), same layout."""
        out = "".join(f"{n} max_abs_diff={d:.6e} rel_err={r:.6e}\n" for n, d, r in self.rows)
        return out + (f"loss_rel_err={self.loss_rel_err:.6e}\nmax_rel_err={self.max_rel_err:.6e}\n"
                      f"mean_rel_err={self.mean_rel_err:.6e}\n")


def compare_gradients(names, a_loss, a, b_loss, b, denom_floor=1e-12) -> GradComparison:
    """Per-tensor max|a-b| / max(max|a|, max|b|, floor) (toy_model.hpp:681-718)."""
    rows = []
    for n, ta, tb in zip(names, a, b):
        diff = float(np.max(np.abs(ta - tb))) if ta.size else 0.0
        mag = max(float(np.max(np.abs(ta))) if ta.size else 0.0, float(np.max(np.abs(tb))) if tb.size else 0.0)
        rows.append((n, diff, diff / max(mag, denom_floor)))
    loss_rel = abs(a_loss - b_loss) / max(abs(a_loss), abs(b_loss), denom_floor)
    rels = [r[2] for r in rows]
    return GradComparison(rows, loss_rel, max(rels) if rels else 0.0, float(np.mean(rels)) if rels else 0.0)


@dataclass
class VerifyReport:
    passed: bool
    loss_rel_err: float
    max_grad_rel_err: float
    comparison: GradComparison
    instrumentation: dict
    chunk_count: int
    event_count: int

    def to_text(self) -> str:
        """VerifyReport::to_text (plan_runner.hpp:352-365), same layout."""
        i = self.instrumentation
        return (f"chunks: {self.chunk_count}\nevents: {self.event_count}\n" + self.comparison.to_text()
                + f"recompute_forwards: {i['recompute_forward_count']}\n"
                + f"recompute_loss_mismatches: {i['recompute_loss_mismatches']}\n"
                + f"kv_completeness_violations: {i['kv_completeness_violations']}\n"
                + f"result: {'PASS' if self.passed else 'FAIL'}\n")


def verify_equivalence(model: Model, lengths, tokens, chunk_size, k, loss_tol=2e-3, grad_tol=3e-2,
                       ids=None, corrupt_kv_grads=False) -> VerifyReport:
    """Chunked-with-state gradients vs the unchunked run, both on the GPU
    (plan_runner.hpp:368-395).  Default tolerances are the bf16/fp32-accumulate
    ones stated in DESIGN.md (the reference's fp64 1e-12/1e-9 do not apply)."""
    cp = construct_chunks(lengths, chunk_size, ids)
    ep = schedule_step(cp, k)
    r = run_plan(model, ep, lengths, tokens, ids, corrupt_kv_grads)
    nt = model.num_tensors()
    names = [model.tensor_info(i)[0] for i in range(nt)]
    ga = [model.get_grad(i) for i in range(nt)]
    f = model.backward_full(lengths, tokens, ids)
    gb = [model.get_grad(i) for i in range(nt)]
    cmp = compare_gradients(names, r.loss, ga, f.loss, gb)
    instr = {"recompute_forward_count": r.recompute_forward_count,
             "recompute_loss_mismatches": r.recompute_loss_mismatches,
             "kv_completeness_violations": r.kv_completeness_violations,
             "peak_retained_tokens": r.peak_retained_tokens}
    ok = (cmp.loss_rel_err <= loss_tol and cmp.max_rel_err <= grad_tol
          and r.recompute_loss_mismatches == 0 and r.kv_completeness_violations == 0)
    return VerifyReport(ok, cmp.loss_rel_err, cmp.max_rel_err, cmp, instr, len(cp.chunks), len(ep.events))
