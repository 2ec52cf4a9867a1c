// chunkflow_b200.hpp — header-only C++ facade with the reference's API shape
// (namespace chunkflow, /root/reference/proj/include/chunkflow/) over the
// C-ABI in chunkflow_b200.h.  A caller of the reference swaps
//   #include <chunkflow/plan_runner.hpp>   for   #include <chunkflow_b200.hpp>
// and keeps construct_chunks / schedule_step / validate_plan / run_plan /
// verify_equivalence call sites; errors are rethrown as the same exception
// types (ValidationError, ParseError, IoError), CUDA/NCCL failures as
// std::runtime_error.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "chunkflow_b200.h"

namespace chunkflow_b200 {

class ValidationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ParseError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == CF_OK) return;
  const std::string msg = cf_last_error();
  if (rc == CF_EVALIDATION) throw ValidationError(msg);
  if (rc == CF_EPARSE) throw ParseError(msg);
  if (rc == CF_EIO) throw IoError(msg);
  throw std::runtime_error(msg);
}

// --- chunker.hpp:16-37 / scheduler.hpp:17-43 types
enum class ChunkKind { kStandalone, kDependent };
enum class ExecKind { kForwardDiscard, kForwardRetain, kBackward };

struct SequenceRecord {  // dataset.hpp:20-27
  int64_t id = 0;
  int64_t length = 0;
  std::vector<int32_t> tokens;
};
using SequenceSet = std::vector<SequenceRecord>;
struct Batch {  // dataset.hpp:75-82
  int64_t step = 0;
  std::vector<SequenceRecord> sequences;
  int64_t global_batch_size = 0;
};

struct ChunkSegment {
  int64_t sequence_id = 0, start_token = 0, length = 0;
};
struct Chunk {
  int64_t chunk_id = 0;
  ChunkKind kind = ChunkKind::kStandalone;
  std::vector<ChunkSegment> segments;
  int64_t group_id = -1, index_in_group = -1, total_tokens = 0;
};
struct KvActions {
  bool save_kv = false, read_kv_prefix = false, accumulate_kv_grad = false;
};
struct ExecEvent {
  ExecKind kind = ExecKind::kForwardRetain;
  int64_t chunk_id = 0, group_id = -1, index_in_group = -1;
  bool is_recompute = false;
  KvActions notes;
};
struct PlanDiagnostics {
  int64_t peak_retained_tokens = 0, recompute_token_count = 0;
  std::vector<std::string> violations;
};

// Owns the library-side plan handle (chunk plan + its schedule).
class PlanHandle {
 public:
  explicit PlanHandle(cf_plan* p) : p_(p, &cf_plan_destroy) {}
  cf_plan* get() const { return p_.get(); }

 private:
  std::shared_ptr<cf_plan> p_;
};

struct ChunkPlan {
  int64_t chunk_size = 0;
  std::vector<Chunk> chunks;
  std::map<int64_t, std::vector<int64_t>> groups;
  std::vector<int64_t> ids, lengths;  // the batch it was built from
};
struct ExecutionPlan {  // scheduler.hpp:35-43
  std::vector<ExecEvent> events;
  int64_t k = 1, chunk_size = 0;
  std::map<int64_t, std::vector<int64_t>> groups;
  std::map<int64_t, int64_t> chunk_tokens;
  std::shared_ptr<PlanHandle> handle;  // the library plan of the chunks (set by schedule_step)
};

namespace detail {
inline std::shared_ptr<PlanHandle> build(const std::vector<int64_t>& ids, const std::vector<int64_t>& lengths,
                                         int64_t cs, int64_t k) {
  cf_plan* p = nullptr;
  check(cf_plan_build(ids.data(), lengths.data(), static_cast<int64_t>(ids.size()), cs, k, &p));
  return std::make_shared<PlanHandle>(p);
}
inline std::map<int64_t, std::vector<int64_t>> groups_of(cf_plan* p) {
  int64_t nc = 0, ns = 0, ne = 0, ng = 0;
  check(cf_plan_counts(p, &nc, &ns, &ne, &ng));
  std::vector<int64_t> gid(static_cast<size_t>(ng) + 1), off(static_cast<size_t>(ng) + 1);
  check(cf_plan_export_groups(p, nullptr, off.data(), nullptr));  // sizes the member list
  std::vector<int64_t> mem(static_cast<size_t>(off[static_cast<size_t>(ng)]) + 1);
  check(cf_plan_export_groups(p, gid.data(), off.data(), mem.data()));
  std::map<int64_t, std::vector<int64_t>> out;
  for (int64_t g = 0; g < ng; ++g) out[gid[g]] = std::vector<int64_t>(mem.begin() + off[g], mem.begin() + off[g + 1]);
  return out;
}
}  // namespace detail

// construct_chunks (chunker.hpp:177)
inline ChunkPlan construct_chunks(const Batch& batch, int64_t chunk_size) {
  ChunkPlan plan;
  plan.chunk_size = chunk_size;
  for (const SequenceRecord& s : batch.sequences) {
    plan.ids.push_back(s.id);
    plan.lengths.push_back(s.length);
  }
  auto h = detail::build(plan.ids, plan.lengths, chunk_size, 1);
  int64_t nc = 0, ns = 0, ne = 0, ng = 0;
  check(cf_plan_counts(h->get(), &nc, &ns, &ne, &ng));
  std::vector<cf_chunk_rec> ch(static_cast<size_t>(nc));
  std::vector<cf_segment_rec> sg(static_cast<size_t>(ns));
  check(cf_plan_export(h->get(), ch.data(), sg.data(), nullptr, nullptr));
  for (const cf_chunk_rec& c : ch) {
    Chunk out;
    out.chunk_id = c.chunk_id;
    out.kind = c.kind == CF_CHUNK_STANDALONE ? ChunkKind::kStandalone : ChunkKind::kDependent;
    out.group_id = c.group_id;
    out.index_in_group = c.index_in_group;
    out.total_tokens = c.total_tokens;
    for (int64_t i = 0; i < c.seg_count; ++i) {
      const cf_segment_rec& s = sg[static_cast<size_t>(c.seg_offset + i)];
      out.segments.push_back({s.sequence_id, s.start_token, s.length});
    }
    plan.chunks.push_back(std::move(out));
  }
  plan.groups = detail::groups_of(h->get());
  return plan;
}

// schedule_step (scheduler.hpp:132)
inline ExecutionPlan schedule_step(const ChunkPlan& chunk_plan, int64_t k) {
  ExecutionPlan plan;
  plan.k = k;
  plan.chunk_size = chunk_plan.chunk_size;
  plan.handle = detail::build(chunk_plan.ids, chunk_plan.lengths, chunk_plan.chunk_size, k);
  int64_t nc = 0, ns = 0, ne = 0, ng = 0;
  check(cf_plan_counts(plan.handle->get(), &nc, &ns, &ne, &ng));
  std::vector<cf_event_rec> ev(static_cast<size_t>(ne));
  check(cf_plan_export(plan.handle->get(), nullptr, nullptr, ev.data(), nullptr));
  for (const cf_event_rec& e : ev) {
    ExecEvent x;
    x.kind = static_cast<ExecKind>(e.kind);
    x.chunk_id = e.chunk_id;
    x.group_id = e.group_id;
    x.index_in_group = e.index_in_group;
    x.is_recompute = e.is_recompute != 0;
    x.notes = {e.save_kv != 0, e.read_kv_prefix != 0, e.accumulate_kv_grad != 0};
    plan.events.push_back(x);
  }
  plan.groups = chunk_plan.groups;
  for (const Chunk& c : chunk_plan.chunks) plan.chunk_tokens[c.chunk_id] = c.total_tokens;
  return plan;
}

namespace detail {
// The plan as the caller holds it (events possibly edited or built by hand),
// replayed by the library; carries the chunks of `plan.handle` when present.
inline std::shared_ptr<PlanHandle> replay(const ExecutionPlan& plan) {
  std::vector<cf_event_rec> ev;
  for (const ExecEvent& e : plan.events)
    ev.push_back({static_cast<int64_t>(e.kind), e.chunk_id, e.group_id, e.index_in_group, e.is_recompute ? 1 : 0,
                  e.notes.save_kv ? 1 : 0, e.notes.read_kv_prefix ? 1 : 0, e.notes.accumulate_kv_grad ? 1 : 0});
  std::vector<int64_t> gid, off{0}, mem, tc, tn;
  for (const auto& [g, members] : plan.groups) {
    gid.push_back(g);
    mem.insert(mem.end(), members.begin(), members.end());
    off.push_back(static_cast<int64_t>(mem.size()));
  }
  for (const auto& [c, t] : plan.chunk_tokens) {
    tc.push_back(c);
    tn.push_back(t);
  }
  cf_plan* p = nullptr;
  check(cf_plan_validate_events(plan.chunk_size, plan.k, ev.data(), static_cast<int64_t>(ev.size()), gid.data(),
                                off.data(), mem.data(), static_cast<int64_t>(gid.size()), tc.data(), tn.data(),
                                static_cast<int64_t>(tc.size()), plan.handle ? plan.handle->get() : nullptr, &p));
  return std::make_shared<PlanHandle>(p);
}
inline PlanDiagnostics diagnostics(cf_plan* p) {
  cf_plan_diag d{};
  check(cf_plan_export(p, nullptr, nullptr, nullptr, &d));
  PlanDiagnostics out{d.peak_retained_tokens, d.recompute_token_count, {}};
  for (int64_t i = 0; i < d.num_violations; ++i) {
    char buf[256];
    check(cf_plan_violation(p, i, buf, sizeof(buf)));
    out.violations.emplace_back(buf);
  }
  return out;
}
}  // namespace detail

// validate_plan (scheduler.hpp:182): replays plan.events as the caller holds
// them (so hand-built or edited plans get the reference's violation texts).
inline PlanDiagnostics validate_plan(const ExecutionPlan& plan) { return detail::diagnostics(detail::replay(plan)->get()); }

// --- pipeline.hpp:24-72 types and the simulator entry points
struct CostModel {  // pipeline.hpp:24-47
  double gamma = 0.0, alpha = 1.0, beta = 0.0, backward_multiplier = 2.0, hop_latency = 0.0;
};
struct PipelineConfig {  // pipeline.hpp:49-53
  int num_stages = 1;
  int64_t k = 1;
  int64_t chunk_size = 0;
};
enum class TraceEventKind { kForward, kRecomputeForward, kBackward };
struct TraceEvent {
  TraceEventKind kind = TraceEventKind::kForward;
  int64_t chunk_id = 0;
  double start = 0.0, end = 0.0;
};
struct PipelineTrace {  // pipeline.hpp:64-72
  std::vector<std::vector<TraceEvent>> stages;
  double makespan = 0.0;
  std::vector<double> busy, busy_total;
  double bubble = 0.0;  // bubble_ratio(), computed by the library
};
enum class DispatchPolicy { kBackwardFirst, kForwardFirst };

namespace detail {
inline PipelineTrace unpack_trace(const std::vector<cf_pp_op>& ops, const std::vector<double>& busy,
                                  const std::vector<double>& busy_total, const cf_pp_result& r, int stages) {
  PipelineTrace t;
  t.makespan = r.makespan;
  t.bubble = r.bubble_ratio;
  t.busy = busy;
  t.busy_total = busy_total;
  t.stages.resize(static_cast<size_t>(stages));
  for (int s = 0; s < stages; ++s)
    for (int64_t i = 0; i < r.ops_per_stage; ++i) {
      const cf_pp_op& o = ops[static_cast<size_t>(s * r.ops_per_stage + i)];
      t.stages[static_cast<size_t>(s)].push_back({static_cast<TraceEventKind>(o.kind), o.chunk_id, o.start, o.end});
    }
  return t;
}
inline cf_pp_cost to_cost(const CostModel& c) {
  return {c.gamma, c.alpha, c.beta, c.backward_multiplier, c.hop_latency};
}
}  // namespace detail

// simulate_state_aware_1f1b (pipeline.hpp:250)
inline PipelineTrace simulate_state_aware_1f1b(const ChunkPlan& plan, const PipelineConfig& cfg, const CostModel& cost,
                                               DispatchPolicy policy = DispatchPolicy::kBackwardFirst) {
  auto h = detail::build(plan.ids, plan.lengths, plan.chunk_size, cfg.k);
  const cf_pp_cost c = detail::to_cost(cost);
  cf_pp_result r{};
  const int bf = policy == DispatchPolicy::kBackwardFirst ? 1 : 0;
  check(cf_pp_simulate(h->get(), cfg.num_stages, cfg.k, &c, bf, nullptr, nullptr, nullptr, nullptr, nullptr, &r));
  std::vector<cf_pp_op> ops(static_cast<size_t>(cfg.num_stages * r.ops_per_stage));
  std::vector<double> busy(static_cast<size_t>(cfg.num_stages)), busy_total(busy.size());
  check(cf_pp_simulate(h->get(), cfg.num_stages, cfg.k, &c, bf, nullptr, nullptr, ops.data(), busy.data(),
                       busy_total.data(), &r));
  return detail::unpack_trace(ops, busy, busy_total, r, cfg.num_stages);
}

// simulate_1f1b (pipeline.hpp:218)
inline PipelineTrace simulate_1f1b(const std::vector<int64_t>& lengths, int num_stages, const CostModel& cost) {
  const cf_pp_cost c = detail::to_cost(cost);
  cf_pp_result r{};
  std::vector<cf_pp_op> ops(static_cast<size_t>(num_stages) * 2 * lengths.size());
  std::vector<double> busy(static_cast<size_t>(num_stages)), busy_total(busy.size());
  check(cf_pp_simulate_1f1b(lengths.data(), static_cast<int64_t>(lengths.size()), num_stages, &c, ops.data(),
                            busy.data(), busy_total.data(), &r));
  return detail::unpack_trace(ops, busy, busy_total, r, num_stages);
}

// bubble_ratio (pipeline.hpp:325): recompute forwards count as bubble.
inline double bubble_ratio(const PipelineTrace& t) { return t.bubble; }

// --- tuner.hpp / memory_model.hpp / wire formats (chunker.hpp:233-292,
//     scheduler.hpp:300-328, dataset.hpp:112-176)
struct MemoryModelCoefficients {  // memory_model.hpp:20-33
  double base = 0.0, per_chunk_token = 0.0, per_context_token = 0.0, gqa_ratio = 1.0;
};
struct MemoryMeasurement {  // memory_model.hpp:13-18
  int64_t chunk_size = 0, k = 1, context_len = 0;
  double peak_gib = 0.0;
};
struct CalibrationResult {
  MemoryModelCoefficients coefficients;
  double max_residual_gib = 0.0;
};
inline double predict_peak(const MemoryModelCoefficients& c, int64_t chunk_size, int64_t k, int64_t context_len) {
  const cf_mem_coeffs m{c.base, c.per_chunk_token, c.per_context_token, c.gqa_ratio};
  double out = 0.0;
  check(cf_mem_predict(&m, chunk_size, k, context_len, &out));
  return out;
}
inline CalibrationResult calibrate(const std::vector<MemoryMeasurement>& ms, double gqa_ratio = 1.0) {
  std::vector<int64_t> cs, k, ctx;
  std::vector<double> pk;
  for (const MemoryMeasurement& m : ms) {
    cs.push_back(m.chunk_size);
    k.push_back(m.k);
    ctx.push_back(m.context_len);
    pk.push_back(m.peak_gib);
  }
  cf_mem_coeffs c{};
  CalibrationResult r;
  check(cf_mem_calibrate(cs.data(), k.data(), ctx.data(), pk.data(), static_cast<int64_t>(ms.size()), gqa_ratio, &c,
                         &r.max_residual_gib));
  r.coefficients = {c.base_gib, c.per_chunk_token_gib, c.per_context_token_gib, c.gqa_ratio};
  return r;
}

struct TunerCandidate {  // tuner.hpp:18-24
  int64_t chunk_size = 0, k = 1;
  double mean_time = 0.0, predicted_peak_gib = 0.0;
  bool feasible = false;
};
struct TunerResult {  // tuner.hpp:26-32
  bool has_best = false;
  int64_t best_chunk_size = 0, best_k = 0, evaluations = 0;
  std::vector<TunerCandidate> table;
  std::string report;  // tuner_report(result)
};
// grid_search (tuner.hpp:39)
inline TunerResult grid_search(const SequenceSet& set, const std::vector<int64_t>& chunk_sizes,
                               const std::vector<int64_t>& ks, const PipelineConfig& cfg, const CostModel& cost,
                               const MemoryModelCoefficients& mem, double budget_gib, int64_t global_batch_size,
                               int64_t batches_to_sample, uint64_t seed) {
  std::vector<int64_t> ids, lengths;
  for (const SequenceRecord& r : set) {
    ids.push_back(r.id);
    lengths.push_back(r.length);
  }
  const cf_pp_cost c = detail::to_cost(cost);
  const cf_mem_coeffs m{mem.base, mem.per_chunk_token, mem.per_context_token, mem.gqa_ratio};
  std::vector<cf_tune_row> rows(chunk_sizes.size() * ks.size());
  int64_t bc = -1, bk = -1, ev = 0;
  size_t len = 0;
  auto call = [&](char* buf, size_t cap) {
    check(cf_tune_grid_search(ids.data(), lengths.data(), static_cast<int64_t>(ids.size()), chunk_sizes.data(),
                              static_cast<int64_t>(chunk_sizes.size()), ks.data(), static_cast<int64_t>(ks.size()),
                              cfg.num_stages, &c, &m, budget_gib, global_batch_size, batches_to_sample, seed,
                              rows.data(), &bc, &bk, &ev, 0, buf, cap, &len));
  };
  call(nullptr, 0);
  std::string text(len + 1, '\0');
  call(&text[0], text.size());
  text.resize(len);
  TunerResult r;
  r.has_best = bc >= 0;
  r.best_chunk_size = r.has_best ? bc : 0;
  r.best_k = r.has_best ? bk : 0;
  r.evaluations = ev;
  for (const cf_tune_row& x : rows) r.table.push_back({x.chunk_size, x.k, x.mean_time, x.predicted_peak_gib, x.feasible != 0});
  r.report = std::move(text);
  return r;
}

namespace detail {
template <class F>
inline std::string text_of(F&& f) {
  size_t len = 0;
  check(f(nullptr, 0, &len));
  std::string s(len + 1, '\0');
  check(f(&s[0], s.size(), &len));
  s.resize(len);
  return s;
}
}  // namespace detail

// chunk_plan_to_json(plan).dump(2) + "\n" (chunker.hpp:233) / execution_plan_to_json (scheduler.hpp:300)
inline std::string chunk_plan_json(const ExecutionPlan& plan) {
  return detail::text_of([&](char* b, size_t c, size_t* l) { return cf_plan_chunk_json(plan.handle->get(), b, c, l); });
}
inline std::string execution_plan_json(const ExecutionPlan& plan) {
  return detail::text_of([&](char* b, size_t c, size_t* l) { return cf_plan_exec_json(plan.handle->get(), b, c, l); });
}

// load_lengths (dataset.hpp:112): JSONL records -> SequenceSet
inline SequenceSet load_lengths(const std::string& jsonl) {
  int64_t n = 0, nt = 0;
  check(cf_dataset_load_jsonl(jsonl.c_str(), &n, nullptr, nullptr, nullptr, &nt, nullptr));
  std::vector<int64_t> ids(static_cast<size_t>(n)), lengths(static_cast<size_t>(n)), has(static_cast<size_t>(n));
  std::vector<int32_t> tokens(static_cast<size_t>(nt) + 1);
  check(cf_dataset_load_jsonl(jsonl.c_str(), &n, ids.data(), lengths.data(), has.data(), &nt, tokens.data()));
  SequenceSet set;
  int64_t off = 0;
  for (int64_t i = 0; i < n; ++i) {
    SequenceRecord r;
    r.id = ids[static_cast<size_t>(i)];
    r.length = lengths[static_cast<size_t>(i)];
    if (has[static_cast<size_t>(i)]) {
      r.tokens.assign(tokens.begin() + off, tokens.begin() + off + r.length);
      off += r.length;
    }
    set.push_back(std::move(r));
  }
  return set;
}

// RAII device context + model (ToyModelParams on the GPU).
class Device {
 public:
  explicit Device(int device = 0) {
    cf_ctx* c = nullptr;
    check(cf_ctx_create(device, &c));
    ctx_.reset(c, &cf_ctx_destroy);
  }
  cf_ctx* get() const { return ctx_.get(); }

 private:
  std::shared_ptr<cf_ctx> ctx_;
};

class Model {
 public:
  Model(const Device& dev, const cf_model_cfg& cfg) : dev_(dev) {
    cf_model* m = nullptr;
    check(cf_model_create(dev.get(), &cfg, &m));
    m_.reset(m, &cf_model_destroy);
  }
  cf_model* get() const { return m_.get(); }
  const Device& device() const { return dev_; }

 private:
  Device dev_;
  std::shared_ptr<cf_model> m_;
};

struct RunPlanOptions {  // plan_runner.hpp:49-54
  bool corrupt_kv_grads = false;
  double normalizer_override = 0.0;
};

// run_plan (plan_runner.hpp:67): loss + gradients stay on the device
// (cf_model_get_grad reads them back in the reference tensor order).
inline cf_run_result run_plan(const Model& model, const ChunkPlan& /*chunk_plan*/, const ExecutionPlan& exec_plan,
                              const SequenceSet& batch, const RunPlanOptions& options = {}) {
  std::vector<int64_t> ids, lengths;
  std::vector<int32_t> tokens;
  for (const SequenceRecord& s : batch) {
    ids.push_back(s.id);
    lengths.push_back(s.length);
    if (static_cast<int64_t>(s.tokens.size()) != s.length)
      throw ValidationError("sequence " + std::to_string(s.id) + " has no token payload");
    tokens.insert(tokens.end(), s.tokens.begin(), s.tokens.end());
  }
  if (!exec_plan.handle) throw ValidationError("execution plan has no chunk plan (build it with schedule_step)");
  // run_plan validates the plan it is given (plan_runner.hpp:78-81): the
  // caller's events are replayed, and an edited but valid schedule runs as is
  const auto plan = detail::replay(exec_plan);
  const PlanDiagnostics diag = detail::diagnostics(plan->get());
  if (!diag.violations.empty()) throw ValidationError("execution plan is invalid: " + diag.violations.front());
  cf_run_opts o{options.corrupt_kv_grads ? 1 : 0, 0, options.normalizer_override, 0, 0, 0};
  cf_run_result r{};
  check(cf_run_plan(model.device().get(), model.get(), plan->get(), ids.data(), lengths.data(), tokens.data(),
                    static_cast<int64_t>(ids.size()), &o, &r));
  return r;
}

// --- GradientSet / compare_gradients / backward_full / verify_equivalence
//     (toy_model.hpp:88-108, :575-596, :654-718; plan_runner.hpp:343-395).
// The GPU keeps gradients in the model's device buffer; read_gradients()
// copies them out in the reference tensor order as fp64.
struct Tensor {  // toy_model.hpp:48-56
  std::string name;
  int64_t rows = 0, cols = 0;
  std::vector<double> data;
  size_t size() const { return data.size(); }
};
struct GradientSet {  // toy_model.hpp:88-93
  std::vector<Tensor> tensors;
  double loss = 0.0;
};

inline GradientSet read_gradients(const Model& model, double loss) {
  GradientSet g;
  g.loss = loss;
  const int64_t n = cf_model_num_tensors(model.get());
  for (int64_t i = 0; i < n; ++i) {
    Tensor t;
    char name[128];
    check(cf_model_tensor_info(model.get(), i, name, sizeof(name), &t.rows, &t.cols));
    t.name = name;
    t.data.resize(static_cast<size_t>(t.rows * t.cols));
    check(cf_model_get_grad(model.get(), i, t.data.data()));
    g.tensors.push_back(std::move(t));
  }
  return g;
}

inline std::string format_scientific(double value) {  // common.hpp:81-85
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.6e", value);
  return std::string(buf);
}

struct GradComparisonRow {  // toy_model.hpp:656-660
  std::string name;
  double max_abs_diff = 0.0;
  double rel_err = 0.0;
};
struct GradComparison {  // toy_model.hpp:662-679
  std::vector<GradComparisonRow> rows;
  double loss_a = 0.0, loss_b = 0.0, loss_rel_err = 0.0, max_rel_err = 0.0, mean_rel_err = 0.0;
  std::string to_text() const {
    std::string out;
    for (const GradComparisonRow& row : rows)
      out += row.name + " max_abs_diff=" + format_scientific(row.max_abs_diff) +
             " rel_err=" + format_scientific(row.rel_err) + "\n";
    out += "loss_rel_err=" + format_scientific(loss_rel_err) + "\n";
    out += "max_rel_err=" + format_scientific(max_rel_err) + "\n";
    out += "mean_rel_err=" + format_scientific(mean_rel_err) + "\n";
    return out;
  }
};

// compare_gradients (toy_model.hpp:681-718): per-tensor max-norm relative
// error, optionally restricted to masked entries.
inline GradComparison compare_gradients(const GradientSet& a, const GradientSet& b,
                                        const std::vector<std::vector<uint8_t>>* mask = nullptr,
                                        double denom_floor = 1e-12) {
  if (a.tensors.size() != b.tensors.size()) throw ValidationError("gradient sets have different tensor counts");
  GradComparison cmp;
  cmp.loss_a = a.loss;
  cmp.loss_b = b.loss;
  cmp.loss_rel_err = std::abs(a.loss - b.loss) / std::max({std::abs(a.loss), std::abs(b.loss), denom_floor});
  double rel_sum = 0.0;
  for (size_t ti = 0; ti < a.tensors.size(); ++ti) {
    const Tensor& ta = a.tensors[ti];
    const Tensor& tb = b.tensors[ti];
    if (ta.size() != tb.size()) throw ValidationError("gradient tensor shape mismatch for " + ta.name);
    double max_diff = 0.0, max_mag = 0.0;
    for (size_t i = 0; i < ta.data.size(); ++i) {
      if (mask && !(*mask)[ti][i]) continue;
      max_diff = std::max(max_diff, std::abs(ta.data[i] - tb.data[i]));
      max_mag = std::max({max_mag, std::abs(ta.data[i]), std::abs(tb.data[i])});
    }
    GradComparisonRow row{ta.name, max_diff, max_diff / std::max(max_mag, denom_floor)};
    cmp.max_rel_err = std::max(cmp.max_rel_err, row.rel_err);
    rel_sum += row.rel_err;
    cmp.rows.push_back(std::move(row));
  }
  cmp.mean_rel_err = cmp.rows.empty() ? 0.0 : rel_sum / static_cast<double>(cmp.rows.size());
  return cmp;
}

namespace detail {
inline void flatten(const SequenceSet& batch, std::vector<int64_t>& ids, std::vector<int64_t>& lengths,
                    std::vector<int32_t>& tokens) {
  for (const SequenceRecord& s : batch) {
    if (static_cast<int64_t>(s.tokens.size()) != s.length)
      throw ValidationError("sequence " + std::to_string(s.id) + " has no token payload");
    ids.push_back(s.id);
    lengths.push_back(s.length);
    tokens.insert(tokens.end(), s.tokens.begin(), s.tokens.end());
  }
}
}  // namespace detail

// backward_full (toy_model.hpp:575-596): every sequence alone, unchunked;
// the model's gradient buffer is overwritten and returned.
inline GradientSet backward_full(const Model& model, const SequenceSet& batch, double normalizer_override = 0.0) {
  std::vector<int64_t> ids, lengths;
  std::vector<int32_t> tokens;
  detail::flatten(batch, ids, lengths, tokens);
  cf_run_result r{};
  check(cf_backward_full(model.device().get(), model.get(), ids.data(), lengths.data(), tokens.data(),
                         static_cast<int64_t>(ids.size()), normalizer_override, &r));
  return read_gradients(model, r.loss);
}

struct RunInstrumentation {  // plan_runner.hpp:36-47
  int64_t peak_retained_tokens = 0, recompute_forward_count = 0, recompute_loss_mismatches = 0,
          kv_completeness_violations = 0;
};

struct VerifyReport {  // plan_runner.hpp:343-366
  bool pass = false;
  double loss_rel_err = 0.0;
  double max_grad_rel_err = 0.0;
  GradComparison comparison;
  RunInstrumentation instrumentation;
  int64_t chunk_count = 0;
  int64_t event_count = 0;
  std::string to_text() const {
    std::string out;
    out += "chunks: " + std::to_string(chunk_count) + "\n";
    out += "events: " + std::to_string(event_count) + "\n";
    out += comparison.to_text();
    out += "recompute_forwards: " + std::to_string(instrumentation.recompute_forward_count) + "\n";
    out += "recompute_loss_mismatches: " + std::to_string(instrumentation.recompute_loss_mismatches) + "\n";
    out += "kv_completeness_violations: " + std::to_string(instrumentation.kv_completeness_violations) + "\n";
    out += std::string("result: ") + (pass ? "PASS" : "FAIL") + "\n";
    return out;
  }
};

// verify_equivalence (plan_runner.hpp:368-395) on the GPU: chunk, schedule
// and run the batch, then compare with backward_full.  The reference's
// defaults (1e-12 / 1e-9) are fp64 tolerances; a bf16/fp32 B200 model needs
// the tolerances of DESIGN.md §4 (e.g. 1e-4 / 1e-2 chunked vs unchunked).
inline VerifyReport verify_equivalence(const Model& model, const SequenceSet& batch, int64_t chunk_size, int64_t k,
                                       double loss_tol = 1e-12, double grad_tol = 1e-9,
                                       const RunPlanOptions& options = {}) {
  Batch wrapped;
  wrapped.sequences = batch;
  wrapped.global_batch_size = static_cast<int64_t>(batch.size());
  const ChunkPlan chunk_plan = construct_chunks(wrapped, chunk_size);
  const ExecutionPlan exec_plan = schedule_step(chunk_plan, k);
  const cf_run_result run = run_plan(model, chunk_plan, exec_plan, batch, options);
  const GradientSet chunked = read_gradients(model, run.loss);
  const GradientSet full = backward_full(model, batch, options.normalizer_override);
  VerifyReport report;
  report.chunk_count = static_cast<int64_t>(chunk_plan.chunks.size());
  report.event_count = static_cast<int64_t>(exec_plan.events.size());
  report.comparison = compare_gradients(chunked, full);
  report.loss_rel_err = report.comparison.loss_rel_err;
  report.max_grad_rel_err = report.comparison.max_rel_err;
  report.instrumentation = {run.peak_retained_tokens, run.recompute_forward_count, run.recompute_loss_mismatches,
                            run.kv_completeness_violations};
  report.pass = report.loss_rel_err <= loss_tol && report.max_grad_rel_err <= grad_tol &&
                run.recompute_loss_mismatches == 0 && run.kv_completeness_violations == 0;
  return report;
}

namespace detail {

// SegmentTape (toy_model.hpp:155-165) for the device operators: the saved
// key/value rows and loss come back to the host; the retained activations
// stay on the device behind `handle` (null for a discarding forward).
struct SegmentTape {
  int64_t len = 0;
  int64_t prefix_len = 0;
  std::vector<std::vector<double>> saved_k;  // per layer, len x kv_width
  std::vector<std::vector<double>> saved_v;
  double loss_sum = 0.0;
  std::shared_ptr<cf_segment> handle;
};

inline std::vector<double> flatten_kv(const std::vector<std::vector<double>>& per_layer, size_t layers, size_t n,
                                      const char* what) {
  std::vector<double> flat;
  if (per_layer.empty()) return flat;
  if (per_layer.size() != layers) throw ValidationError(std::string(what) + ": one entry per layer required");
  for (const auto& v : per_layer) {
    if (v.size() != n) throw ValidationError(std::string(what) + ": wrong row count");
    flat.insert(flat.end(), v.begin(), v.end());
  }
  return flat;
}

// segment_forward (toy_model.hpp:206): prefix_k / prefix_v per layer,
// prefix_len x kv_width (empty when prefix_len is 0).
inline SegmentTape segment_forward(const Model& model, const cf_model_cfg& cfg, const int32_t* tokens, int64_t len,
                                   const int64_t* targets, const std::vector<std::vector<double>>& prefix_k,
                                   const std::vector<std::vector<double>>& prefix_v, int64_t prefix_len,
                                   bool keep_tape) {
  const size_t L = static_cast<size_t>(cfg.num_layers);
  const size_t kvw = static_cast<size_t>(cfg.num_kv_heads * (cfg.d_model / cfg.num_heads));
  const std::vector<double> pk = flatten_kv(prefix_k, L, static_cast<size_t>(prefix_len) * kvw, "prefix_k");
  const std::vector<double> pv = flatten_kv(prefix_v, L, static_cast<size_t>(prefix_len) * kvw, "prefix_v");
  std::vector<double> sk(L * static_cast<size_t>(len) * kvw), sv(sk.size());
  SegmentTape t;
  t.len = len;
  t.prefix_len = prefix_len;
  cf_segment* h = nullptr;
  check(cf_segment_forward(model.device().get(), model.get(), tokens, len, targets, pk.empty() ? nullptr : pk.data(),
                           pv.empty() ? nullptr : pv.data(), prefix_len, keep_tape ? 1 : 0, &t.loss_sum, sk.data(),
                           sv.data(), &h));
  if (h) t.handle.reset(h, &cf_segment_destroy);
  const size_t per = static_cast<size_t>(len) * kvw;
  for (size_t l = 0; l < L; ++l) {
    t.saved_k.emplace_back(sk.begin() + l * per, sk.begin() + (l + 1) * per);
    t.saved_v.emplace_back(sv.begin() + l * per, sv.begin() + (l + 1) * per);
  }
  return t;
}

// segment_backward (toy_model.hpp:341): parameter gradients accumulate in
// the model's device buffer (the GradientSet); d_prefix_k / d_prefix_v are
// accumulated, incoming_dk / incoming_dv may be null.
inline void segment_backward(const Model& model, const cf_model_cfg& cfg, const SegmentTape& tape,
                             const std::vector<std::vector<double>>& prefix_k,
                             const std::vector<std::vector<double>>& prefix_v,
                             std::vector<std::vector<double>>* d_prefix_k, std::vector<std::vector<double>>* d_prefix_v,
                             const std::vector<std::vector<double>>* incoming_dk,
                             const std::vector<std::vector<double>>* incoming_dv, double normalizer) {
  if (!tape.handle) throw ValidationError("segment backward requires a retained tape");
  const size_t L = static_cast<size_t>(cfg.num_layers);
  const size_t kvw = static_cast<size_t>(cfg.num_kv_heads * (cfg.d_model / cfg.num_heads));
  const size_t np = static_cast<size_t>(tape.prefix_len) * kvw, nl = static_cast<size_t>(tape.len) * kvw;
  const std::vector<double> pk = flatten_kv(prefix_k, L, np, "prefix_k");
  const std::vector<double> pv = flatten_kv(prefix_v, L, np, "prefix_v");
  const std::vector<double> ik = incoming_dk ? flatten_kv(*incoming_dk, L, nl, "incoming_dk") : std::vector<double>{};
  const std::vector<double> iv = incoming_dv ? flatten_kv(*incoming_dv, L, nl, "incoming_dv") : std::vector<double>{};
  std::vector<double> dk(L * np, 0.0), dv(L * np, 0.0);
  check(cf_segment_backward(model.device().get(), model.get(), tape.handle.get(), pk.empty() ? nullptr : pk.data(),
                            pv.empty() ? nullptr : pv.data(), dk.data(), dv.data(), ik.empty() ? nullptr : ik.data(),
                            iv.empty() ? nullptr : iv.data(), normalizer));
  for (int kv = 0; kv < 2; ++kv) {
    std::vector<std::vector<double>>* out = kv ? d_prefix_v : d_prefix_k;
    const std::vector<double>& src = kv ? dv : dk;
    if (!out || np == 0) continue;
    if (out->empty()) out->assign(L, std::vector<double>(np, 0.0));
    for (size_t l = 0; l < L; ++l)
      for (size_t i = 0; i < np; ++i) (*out)[l][i] += src[l * np + i];
  }
}

}  // namespace detail

}  // namespace chunkflow_b200
