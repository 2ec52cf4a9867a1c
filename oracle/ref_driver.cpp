// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never
// measured as the product).
//
// Thin extern "C" shim that compiles the *unmodified* reference headers from
// /root/reference/proj/include (read in place, not copied) into
// oracle/_ref/libcfref.so, so tests can pin the CPU restatement
// (oracle/cf_oracle.cpp) and the B200 product against the reference itself.
// Built by oracle/Makefile; outputs only into oracle/_ref/.
#include <chunkflow/chunker.hpp>
#include <chunkflow/dataset.hpp>
#include <chunkflow/memory_model.hpp>
#include <chunkflow/pipeline.hpp>
#include <chunkflow/plan_runner.hpp>
#include <chunkflow/scheduler.hpp>
#include <chunkflow/tuner.hpp>
#include <chunkflow/toy_model.hpp>

#include <cstring>
#include <sstream>
#include <string>

#include "../include/chunkflow_b200.h"

namespace cf = chunkflow;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return CF_OK;
  } catch (const cf::ValidationError& e) {
    g_err = e.what();
    return CF_EVALIDATION;
  } catch (const cf::ParseError& e) {
    g_err = e.what();
    return CF_EPARSE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CF_EINTERNAL;
  }
}

cf::Batch make_batch(const int64_t* ids, const int64_t* lengths, int64_t n,
                     const int32_t* tokens) {
  cf::Batch b;
  int64_t off = 0;
  for (int64_t i = 0; i < n; ++i) {
    cf::SequenceRecord r;
    r.id = ids[i];
    r.length = lengths[i];
    if (tokens) r.tokens.assign(tokens + off, tokens + off + lengths[i]);
    off += lengths[i];
    b.sequences.push_back(std::move(r));
  }
  b.global_batch_size = n;
  return b;
}

cf::ToyModelConfig toy_cfg(const cf_model_cfg* c) {
  cf::ToyModelConfig t;
  t.vocab_size = c->vocab_size;
  t.d_model = c->d_model;
  t.num_heads = c->num_heads;
  t.num_kv_heads = c->num_kv_heads;
  t.num_layers = c->num_layers;
  t.seed = c->seed;
  return t;
}

void export_events(const cf::ExecutionPlan& plan, cf_event_rec* ev,
                   int64_t cap, int64_t* n_events, cf_plan_diag* diag) {
  const int64_t n = static_cast<int64_t>(plan.events.size());
  if (n > cap) throw cf::ValidationError("event buffer too small");
  for (int64_t i = 0; i < n; ++i) {
    const cf::ExecEvent& e = plan.events[i];
    ev[i].kind = static_cast<int64_t>(e.kind);
    ev[i].chunk_id = e.chunk_id;
    ev[i].group_id = e.group_id;
    ev[i].index_in_group = e.index_in_group;
    ev[i].is_recompute = e.is_recompute;
    ev[i].save_kv = e.notes.save_kv;
    ev[i].read_kv_prefix = e.notes.read_kv_prefix;
    ev[i].accumulate_kv_grad = e.notes.accumulate_kv_grad;
  }
  *n_events = n;
  if (diag) {
    const cf::PlanDiagnostics d = cf::validate_plan(plan);
    diag->peak_retained_tokens = d.peak_retained_tokens;
    diag->recompute_token_count = d.recompute_token_count;
    diag->num_violations = static_cast<int64_t>(d.violations.size());
  }
}

void flatten(const cf::GradientSet& g, double* out) {
  int64_t off = 0;
  for (const cf::Tensor& t : g.tensors) {
    std::memcpy(out + off, t.data.data(), sizeof(double) * t.data.size());
    off += static_cast<int64_t>(t.data.size());
  }
}
}  // namespace

extern "C" {

const char* cfr_last_error(void) { return g_err.c_str(); }

int cfr_construct_chunks(const int64_t* ids, const int64_t* lengths, int64_t n,
                         int64_t cs, cf_chunk_rec* chunks, int64_t cap_c,
                         cf_segment_rec* segs, int64_t cap_s,
                         int64_t* n_chunks, int64_t* n_segs) {
  return guarded([&] {
    const cf::ChunkPlan p = cf::construct_chunks(make_batch(ids, lengths, n, nullptr), cs);
    int64_t si = 0;
    if (static_cast<int64_t>(p.chunks.size()) > cap_c) throw cf::ValidationError("chunk buffer too small");
    for (size_t c = 0; c < p.chunks.size(); ++c) {
      const cf::Chunk& ch = p.chunks[c];
      chunks[c] = {ch.chunk_id, static_cast<int64_t>(ch.kind), ch.group_id,
                   ch.index_in_group, ch.total_tokens, si,
                   static_cast<int64_t>(ch.segments.size())};
      for (const cf::ChunkSegment& s : ch.segments) {
        if (si >= cap_s) throw cf::ValidationError("segment buffer too small");
        segs[si++] = {s.sequence_id, s.start_token, s.length};
      }
    }
    *n_chunks = static_cast<int64_t>(p.chunks.size());
    *n_segs = si;
  });
}

int cfr_schedule_step(const int64_t* ids, const int64_t* lengths, int64_t n,
                      int64_t cs, int64_t k, cf_event_rec* ev, int64_t cap,
                      int64_t* n_events, cf_plan_diag* diag) {
  return guarded([&] {
    const cf::ChunkPlan p = cf::construct_chunks(make_batch(ids, lengths, n, nullptr), cs);
    export_events(cf::schedule_step(p, k), ev, cap, n_events, diag);
  });
}

int cfr_schedule_group(int64_t n, int64_t k, int64_t cs, cf_event_rec* ev,
                       int64_t cap, int64_t* n_events, cf_plan_diag* diag) {
  return guarded([&] { export_events(cf::schedule_group(n, k, cs), ev, cap, n_events, diag); });
}

int cfr_listing(const int64_t* ids, const int64_t* lengths, int64_t n,
                int64_t cs, int64_t k, char* buf, int64_t cap) {
  return guarded([&] {
    const cf::ChunkPlan p = cf::construct_chunks(make_batch(ids, lengths, n, nullptr), cs);
    const std::string s = cf::execution_plan_listing(cf::schedule_step(p, k));
    if (static_cast<int64_t>(s.size()) + 1 > cap) throw cf::ValidationError("listing buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// synthesize (dataset.hpp:207) with explicit buckets; preset 1 = Table 5.
int cfr_synthesize(const int64_t* bounds, const double* fracs, int64_t nb,
                   int64_t max_length, int64_t preset, int64_t count,
                   uint64_t seed, int64_t* lengths_out) {
  return guarded([&] {
    cf::DistributionSpec spec;
    if (preset == 1) {
      spec = cf::eval_table5_spec();
    } else if (preset == 2) {
      spec = cf::lmsys_table2_spec();
    } else {
      for (int64_t i = 0; i < nb; ++i) spec.buckets.push_back({bounds[i], fracs[i]});
      spec.max_length = max_length;
    }
    const cf::SequenceSet s = cf::synthesize(spec, count, seed);
    for (int64_t i = 0; i < count; ++i) lengths_out[i] = s[i].length;
  });
}

int cfr_sample_batch(const int64_t* lengths, int64_t n, int64_t gbs,
                     int64_t step, uint64_t seed, int64_t* ids_out,
                     int64_t* count_out) {
  return guarded([&] {
    cf::SequenceSet set;
    for (int64_t i = 0; i < n; ++i) {
      cf::SequenceRecord r;
      r.id = i;
      r.length = lengths[i];
      set.push_back(r);
    }
    const auto b = cf::sample_batch(set, gbs, step, seed);
    *count_out = 0;
    if (!b) return;
    for (const auto& r : b->sequences) ids_out[(*count_out)++] = r.id;
  });
}

int64_t cfr_toy_num_params(const cf_model_cfg* c) {
  const cf::ToyModelParams p = cf::init_model(toy_cfg(c));
  int64_t total = 0;
  for (const auto& t : p.tensors) total += t.size();
  return total;
}

int cfr_toy_init(const cf_model_cfg* c, double* out) {
  return guarded([&] {
    const cf::ToyModelParams p = cf::init_model(toy_cfg(c));
    int64_t off = 0;
    for (const auto& t : p.tensors) {
      std::memcpy(out + off, t.data.data(), sizeof(double) * t.data.size());
      off += t.size();
    }
  });
}

// run_plan (plan_runner.hpp:67) on the toy model; instr = {peak_retained,
// recompute_forwards, recompute_loss_mismatches, kv_completeness_violations}.
int cfr_run_plan(const cf_model_cfg* c, const int64_t* ids,
                 const int64_t* lengths, const int32_t* tokens, int64_t n,
                 int64_t cs, int64_t k, int corrupt, double* loss,
                 double* grads, int64_t* instr) {
  return guarded([&] {
    const cf::ToyModelParams params = cf::init_model(toy_cfg(c));
    const cf::Batch b = make_batch(ids, lengths, n, tokens);
    const cf::ChunkPlan cp = cf::construct_chunks(b, cs);
    const cf::ExecutionPlan ep = cf::schedule_step(cp, k);
    cf::RunPlanOptions o;
    o.corrupt_kv_grads = corrupt != 0;
    const cf::RunPlanResult r = cf::run_plan(params, cp, ep, b.sequences, o);
    *loss = r.loss;
    if (grads) flatten(r.gradients, grads);
    instr[0] = r.instrumentation.peak_retained_tokens;
    instr[1] = r.instrumentation.recompute_forward_count;
    instr[2] = r.instrumentation.recompute_loss_mismatches;
    instr[3] = r.instrumentation.kv_completeness_violations;
  });
}

int cfr_backward_full(const cf_model_cfg* c, const int64_t* ids,
                      const int64_t* lengths, const int32_t* tokens, int64_t n,
                      double* loss, double* grads) {
  return guarded([&] {
    const cf::ToyModelParams params = cf::init_model(toy_cfg(c));
    const cf::Batch b = make_batch(ids, lengths, n, tokens);
    const cf::GradientSet g = cf::backward_full(params, b.sequences);
    *loss = g.loss;
    if (grads) flatten(g, grads);
  });
}

// verify_equivalence (plan_runner.hpp:368); out = {loss_rel, max_rel}.
int cfr_verify(const cf_model_cfg* c, const int64_t* ids,
               const int64_t* lengths, const int32_t* tokens, int64_t n,
               int64_t cs, int64_t k, int corrupt, double* out, int* pass) {
  return guarded([&] {
    const cf::ToyModelParams params = cf::init_model(toy_cfg(c));
    const cf::Batch b = make_batch(ids, lengths, n, tokens);
    cf::RunPlanOptions o;
    o.corrupt_kv_grads = corrupt != 0;
    const cf::VerifyReport r = cf::verify_equivalence(params, b.sequences, cs, k, 1e-12, 1e-9, o);
    out[0] = r.loss_rel_err;
    out[1] = r.max_grad_rel_err;
    *pass = r.pass ? 1 : 0;
  });
}

// simulate_state_aware_1f1b / simulate_1f1b + bubble_ratio (pipeline.hpp).
// mode 0 = plain 1F1B on whole sequences; 1 = state-aware on the chunk plan.
int cfr_simulate(const int64_t* ids, const int64_t* lengths, int64_t n,
                 int64_t cs, int64_t k, int64_t stages, double alpha,
                 double beta, double gamma, double hop, int mode,
                 double* makespan, double* bubble) {
  return guarded([&] {
    cf::CostModel cm;
    cm.alpha = alpha;
    cm.beta = beta;
    cm.gamma = gamma;
    cm.hop_latency = hop;
    cf::PipelineTrace tr;
    if (mode == 0) {
      std::vector<std::int64_t> lens(lengths, lengths + n);
      tr = cf::simulate_1f1b(lens, static_cast<int>(stages), cm);
    } else {
      const cf::ChunkPlan cp = cf::construct_chunks(make_batch(ids, lengths, n, nullptr), cs);
      cf::PipelineConfig pc;
      pc.num_stages = static_cast<int>(stages);
      pc.k = k;
      pc.chunk_size = cs;
      tr = cf::simulate_state_aware_1f1b(cp, pc, cm);
    }
    *makespan = tr.makespan;
    *bubble = cf::bubble_ratio(tr);
  });
}

}  // extern "C"

extern "C" {
// Full trace export of the reference simulator (pipeline.hpp): per stage the
// dispatched ops (kind, chunk id, start, end), stage-major; busy/busy_total
// per stage.  mode 0 = simulate_1f1b, 1 = simulate_state_aware_1f1b.
// Returns ops per stage through *per (call with ops = NULL to size).
int cfr_pp_trace(const int64_t* ids, const int64_t* lengths, int64_t n, int64_t cs, int64_t k, int64_t stages,
                 const double* cost5, int mode, int backward_first, double* ops, int64_t* per, double* busy,
                 double* busy_total, double* makespan, double* bubble) {
  return guarded([&] {
    cf::CostModel cm;
    cm.gamma = cost5[0];
    cm.alpha = cost5[1];
    cm.beta = cost5[2];
    cm.backward_multiplier = cost5[3];
    cm.hop_latency = cost5[4];
    cf::PipelineTrace tr;
    if (mode == 0) {
      std::vector<std::int64_t> lens(lengths, lengths + n);
      tr = cf::simulate_1f1b(lens, static_cast<int>(stages), cm);
    } else {
      const cf::ChunkPlan cp = cf::construct_chunks(make_batch(ids, lengths, n, nullptr), cs);
      cf::PipelineConfig pc;
      pc.num_stages = static_cast<int>(stages);
      pc.k = k;
      pc.chunk_size = cs;
      tr = cf::simulate_state_aware_1f1b(cp, pc, cm,
                                         backward_first ? cf::DispatchPolicy::kBackwardFirst
                                                        : cf::DispatchPolicy::kForwardFirst);
    }
    *per = static_cast<int64_t>(tr.stages[0].size());
    for (size_t s = 0; s < tr.stages.size(); ++s) {
      if (busy) busy[s] = tr.busy[s];
      if (busy_total) busy_total[s] = tr.busy_total[s];
      if (ops)
        for (size_t i = 0; i < tr.stages[s].size(); ++i) {
          double* o = ops + 4 * (s * static_cast<size_t>(*per) + i);
          const cf::TraceEvent& e = tr.stages[s][i];
          o[0] = static_cast<double>(static_cast<int>(e.kind));
          o[1] = static_cast<double>(e.chunk_id);
          o[2] = e.start;
          o[3] = e.end;
        }
    }
    *makespan = tr.makespan;
    *bubble = cf::bubble_ratio(tr);
  });
}
}  // extern "C"

// ---- wire formats + memory model of the reference (chunker.hpp:233-292,
//      scheduler.hpp:300-328, dataset.hpp:112-176, memory_model.hpp)
namespace {
void put(const std::string& s, char* buf, size_t cap, size_t* len) {
  *len = s.size();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
}
}  // namespace

extern "C" {
// which: 0 = chunk_plan.json of `pack`, 1 = execution_plan.json of `schedule`
int cfr_plan_json(const int64_t* ids, const int64_t* lengths, int64_t n, int64_t cs, int64_t k, int which,
                  char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    const cf::ChunkPlan p = cf::construct_chunks(make_batch(ids, lengths, n, nullptr), cs);
    if (which == 0) {
      put(cf::chunk_plan_to_json(p).dump(2) + "\n", buf, cap, len);
    } else {
      put(cf::execution_plan_to_json(cf::schedule_step(p, k)).dump(2) + "\n", buf, cap, len);
    }
  });
}
// `schedule` on a chunk-plan document: chunk_plan_from_json -> schedule_step -> execution_plan.json
int cfr_schedule_json(const char* doc, int64_t k, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(doc);
    } catch (const nlohmann::json::exception& e) {
      throw cf::ParseError(e.what());
    }
    put(cf::execution_plan_to_json(cf::schedule_step(cf::chunk_plan_from_json(j), k)).dump(2) + "\n", buf, cap,
        len);
  });
}
// load_lengths -> write_records round trip (the canonical JSONL of a file)
int cfr_jsonl_roundtrip(const char* text, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    std::istringstream in(text);
    std::ostringstream out;
    cf::write_records(out, cf::load_lengths(in));
    put(out.str(), buf, cap, len);
  });
}
int cfr_calibrate(const char* csv, double gqa, double* coeffs4, double* max_resid, char* buf, size_t cap,
                  size_t* len) {
  return guarded([&] {
    std::istringstream in(csv);
    const cf::CalibrationResult r = cf::calibrate(cf::parse_measurements(in), gqa);
    coeffs4[0] = r.coefficients.base;
    coeffs4[1] = r.coefficients.per_chunk_token;
    coeffs4[2] = r.coefficients.per_context_token;
    coeffs4[3] = r.coefficients.gqa_ratio;
    *max_resid = r.max_residual_gib;
    put(cf::coefficients_to_json(r.coefficients).dump(2) + "\n", buf, cap, len);
  });
}
}  // extern "C"

extern "C" int cfr_export_trace(const int64_t* ids, const int64_t* lengths, int64_t n, int64_t cs, int64_t k,
                                int64_t stages, const double* cost5, int mode, int format, char* buf, size_t cap,
                                size_t* len) {
  return guarded([&] {
    cf::CostModel cm;
    cm.gamma = cost5[0];
    cm.alpha = cost5[1];
    cm.beta = cost5[2];
    cm.backward_multiplier = cost5[3];
    cm.hop_latency = cost5[4];
    cf::PipelineTrace tr;
    if (mode == 0) {
      tr = cf::simulate_1f1b(std::vector<std::int64_t>(lengths, lengths + n), static_cast<int>(stages), cm);
    } else {
      cf::PipelineConfig pc;
      pc.num_stages = static_cast<int>(stages);
      pc.k = k;
      tr = cf::simulate_state_aware_1f1b(cf::construct_chunks(make_batch(ids, lengths, n, nullptr), cs), pc, cm);
    }
    put(cf::export_trace(tr, format == 0 ? cf::TraceFormat::kChromeTrace : cf::TraceFormat::kTable), buf, cap, len);
  });
}

// grid_search + its CSV table and ranked report (tuner.hpp)
extern "C" int cfr_tune(const int64_t* ids, const int64_t* lengths, int64_t n, const int64_t* css, int64_t ncs,
                        const int64_t* ks, int64_t nk, int64_t stages, const double* cost5, const double* mem4,
                        double budget, int64_t gbs, int64_t nb, uint64_t seed, int csv, char* buf, size_t cap,
                        size_t* len) {
  return guarded([&] {
    cf::SequenceSet set = make_batch(ids, lengths, n, nullptr).sequences;
    cf::PipelineConfig pc;
    pc.num_stages = static_cast<int>(stages);
    cf::CostModel cm;
    cm.gamma = cost5[0];
    cm.alpha = cost5[1];
    cm.beta = cost5[2];
    cm.backward_multiplier = cost5[3];
    cm.hop_latency = cost5[4];
    cf::MemoryModelCoefficients mc;
    mc.base = mem4[0];
    mc.per_chunk_token = mem4[1];
    mc.per_context_token = mem4[2];
    mc.gqa_ratio = mem4[3];
    const cf::TunerResult r = cf::grid_search(set, std::vector<std::int64_t>(css, css + ncs),
                                              std::vector<std::int64_t>(ks, ks + nk), pc, cm, mc, budget, gbs, nb,
                                              seed);
    put(csv ? cf::tuner_table_csv(r) : cf::tuner_report(r), buf, cap, len);
  });
}

// validate_plan (scheduler.hpp:182) over a caller-built ExecutionPlan:
// groups in CSR form, chunk_tokens as parallel arrays.  Writes peak / recompute
// tokens and the violation texts joined by '\n' (for pinning
// cf_plan_validate_events' texts against the reference verbatim).
extern "C" int cfr_validate_events(int64_t chunk_size, int64_t k, const cf_event_rec* ev, int64_t n_ev,
                                   const int64_t* gids, const int64_t* goff, const int64_t* mem, int64_t ng,
                                   const int64_t* tc, const int64_t* tn, int64_t nt, int64_t* peak,
                                   int64_t* recompute, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    cf::ExecutionPlan p;
    p.chunk_size = chunk_size;
    p.k = k;
    for (int64_t g = 0; g < ng; ++g) p.groups[gids[g]] = std::vector<int64_t>(mem + goff[g], mem + goff[g + 1]);
    for (int64_t i = 0; i < nt; ++i) p.chunk_tokens[tc[i]] = tn[i];
    for (int64_t i = 0; i < n_ev; ++i) {
      cf::ExecEvent e;
      e.kind = static_cast<cf::ExecKind>(ev[i].kind);
      e.chunk_id = ev[i].chunk_id;
      e.group_id = ev[i].group_id;
      e.index_in_group = ev[i].index_in_group;
      e.is_recompute = ev[i].is_recompute != 0;
      e.notes.save_kv = ev[i].save_kv != 0;
      e.notes.read_kv_prefix = ev[i].read_kv_prefix != 0;
      e.notes.accumulate_kv_grad = ev[i].accumulate_kv_grad != 0;
      p.events.push_back(e);
    }
    const cf::PlanDiagnostics d = cf::validate_plan(p);
    *peak = d.peak_retained_tokens;
    *recompute = d.recompute_token_count;
    std::string s;
    for (const std::string& v : d.violations) s += v + "\n";
    *len = s.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}
