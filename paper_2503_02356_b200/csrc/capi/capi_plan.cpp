// C-ABI: errors + planning entry points (include/chunkflow_b200.h).
#include <cstring>
#include <memory>
#include <string>

#include "../../../include/chunkflow_b200.h"
#include "../host/plan.hpp"
#include "../host/pp.hpp"
#include "../host/wire.hpp"
#include "capi_util.hpp"

namespace cfb {
thread_local std::string g_last_error;
}

extern "C" {

const char* cf_last_error(void) { return cfb::g_last_error.c_str(); }
const char* cf_version(void) { return "chunkflow_b200 0.1 (sm_100a)"; }

int cf_plan_build(const int64_t* seq_ids, const int64_t* lengths, int64_t n, int64_t chunk_size, int64_t k,
                  cf_plan** out) {
  return cfb::guard([&] {
    if (n < 0 || (n > 0 && (!seq_ids || !lengths))) throw cfb::ValidationError("bad batch arrays");
    for (int64_t i = 0; i < n; ++i)
      if (lengths[i] < 1) throw cfb::ValidationError("sequence lengths must be positive");
    auto h = std::make_unique<cf_plan>();
    h->p = cfb::construct_chunks(seq_ids, lengths, n, chunk_size);
    cfb::schedule_step(h->p, k);
    *out = h.release();
  });
}

int cf_plan_build_group(int64_t n, int64_t k, int64_t chunk_size, cf_plan** out) {
  return cfb::guard([&] {
    auto h = std::make_unique<cf_plan>();
    h->p = cfb::schedule_group(n, k, chunk_size);
    *out = h.release();
  });
}

int cf_plan_validate_events(int64_t chunk_size, int64_t k, const cf_event_rec* events, int64_t n_events,
                            const int64_t* group_ids, const int64_t* group_offsets, const int64_t* members,
                            int64_t n_groups, const int64_t* token_chunk_ids, const int64_t* token_counts,
                            int64_t n_token_entries, const cf_plan* chunk_plan, cf_plan** out) {
  return cfb::guard([&] {
    if (!out) throw cfb::ValidationError("out is null");
    if (n_events < 0 || n_groups < 0 || n_token_entries < 0) throw cfb::ValidationError("negative count");
    if ((n_events && !events) || (n_groups && (!group_ids || !group_offsets || !members)) ||
        (n_token_entries && (!token_chunk_ids || !token_counts)))
      throw cfb::ValidationError("null array with a non-zero count");
    auto h = std::make_unique<cf_plan>();
    cfb::Plan& p = h->p;
    if (chunk_plan) {  // the chunks the events refer to, so the result can be executed
      p.chunks = chunk_plan->p.chunks;
      p.segments = chunk_plan->p.segments;
      p.index_of = chunk_plan->p.index_of;
      p.chunk_tokens = chunk_plan->p.chunk_tokens;
    }
    p.chunk_size = chunk_size;
    p.k = k;
    for (int64_t g = 0; g < n_groups; ++g) {
      if (group_offsets[g] < 0 || group_offsets[g + 1] < group_offsets[g])
        throw cfb::ValidationError("group offsets must be non-decreasing");
      p.groups[group_ids[g]] = std::vector<int64_t>(members + group_offsets[g], members + group_offsets[g + 1]);
    }
    for (int64_t i = 0; i < n_token_entries; ++i) p.chunk_tokens[token_chunk_ids[i]] = token_counts[i];
    for (int64_t i = 0; i < n_events; ++i) {
      const cf_event_rec& e = events[i];
      if (e.kind < CF_EXEC_FORWARD_DISCARD || e.kind > CF_EXEC_BACKWARD)
        throw cfb::ValidationError("unknown event kind " + std::to_string(e.kind));
      p.events.push_back({e.kind, e.chunk_id, e.group_id, e.index_in_group, e.is_recompute != 0, e.save_kv != 0,
                          e.read_kv_prefix != 0, e.accumulate_kv_grad != 0});
    }
    cfb::validate(p);
    *out = h.release();
  });
}

int cf_plan_counts(const cf_plan* plan, int64_t* n_chunks, int64_t* n_segments, int64_t* n_events,
                   int64_t* n_groups) {
  return cfb::guard([&] {
    if (n_chunks) *n_chunks = static_cast<int64_t>(plan->p.chunks.size());
    if (n_segments) *n_segments = static_cast<int64_t>(plan->p.segments.size());
    if (n_events) *n_events = static_cast<int64_t>(plan->p.events.size());
    if (n_groups) *n_groups = static_cast<int64_t>(plan->p.groups.size());
  });
}

int cf_plan_export(const cf_plan* plan, cf_chunk_rec* chunks, cf_segment_rec* segments, cf_event_rec* events,
                   cf_plan_diag* diag) {
  return cfb::guard([&] {
    const cfb::Plan& p = plan->p;
    if (chunks)
      for (size_t i = 0; i < p.chunks.size(); ++i) {
        const cfb::Chunk& c = p.chunks[i];
        chunks[i] = {c.id, c.kind, c.group, c.index, c.total, c.seg_off, c.seg_cnt};
      }
    if (segments)
      for (size_t i = 0; i < p.segments.size(); ++i)
        segments[i] = {p.segments[i].seq, p.segments[i].start, p.segments[i].len};
    if (events)
      for (size_t i = 0; i < p.events.size(); ++i) {
        const cfb::Event& e = p.events[i];
        events[i] = {e.kind, e.chunk, e.group, e.index, e.recompute, e.save_kv, e.read_prefix, e.acc_grad};
      }
    if (diag) *diag = {p.peak_retained, p.recompute_tokens, static_cast<int64_t>(p.violations.size())};
  });
}

int cf_plan_export_groups(const cf_plan* plan, int64_t* group_ids, int64_t* offsets, int64_t* members) {
  return cfb::guard([&] {
    if (!plan || !offsets) throw cfb::ValidationError("plan and offsets are required");
    int64_t g = 0, m = 0;
    offsets[0] = 0;
    for (const auto& [gid, mem] : plan->p.groups) {  // group_ids / members may be NULL (sizing call)
      if (group_ids) group_ids[g] = gid;
      for (int64_t c : mem) {
        if (members) members[m] = c;
        ++m;
      }
      offsets[++g] = m;
    }
  });
}

int cf_plan_violation(const cf_plan* plan, int64_t i, char* buf, size_t cap) {
  return cfb::guard([&] {
    if (i < 0 || i >= static_cast<int64_t>(plan->p.violations.size())) throw cfb::ValidationError("violation index");
    const std::string& s = plan->p.violations[static_cast<size_t>(i)];
    if (cap == 0) return;
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  });
}

int cf_plan_listing(const cf_plan* plan, char* buf, size_t cap, size_t* len) {
  return cfb::guard([&] {
    const std::string s = cfb::listing(plan->p);
    if (len) *len = s.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

int cf_plan_partition(const cf_plan* global, int64_t world, int64_t rank, cf_plan** out) {
  return cfb::guard([&] {
    if (rank < 0 || rank >= world) throw cfb::ValidationError("rank out of range");
    const auto units = cfb::plan_units(global->p, 1.0, cfb::kPairWeight);
    const auto assign = cfb::lpt_assign(units, world);
    auto h = std::make_unique<cf_plan>();
    h->p = cfb::sub_plan(global->p, units, assign[static_cast<size_t>(rank)], global->p.k);
    *out = h.release();
  });
}

int cf_plan_rank_tokens(const cf_plan* global, int64_t world, int64_t* tokens) {
  return cfb::guard([&] {
    const auto units = cfb::plan_units(global->p, 1.0, cfb::kPairWeight);
    const auto assign = cfb::lpt_assign(units, world);
    for (int64_t r = 0; r < world; ++r) {
      tokens[r] = 0;
      for (int64_t u : assign[static_cast<size_t>(r)]) tokens[r] += units[static_cast<size_t>(u)].tokens;
    }
  });
}

void cf_plan_destroy(cf_plan* plan) { delete plan; }

int cf_synthesize(const int64_t* bounds, const double* fracs, int64_t nb, int64_t max_length, int64_t preset,
                  int64_t count, uint64_t seed, int64_t* lengths_out) {
  return cfb::guard([&] {
    std::vector<int64_t> b;
    std::vector<double> f;
    int64_t mx = max_length;
    if (preset == 1) {
      b = {1024, 4096, 8192, 32768, 131072};
      f = {0.9817, 0.9972, 0.9983, 0.9992, 0.9998};
      mx = 262144;
    } else if (preset == 2) {
      b = {1024, 4096, 8192, 32768, 131072};
      f = {0.90499, 0.99539, 0.99908, 0.99987, 0.99996};
      mx = 303 * 1024;
    } else {
      b.assign(bounds, bounds + nb);
      f.assign(fracs, fracs + nb);
    }
    const auto v = cfb::synthesize(b, f, mx, count, seed);
    std::copy(v.begin(), v.end(), lengths_out);
  });
}

int cf_sample_batch(int64_t n, int64_t global_batch, int64_t step, uint64_t seed, int64_t* idx_out,
                    int64_t* count_out) {
  return cfb::guard([&] {
    const auto v = cfb::sample_batch(n, global_batch, step, seed);
    std::copy(v.begin(), v.end(), idx_out);
    *count_out = static_cast<int64_t>(v.size());
  });
}

int cf_gen_tokens(const int64_t* lengths, int64_t n, int64_t vocab, uint64_t seed, int32_t* tokens_out) {
  return cfb::guard([&] {
    if (vocab < 1) throw cfb::ValidationError("vocab must be positive");
    uint64_t s = seed;
    int64_t o = 0;
    const uint64_t v = static_cast<uint64_t>(vocab);
    const uint64_t thr = (0 - v) % v;  // next_below rejection (common.hpp:52-58)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t t = 0; t < lengths[i]; ++t) {
        uint64_t r;
        do r = cfb::splitmix_next(s);
        while (r < thr);
        tokens_out[o++] = static_cast<int32_t>(r % v);
      }
  });
}

}  // extern "C"

// ---------------------------------------------------------------- pipeline
namespace {

cfb::PpCost to_cost(const cf_pp_cost* c) {
  cfb::PpCost pc;
  if (c) {
    pc.gamma = c->gamma;
    pc.alpha = c->alpha;
    pc.beta = c->beta;
    pc.bwd_mult = c->backward_multiplier;
    pc.hop = c->hop_latency;
  }
  return pc;
}

void emit(const cfb::PpChunks& info, const cfb::PpTrace& tr, cf_pp_op* ops, double* busy, double* busy_total,
          cf_pp_result* res) {
  const size_t per = tr.stages.empty() ? 0 : tr.stages[0].size();
  for (size_t s = 0; s < tr.stages.size(); ++s) {
    if (tr.stages[s].size() != per) throw std::logic_error("stages ran different op counts");
    if (busy) busy[s] = tr.busy[s];
    if (busy_total) busy_total[s] = tr.busy_total[s];
    if (ops)
      for (size_t i = 0; i < per; ++i) {
        const cfb::PpTimedOp& o = tr.stages[s][i];
        ops[s * per + i] = {o.kind, info.ids[static_cast<size_t>(o.pos)], o.start, o.end};
      }
  }
  if (res) {
    res->makespan = tr.makespan;
    res->bubble_ratio = cfb::pp_bubble(tr);
    double idle = 0;
    for (double b : tr.busy_total) idle += tr.makespan - b;
    res->occupancy_bubble = tr.makespan > 0 ? idle / (static_cast<double>(tr.stages.size()) * tr.makespan) : 0.0;
    res->ops_per_stage = static_cast<int64_t>(per);
  }
}

}  // namespace

extern "C" {

int cf_pp_simulate(const cf_plan* plan, int64_t num_stages, int64_t k, const cf_pp_cost* cost, int backward_first,
                   const double* fwd_cost, const double* bwd_cost, cf_pp_op* ops, double* busy, double* busy_total,
                   cf_pp_result* result) {
  return cfb::guard([&] {
    if (num_stages < 1) throw cfb::ValidationError("num_stages must be at least 1");
    cfb::PpChunks info = cfb::pp_chunks(plan->p, k, to_cost(cost));
    for (size_t i = 0; i < info.fwd.size(); ++i) {
      if (fwd_cost) info.fwd[i] = fwd_cost[i];
      if (bwd_cost) info.bwd[i] = bwd_cost[i];
      if (info.fwd[i] < 0 || info.bwd[i] < 0) throw cfb::ValidationError("measured costs must be non-negative");
    }
    std::vector<std::vector<cfb::PpOp>> orders;
    for (int64_t s = 0; s < num_stages; ++s)
      orders.push_back(cfb::pp_stage_order(info, s, num_stages, backward_first != 0));
    emit(info, cfb::pp_dispatch(orders, info.fwd, info.bwd, to_cost(cost).hop), ops, busy, busy_total, result);
  });
}

int cf_pp_simulate_budget(const cf_plan* plan, int64_t num_stages, int64_t k, const cf_pp_cost* cost,
                          int backward_first, const double* fwd_cost, const double* bwd_cost, int64_t tape_budget,
                          cf_pp_op* ops, double* busy, double* busy_total, cf_pp_result* result) {
  return cfb::guard([&] {
    if (num_stages < 1) throw cfb::ValidationError("num_stages must be at least 1");
    if (tape_budget < 0) throw cfb::ValidationError("tape budget must be non-negative");
    cfb::PpChunks info = cfb::pp_chunks(plan->p, k, to_cost(cost));
    for (size_t i = 0; i < info.fwd.size(); ++i) {
      if (fwd_cost) info.fwd[i] = fwd_cost[i];
      if (bwd_cost) info.bwd[i] = bwd_cost[i];
      if (info.fwd[i] < 0 || info.bwd[i] < 0) throw cfb::ValidationError("measured costs must be non-negative");
    }
    std::vector<int64_t> tok;
    for (const cfb::Chunk& c : plan->p.chunks) tok.push_back(c.total);
    std::vector<std::vector<cfb::PpOp>> orders;
    std::vector<std::vector<double>> extra;
    for (int64_t s = 0; s < num_stages; ++s) {
      orders.push_back(cfb::pp_stage_order(info, s, num_stages, backward_first != 0));
      const cfb::PpStageMem m = cfb::pp_stage_memory(info, orders.back(), tok, tape_budget, s == 0);
      std::vector<double> e(info.fwd.size(), 0.0);
      for (size_t p = 0; p < e.size(); ++p)
        if (m.ckpt[p]) e[p] = info.fwd[p];
      extra.push_back(std::move(e));
    }
    emit(info, cfb::pp_dispatch(orders, info.fwd, info.bwd, to_cost(cost).hop, &extra), ops, busy, busy_total,
         result);
  });
}

int cf_pp_simulate_1f1b(const int64_t* lengths, int64_t n, int64_t num_stages, const cf_pp_cost* cost,
                        cf_pp_op* ops, double* busy, double* busy_total, cf_pp_result* result) {
  return cfb::guard([&] {
    if (num_stages < 1) throw cfb::ValidationError("num_stages must be at least 1");
    const cfb::PpChunks info = cfb::pp_microbatches(std::vector<int64_t>(lengths, lengths + n), to_cost(cost));
    std::vector<std::vector<cfb::PpOp>> orders;
    for (int64_t s = 0; s < num_stages; ++s) orders.push_back(cfb::pp_stage_order(info, s, num_stages, false));
    emit(info, cfb::pp_dispatch(orders, info.fwd, info.bwd, to_cost(cost).hop), ops, busy, busy_total, result);
  });
}

int cf_pp_stage_layers(int64_t num_layers, int64_t stage, int64_t num_stages, int64_t* begin, int64_t* end) {
  return cfb::guard([&] { cfb::pp_stage_layers(num_layers, stage, num_stages, begin, end); });
}

}  // extern "C"

// ---------------------------------------------------------- wire formats
namespace {
void put_text(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
}
cfb::MemCoeffs from_c(const cf_mem_coeffs* c) {
  return {c->base_gib, c->per_chunk_token_gib, c->per_context_token_gib, c->gqa_ratio};
}
}  // namespace

extern "C" {

int cf_plan_chunk_json(const cf_plan* plan, char* buf, size_t cap, size_t* len) {
  return cfb::guard([&] { put_text(cfb::chunk_plan_to_json(plan->p).dump(2) + "\n", buf, cap, len); });
}

int cf_plan_exec_json(const cf_plan* plan, char* buf, size_t cap, size_t* len) {
  return cfb::guard([&] { put_text(cfb::execution_plan_to_json(plan->p).dump(2) + "\n", buf, cap, len); });
}

int cf_plan_from_chunk_json(const char* json, int64_t k, cf_plan** out) {
  return cfb::guard([&] {
    if (!json || !out) throw cfb::ValidationError("null argument");
    auto h = std::make_unique<cf_plan>();
    h->p = cfb::chunk_plan_from_json(cfb::Json::parse(json));
    cfb::schedule_step(h->p, k);
    *out = h.release();
  });
}

int cf_dataset_load_jsonl(const char* text, int64_t* n, int64_t* ids, int64_t* lengths, int64_t* has_tokens,
                          int64_t* n_tokens, int32_t* tokens) {
  return cfb::guard([&] {
    if (!text || !n) throw cfb::ValidationError("null argument");
    const std::vector<cfb::SeqRecord> recs = cfb::load_lengths(text);
    *n = static_cast<int64_t>(recs.size());
    int64_t nt = 0;
    for (size_t i = 0; i < recs.size(); ++i) {
      if (ids) ids[i] = recs[i].id;
      if (lengths) lengths[i] = recs[i].length;
      if (has_tokens) has_tokens[i] = recs[i].tokens.empty() ? 0 : 1;
      if (tokens) std::copy(recs[i].tokens.begin(), recs[i].tokens.end(), tokens + nt);
      nt += static_cast<int64_t>(recs[i].tokens.size());
    }
    if (n_tokens) *n_tokens = nt;
  });
}

int cf_dataset_write_jsonl(const int64_t* ids, const int64_t* lengths, const int32_t* tokens, int64_t n, char* buf,
                           size_t cap, size_t* len) {
  return cfb::guard([&] {
    std::vector<cfb::SeqRecord> recs(static_cast<size_t>(n));
    int64_t off = 0;
    for (int64_t i = 0; i < n; ++i) {
      recs[static_cast<size_t>(i)].id = ids[i];
      recs[static_cast<size_t>(i)].length = lengths[i];
      if (tokens) {
        recs[static_cast<size_t>(i)].tokens.assign(tokens + off, tokens + off + lengths[i]);
        off += lengths[i];
      }
    }
    put_text(cfb::write_records(recs), buf, cap, len);
  });
}

int cf_mem_calibrate(const int64_t* chunk_size, const int64_t* k, const int64_t* context_len, const double* peak_gib,
                     int64_t n, double gqa_ratio, cf_mem_coeffs* out, double* max_residual_gib) {
  return cfb::guard([&] {
    std::vector<cfb::MemMeasurement> ms;
    for (int64_t i = 0; i < n; ++i) ms.push_back({chunk_size[i], k[i], context_len[i], peak_gib[i]});
    const cfb::MemCoeffs c = cfb::calibrate(ms, gqa_ratio, max_residual_gib);
    *out = {c.base, c.per_chunk_token, c.per_context_token, c.gqa_ratio};
  });
}

int cf_mem_predict(const cf_mem_coeffs* c, int64_t chunk_size, int64_t k, int64_t context_len, double* peak_gib) {
  return cfb::guard([&] { *peak_gib = cfb::predict_peak(from_c(c), chunk_size, k, context_len); });
}

int cf_mem_parse_csv(const char* csv, int64_t* n, int64_t* chunk_size, int64_t* k, int64_t* context_len,
                     double* peak_gib) {
  return cfb::guard([&] {
    const auto ms = cfb::parse_measurements(csv ? csv : "");
    *n = static_cast<int64_t>(ms.size());
    for (size_t i = 0; i < ms.size(); ++i) {
      if (chunk_size) chunk_size[i] = ms[i].chunk_size;
      if (k) k[i] = ms[i].k;
      if (context_len) context_len[i] = ms[i].context_len;
      if (peak_gib) peak_gib[i] = ms[i].peak_gib;
    }
  });
}

int cf_mem_coeffs_json(const cf_mem_coeffs* c, char* buf, size_t cap, size_t* len) {
  return cfb::guard([&] { put_text(cfb::coefficients_to_json(from_c(c)).dump(2) + "\n", buf, cap, len); });
}

}  // extern "C"

extern "C" int cf_pp_export_trace(const cf_pp_op* ops, int64_t num_stages, int64_t ops_per_stage, int format,
                                  char* buf, size_t cap, size_t* len) {
  return cfb::guard([&] {
    if (format != 0 && format != 1) throw cfb::ValidationError("unknown trace format");
    if (num_stages < 0 || ops_per_stage < 0 || (num_stages * ops_per_stage > 0 && !ops))
      throw cfb::ValidationError("bad trace arrays");
    std::vector<std::vector<cfb::TraceOp>> st(static_cast<size_t>(num_stages));
    for (int64_t s = 0; s < num_stages; ++s)
      for (int64_t i = 0; i < ops_per_stage; ++i) {
        const cf_pp_op& o = ops[s * ops_per_stage + i];
        st[static_cast<size_t>(s)].push_back({o.kind, o.chunk_id, o.start, o.end});
      }
    put_text(cfb::export_trace(st, format == 0), buf, cap, len);
  });
}

extern "C" int cf_pp_stage_memory(const cf_plan* plan, int64_t num_stages, int64_t k, int64_t tape_budget,
                                  int64_t* peak_tapes, int64_t* peak_tape_tokens, int64_t* peak_kept_tokens,
                                  int64_t* checkpointed) {
  return cfb::guard([&] {
    if (!plan) throw cfb::ValidationError("plan is null");
    if (num_stages < 1 || k < 1 || tape_budget < 0) throw cfb::ValidationError("bad pipeline arguments");
    const cfb::PpChunks info = cfb::pp_chunks(plan->p, k, cfb::PpCost{});
    std::vector<int64_t> tok;
    for (const cfb::Chunk& c : plan->p.chunks) tok.push_back(c.total);
    for (int64_t s = 0; s < num_stages; ++s) {
      const auto order = cfb::pp_stage_order(info, s, num_stages, true);
      const cfb::PpStageMem m = cfb::pp_stage_memory(info, order, tok, tape_budget, s == 0);
      if (peak_tapes) peak_tapes[s] = m.peak_tapes;
      if (peak_tape_tokens) peak_tape_tokens[s] = m.peak_tape_tokens;
      if (peak_kept_tokens) peak_kept_tokens[s] = m.peak_kept_tokens;
      if (checkpointed) checkpointed[s] = m.checkpointed;
    }
  });
}

extern "C" int cf_tune_grid_search_pp(const int64_t* ids, const int64_t* lengths, int64_t n,
                                      const int64_t* chunk_sizes, int64_t ncs, const int64_t* ks, int64_t nk,
                                      int64_t num_stages, const cf_pp_cost* cost, const cf_mem_coeffs* mem,
                                      double kept_token_gib, int64_t tape_budget, double budget_gib,
                                      int64_t global_batch_size, int64_t batches_to_sample, uint64_t seed,
                                      cf_tune_row* table, int64_t* best_chunk_size, int64_t* best_k,
                                      int64_t* evaluations, int csv, char* buf, size_t cap, size_t* len) {
  return cfb::guard([&] {
    if (n < 0 || ncs < 0 || nk < 0 || !mem) throw cfb::ValidationError("bad tuner arguments");
    const cfb::TuneResult r = cfb::grid_search_pp(
        std::vector<int64_t>(ids, ids + n), std::vector<int64_t>(lengths, lengths + n),
        std::vector<int64_t>(chunk_sizes, chunk_sizes + ncs), std::vector<int64_t>(ks, ks + nk), num_stages,
        to_cost(cost), from_c(mem), kept_token_gib, tape_budget, budget_gib, global_batch_size, batches_to_sample,
        seed);
    for (size_t i = 0; table && i < r.table.size(); ++i)
      table[i] = {r.table[i].chunk_size, r.table[i].k, r.table[i].mean_time, r.table[i].predicted_peak_gib,
                  r.table[i].feasible ? 1 : 0};
    if (best_chunk_size) *best_chunk_size = r.has_best ? r.best_chunk_size : -1;
    if (best_k) *best_k = r.has_best ? r.best_k : -1;
    if (evaluations) *evaluations = r.evaluations;
    if (buf || len) put_text(csv ? cfb::tuner_table_csv(r) : cfb::tuner_report(r), buf, cap, len);
  });
}

extern "C" int cf_tune_grid_search(const int64_t* ids, const int64_t* lengths, int64_t n, const int64_t* chunk_sizes,
                                   int64_t ncs, const int64_t* ks, int64_t nk, int64_t num_stages,
                                   const cf_pp_cost* cost, const cf_mem_coeffs* mem, double budget_gib,
                                   int64_t global_batch_size, int64_t batches_to_sample, uint64_t seed,
                                   cf_tune_row* table, int64_t* best_chunk_size, int64_t* best_k,
                                   int64_t* evaluations, int csv, char* buf, size_t cap, size_t* len) {
  return cfb::guard([&] {
    if (n < 0 || ncs < 0 || nk < 0 || !mem) throw cfb::ValidationError("bad tuner arguments");
    const cfb::TuneResult r = cfb::grid_search(
        std::vector<int64_t>(ids, ids + n), std::vector<int64_t>(lengths, lengths + n),
        std::vector<int64_t>(chunk_sizes, chunk_sizes + ncs), std::vector<int64_t>(ks, ks + nk), num_stages,
        to_cost(cost), from_c(mem), budget_gib, global_batch_size, batches_to_sample, seed);
    for (size_t i = 0; table && i < r.table.size(); ++i)
      table[i] = {r.table[i].chunk_size, r.table[i].k, r.table[i].mean_time, r.table[i].predicted_peak_gib,
                  r.table[i].feasible ? 1 : 0};
    if (best_chunk_size) *best_chunk_size = r.has_best ? r.best_chunk_size : -1;
    if (best_k) *best_k = r.has_best ? r.best_k : -1;
    if (evaluations) *evaluations = r.evaluations;
    if (buf || len) put_text(csv ? cfb::tuner_table_csv(r) : cfb::tuner_report(r), buf, cap, len);
  });
}
