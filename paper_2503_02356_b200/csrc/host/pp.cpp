// Pipeline-parallel planning: see pp.hpp.
#include "pp.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <set>
#include <stdexcept>

#include "wire.hpp"

namespace cfb {

void PpCost::validate() const {
  if (gamma < 0 || alpha < 0 || beta < 0 || hop < 0)
    throw ValidationError("cost-model coefficients must be non-negative");
  if (bwd_mult <= 0) throw ValidationError("backward multiplier must be positive");
}

PpChunks pp_chunks(const Plan& plan, int64_t k, const PpCost& cost) {
  if (plan.chunks.empty()) throw ValidationError("chunk plan has no chunks");
  if (k < 1) throw ValidationError("retention budget k must be at least 1");
  cost.validate();
  const size_t m = plan.chunks.size();
  PpChunks c;
  c.fwd.resize(m);
  c.bwd.resize(m);
  c.discarded.assign(m, 0);
  c.ids.resize(m);
  c.prefix.assign(m, 0);
  std::map<int64_t, size_t> pos;
  for (size_t i = 0; i < m; ++i) pos[plan.chunks[i].id] = i;
  // group id -> running token count while walking members in index order
  for (const auto& [g, members] : plan.groups) {
    int64_t run = 0;
    const int64_t n = static_cast<int64_t>(members.size());
    for (int64_t j = 0; j < n; ++j) {
      const size_t p = pos.at(members[static_cast<size_t>(j)]);
      c.prefix[p] = run;
      run += plan.chunks[p].total;
      if (n > k && plan.chunks[p].index < n - k) c.discarded[p] = 1;
    }
  }
  for (size_t i = 0; i < m; ++i) {
    const Chunk& ch = plan.chunks[i];
    c.ids[i] = ch.id;
    const double len = static_cast<double>(ch.total);
    const double pre = ch.kind == kDependent ? static_cast<double>(c.prefix[i]) : 0.0;
    c.fwd[i] = cost.fwd(len, pre);
    c.bwd[i] = cost.bwd_mult * c.fwd[i];
  }
  std::set<int64_t> seen;
  for (size_t i = 0; i < m; ++i) {
    const Chunk& ch = plan.chunks[i];
    if (ch.kind != kDependent) {
      c.bwd_queue.push_back(static_cast<int64_t>(i));
    } else if (seen.insert(ch.group).second) {
      const std::vector<int64_t>& members = plan.groups.at(ch.group);
      for (auto it = members.rbegin(); it != members.rend(); ++it)
        c.bwd_queue.push_back(static_cast<int64_t>(pos.at(*it)));
    }
  }
  return c;
}

PpChunks pp_microbatches(const std::vector<int64_t>& lengths, const PpCost& cost) {
  if (lengths.empty()) throw ValidationError("no microbatches to simulate");
  cost.validate();
  PpChunks c;
  for (size_t i = 0; i < lengths.size(); ++i) {
    c.fwd.push_back(cost.fwd(static_cast<double>(lengths[i]), 0.0));
    c.bwd.push_back(cost.bwd_mult * c.fwd.back());
    c.discarded.push_back(0);
    c.ids.push_back(static_cast<int64_t>(i));
    c.bwd_queue.push_back(static_cast<int64_t>(i));
    c.prefix.push_back(0);
  }
  return c;
}

std::vector<PpOp> pp_stage_order(const PpChunks& c, int64_t stage, int64_t stages, bool backward_first) {
  const int64_t m = static_cast<int64_t>(c.fwd.size());
  std::vector<PpOp> ops;
  ops.reserve(static_cast<size_t>(2 * m + 1));
  int64_t next = 0;  // forwards are issued in plan order; `next` is the first not yet issued
  const int64_t warm = std::min(stages - stage, m);
  while (next < warm) ops.push_back({kPpForward, next++});
  for (int64_t b : c.bwd_queue) {
    if (!backward_first && next < m) ops.push_back({kPpForward, next++});
    while (next <= b) ops.push_back({kPpForward, next++});  // enablers: b and everything before it
    if (c.discarded[static_cast<size_t>(b)]) ops.push_back({kPpRecompute, b});
    ops.push_back({kPpBackward, b});
    if (backward_first && next < m) ops.push_back({kPpForward, next++});
  }
  return ops;
}

PpTrace pp_dispatch(const std::vector<std::vector<PpOp>>& orders, const std::vector<double>& fwd,
                    const std::vector<double>& bwd, double hop, const std::vector<std::vector<double>>* bwd_extra) {
  const int64_t P = static_cast<int64_t>(orders.size());
  const size_t m = fwd.size();
  PpTrace t;
  t.stages.resize(static_cast<size_t>(P));
  t.busy.assign(static_cast<size_t>(P), 0.0);
  t.busy_total.assign(static_cast<size_t>(P), 0.0);
  const double kUnset = -1.0;
  // end time of (stage, first-pass forward | backward, position)
  std::vector<std::vector<double>> f_end(static_cast<size_t>(P), std::vector<double>(m, kUnset));
  std::vector<std::vector<double>> b_end(static_cast<size_t>(P), std::vector<double>(m, kUnset));
  std::vector<size_t> next(static_cast<size_t>(P), 0);
  std::vector<double> free_at(static_cast<size_t>(P), 0.0);
  size_t left = 0;
  for (const auto& o : orders) left += o.size();
  while (left) {
    bool moved = false;
    for (int64_t s = 0; s < P; ++s) {
      const auto& ord = orders[static_cast<size_t>(s)];
      size_t& i = next[static_cast<size_t>(s)];
      for (; i < ord.size(); ++i) {
        const PpOp& op = ord[i];
        const size_t p = static_cast<size_t>(op.pos);
        double ready = 0.0;
        if (op.kind == kPpForward) {
          if (s > 0) {  // activation from the previous stage
            const double e = f_end[static_cast<size_t>(s - 1)][p];
            if (e == kUnset) break;
            ready = e + hop;
          }
        } else if (s + 1 < P) {  // F' and B wait for the next stage's backward
          const double e = b_end[static_cast<size_t>(s + 1)][p];
          if (e == kUnset) break;
          ready = e + hop;
        }
        double dur = op.kind == kPpBackward ? bwd[p] : fwd[p];
        if (bwd_extra && op.kind == kPpBackward) dur += (*bwd_extra)[static_cast<size_t>(s)][p];
        const double start = std::max(free_at[static_cast<size_t>(s)], ready);
        const double end = start + dur;
        t.stages[static_cast<size_t>(s)].push_back({op.kind, op.pos, start, end});
        if (op.kind == kPpForward) f_end[static_cast<size_t>(s)][p] = end;
        if (op.kind == kPpBackward) b_end[static_cast<size_t>(s)][p] = end;
        free_at[static_cast<size_t>(s)] = end;
        t.busy_total[static_cast<size_t>(s)] += dur;
        if (op.kind != kPpRecompute) t.busy[static_cast<size_t>(s)] += dur;
        t.makespan = std::max(t.makespan, end);
        --left;
        moved = true;
      }
    }
    if (!moved) throw std::logic_error("pipeline dispatch reached a dependency deadlock");
  }
  return t;
}

PpStageMem pp_stage_memory(const PpChunks& c, const std::vector<PpOp>& order, const std::vector<int64_t>& tokens,
                           int64_t tape_budget, bool first_stage) {
  PpStageMem r;
  const size_t m = c.fwd.size();
  r.ckpt.assign(m, 0);
  std::vector<uint8_t> live(m, 0), kept(m, 0), seen(m, 0);
  int64_t tapes = 0, tape_tok = 0, kept_tok = 0;
  auto take_tape = [&](size_t p) {
    live[p] = 1;
    ++tapes;
    tape_tok += tokens[p];
    r.peak_tapes = std::max(r.peak_tapes, tapes);
    r.peak_tape_tokens = std::max(r.peak_tape_tokens, tape_tok);
  };
  auto keep = [&](size_t p) {
    if (first_stage) return;  // the first stage re-embeds its tokens
    kept[p] = 1;
    kept_tok += tokens[p];
    r.peak_kept_tokens = std::max(r.peak_kept_tokens, kept_tok);
  };
  auto unkeep = [&](size_t p) {
    if (!kept[p]) return;
    kept[p] = 0;
    kept_tok -= tokens[p];
  };
  for (const PpOp& op : order) {
    const size_t p = static_cast<size_t>(op.pos);
    if (op.kind == kPpForward) {
      seen[p] = 1;
      if (c.discarded[p]) {
        keep(p);
      } else if (tape_budget > 0 && tapes + 1 >= tape_budget) {
        r.ckpt[p] = 1;
        ++r.checkpointed;
        keep(p);
      } else {
        take_tape(p);
      }
    } else if (op.kind == kPpRecompute) {
      unkeep(p);
      take_tape(p);
    } else {
      if (r.ckpt[p] && !live[p]) {  // just-in-time restore
        unkeep(p);
        take_tape(p);
      }
      if (live[p]) {
        live[p] = 0;
        --tapes;
        tape_tok -= tokens[p];
      }
    }
  }
  return r;
}

double pp_bubble(const PpTrace& t) {
  if (t.stages.empty()) throw ValidationError("empty trace");
  if (t.makespan <= 0.0) return 0.0;
  double idle = 0.0;
  for (double b : t.busy) idle += t.makespan - b;
  return idle / (static_cast<double>(t.stages.size()) * t.makespan);
}

void pp_stage_layers(int64_t layers, int64_t stage, int64_t stages, int64_t* begin, int64_t* end) {
  if (stages < 1 || stage < 0 || stage >= stages) throw ValidationError("stage index out of range");
  if (layers < stages) throw ValidationError("fewer layers than pipeline stages");
  *begin = layers * stage / stages;
  *end = layers * (stage + 1) / stages;
}

}  // namespace cfb

// ------------------------------------------------------------------ tuner
namespace cfb {

TuneResult grid_search(const std::vector<int64_t>& ids, const std::vector<int64_t>& lengths,
                       const std::vector<int64_t>& chunk_sizes, const std::vector<int64_t>& ks, int64_t stages,
                       const PpCost& cost, const MemCoeffs& mem, double budget_gib, int64_t global_batch_size,
                       int64_t batches_to_sample, uint64_t seed) {
  if (chunk_sizes.empty() || ks.empty()) throw ValidationError("tuner grid must not be empty");
  if (budget_gib <= 0) throw ValidationError("memory budget must be positive");
  if (batches_to_sample < 1) throw ValidationError("batches_to_sample must be at least 1");
  if (lengths.empty()) throw ValidationError("cannot tune on an empty sequence set");
  if (global_batch_size < 1) throw ValidationError("global batch size must be at least 1");
  cost.validate();
  if (mem.base < 0 || mem.per_chunk_token < 0 || mem.per_context_token < 0 || mem.gqa_ratio < 0)
    throw ValidationError("memory-model coefficients must be non-negative");
  if (stages < 1) throw ValidationError("num_stages must be at least 1");
  const int64_t n = static_cast<int64_t>(lengths.size());
  const int64_t steps = (n + global_batch_size - 1) / global_batch_size;
  std::vector<std::pair<std::vector<int64_t>, std::vector<int64_t>>> batches;  // (ids, lengths)
  int64_t max_len = 0;
  for (int64_t t = 0; t < batches_to_sample; ++t) {
    const std::vector<int64_t> idx = sample_batch(n, global_batch_size, t % steps, seed);
    if (idx.empty()) break;
    std::vector<int64_t> bi, bl;
    for (int64_t i : idx) {
      bi.push_back(ids[static_cast<size_t>(i)]);
      bl.push_back(lengths[static_cast<size_t>(i)]);
      max_len = std::max(max_len, lengths[static_cast<size_t>(i)]);
    }
    batches.emplace_back(std::move(bi), std::move(bl));
  }
  TuneResult r;
  for (int64_t cs : chunk_sizes)
    for (int64_t k : ks) {
      const int64_t k_eff = stages == 1 ? 1 : k;
      TuneRow row;
      row.chunk_size = cs;
      row.k = k;
      row.predicted_peak_gib = predict_peak(mem, cs, k_eff, max_len);
      row.feasible = row.predicted_peak_gib <= budget_gib;
      double total = 0.0;
      for (const auto& [bi, bl] : batches) {
        const Plan plan = construct_chunks(bi.data(), bl.data(), static_cast<int64_t>(bi.size()), cs);
        const PpChunks info = pp_chunks(plan, k_eff, cost);
        std::vector<std::vector<PpOp>> orders;
        for (int64_t s = 0; s < stages; ++s) orders.push_back(pp_stage_order(info, s, stages, true));
        total += pp_dispatch(orders, info.fwd, info.bwd, cost.hop).makespan;
        ++r.evaluations;
      }
      row.mean_time = total / static_cast<double>(batches.size());
      r.table.push_back(row);
    }
  const TuneRow* best = nullptr;
  for (const TuneRow& c : r.table) {
    if (!c.feasible) continue;
    if (!best || c.mean_time < best->mean_time ||
        (c.mean_time == best->mean_time &&
         (c.chunk_size > best->chunk_size || (c.chunk_size == best->chunk_size && c.k < best->k))))
      best = &c;
  }
  if (best) {
    r.has_best = true;
    r.best_chunk_size = best->chunk_size;
    r.best_k = best->k;
  }
  return r;
}

namespace {
std::string fixed(double v, int prec) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.*f", prec, v);
  return buf;
}
}  // namespace

TuneResult grid_search_pp(const std::vector<int64_t>& ids, const std::vector<int64_t>& lengths,
                          const std::vector<int64_t>& chunk_sizes, const std::vector<int64_t>& ks, int64_t stages,
                          const PpCost& cost, const MemCoeffs& mem, double kept_token_gib, int64_t tape_budget,
                          double budget_gib, int64_t global_batch_size, int64_t batches_to_sample, uint64_t seed) {
  if (chunk_sizes.empty() || ks.empty()) throw ValidationError("tuner grid must not be empty");
  if (budget_gib <= 0) throw ValidationError("memory budget must be positive");
  if (batches_to_sample < 1) throw ValidationError("batches_to_sample must be at least 1");
  if (lengths.empty()) throw ValidationError("cannot tune on an empty sequence set");
  if (global_batch_size < 1) throw ValidationError("global batch size must be at least 1");
  if (tape_budget < 0 || kept_token_gib < 0) throw ValidationError("tape budget and kept-token size must be non-negative");
  cost.validate();
  if (mem.base < 0 || mem.per_chunk_token < 0 || mem.per_context_token < 0 || mem.gqa_ratio < 0)
    throw ValidationError("memory-model coefficients must be non-negative");
  if (stages < 1) throw ValidationError("num_stages must be at least 1");
  const int64_t n = static_cast<int64_t>(lengths.size());
  const int64_t steps = (n + global_batch_size - 1) / global_batch_size;
  std::vector<std::pair<std::vector<int64_t>, std::vector<int64_t>>> batches;
  int64_t max_len = 0;
  for (int64_t t = 0; t < batches_to_sample; ++t) {
    const std::vector<int64_t> idx = sample_batch(n, global_batch_size, t % steps, seed);
    if (idx.empty()) break;
    std::vector<int64_t> bi, bl;
    for (int64_t i : idx) {
      bi.push_back(ids[static_cast<size_t>(i)]);
      bl.push_back(lengths[static_cast<size_t>(i)]);
      max_len = std::max(max_len, lengths[static_cast<size_t>(i)]);
    }
    batches.emplace_back(std::move(bi), std::move(bl));
  }
  TuneResult r;
  for (int64_t cs : chunk_sizes)
    for (int64_t k : ks) {
      TuneRow row;
      row.chunk_size = cs;
      row.k = k;
      double total = 0.0, peak = 0.0;
      for (const auto& [bi, bl] : batches) {
        const Plan plan = construct_chunks(bi.data(), bl.data(), static_cast<int64_t>(bi.size()), cs);
        const PpChunks info = pp_chunks(plan, k, cost);
        std::vector<int64_t> tok;
        for (const Chunk& ch : plan.chunks) tok.push_back(ch.total);
        std::vector<std::vector<PpOp>> orders;
        std::vector<std::vector<double>> extra;
        for (int64_t s = 0; s < stages; ++s) {
          orders.push_back(pp_stage_order(info, s, stages, true));
          const PpStageMem sm = pp_stage_memory(info, orders.back(), tok, tape_budget, s == 0);
          peak = std::max(peak, mem.base + mem.per_chunk_token * static_cast<double>(sm.peak_tape_tokens) +
                                    kept_token_gib * static_cast<double>(sm.peak_kept_tokens) +
                                    mem.per_context_token * mem.gqa_ratio * static_cast<double>(max_len));
          std::vector<double> e(info.fwd.size(), 0.0);
          for (size_t p = 0; p < e.size(); ++p)
            if (sm.ckpt[p]) e[p] = info.fwd[p];
          extra.push_back(std::move(e));
        }
        total += pp_dispatch(orders, info.fwd, info.bwd, cost.hop, &extra).makespan;
        ++r.evaluations;
      }
      row.predicted_peak_gib = peak;
      row.feasible = peak <= budget_gib;
      row.mean_time = total / static_cast<double>(batches.size());
      r.table.push_back(row);
    }
  const TuneRow* best = nullptr;
  for (const TuneRow& c : r.table) {
    if (!c.feasible) continue;
    if (!best || c.mean_time < best->mean_time ||
        (c.mean_time == best->mean_time &&
         (c.chunk_size > best->chunk_size || (c.chunk_size == best->chunk_size && c.k < best->k))))
      best = &c;
  }
  if (best) {
    r.has_best = true;
    r.best_chunk_size = best->chunk_size;
    r.best_k = best->k;
  }
  return r;
}

std::string tuner_table_csv(const TuneResult& r) {
  std::string out = "chunk_size,k,mean_time,predicted_peak_gib,feasible\n";
  for (const TuneRow& row : r.table)
    out += std::to_string(row.chunk_size) + "," + std::to_string(row.k) + "," + fixed(row.mean_time, 6) + "," +
           fixed(row.predicted_peak_gib, 3) + "," + (row.feasible ? "1" : "0") + "\n";
  return out;
}

std::string tuner_report(const TuneResult& r) {
  std::vector<TuneRow> ranked = r.table;
  std::stable_sort(ranked.begin(), ranked.end(), [](const TuneRow& a, const TuneRow& b) {
    if (a.feasible != b.feasible) return a.feasible;
    if (a.mean_time != b.mean_time) return a.mean_time < b.mean_time;
    if (a.chunk_size != b.chunk_size) return a.chunk_size > b.chunk_size;
    return a.k < b.k;
  });
  std::string out = r.has_best ? "best: chunk_size=" + std::to_string(r.best_chunk_size) +
                                     " k=" + std::to_string(r.best_k) + "\n"
                               : std::string("no feasible configuration\n");
  out += "evaluations: " + std::to_string(r.evaluations) + "\n";
  for (const TuneRow& row : ranked)
    out += "chunk_size=" + std::to_string(row.chunk_size) + " k=" + std::to_string(row.k) +
           " mean_time=" + fixed(row.mean_time, 3) + " predicted_peak_gib=" + fixed(row.predicted_peak_gib, 3) +
           (row.feasible ? " feasible" : " infeasible") + "\n";
  return out;
}

}  // namespace cfb
