// Pipeline-parallel planning for the chunk-aware 1F1B schedule (config C5).
//
// The reference only *simulates* pipelines (pipeline.hpp:164-331); here the
// same per-stage instruction streams drive the real stage executor
// (runtime/engine.cu), and the same earliest-feasible dispatch times them
// for the bubble prediction.  Output is bit-exact with the reference
// (tests/test_pp_plan.py pins op order, start/end times and bubble ratio).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "plan.hpp"

namespace cfb {

// TraceEventKind (pipeline.hpp:51): first-pass forward, just-in-time
// recompute forward of a discarded chunk, backward.
enum : int64_t { kPpForward = 0, kPpRecompute = 1, kPpBackward = 2 };

// CostModel (pipeline.hpp:24-47): fwd = gamma + alpha*len + beta*len^2 +
// beta*len*prefix (beta*len^2, not the causal half: Appendix B-8),
// bwd = backward_multiplier * fwd.
struct PpCost {
  double gamma = 0.0, alpha = 1.0, beta = 0.0, bwd_mult = 2.0, hop = 0.0;
  void validate() const;
  double fwd(double len, double prefix) const { return gamma + alpha * len + beta * len * len + beta * len * prefix; }
};

struct PpOp {
  int64_t kind;
  int64_t pos;  // plan position (index into plan.chunks)
};

// ChunkTimingInfo (pipeline.hpp:164-170) for one microbatch list.
struct PpChunks {
  std::vector<double> fwd, bwd;
  std::vector<uint8_t> discarded;     // needs F' before its B
  std::vector<int64_t> ids;           // chunk id per position
  std::vector<int64_t> bwd_queue;     // plan order, dependent groups reversed
  std::vector<int64_t> prefix;        // tokens of earlier group members
};

// State-aware view of a chunk plan under retention budget k
// (simulate_state_aware_1f1b, pipeline.hpp:258-304).
PpChunks pp_chunks(const Plan& plan, int64_t k, const PpCost& cost);
// Plain 1F1B over whole sequences (simulate_1f1b, pipeline.hpp:218-236).
PpChunks pp_microbatches(const std::vector<int64_t>& lengths, const PpCost& cost);

// Per-stage static op stream (build_stage_order, pipeline.hpp:178-210):
// min(P-s, M) warm-up forwards, then per backward-queue entry the enabling
// forwards, F' for a discarded chunk, B, and one more forward (backward-
// first policy; forward-first places that forward before the entry).
std::vector<PpOp> pp_stage_order(const PpChunks& c, int64_t stage, int64_t stages, bool backward_first);

struct PpTimedOp {
  int64_t kind, pos;
  double start, end;
};
struct PpTrace {
  std::vector<std::vector<PpTimedOp>> stages;
  double makespan = 0.0;
  std::vector<double> busy, busy_total;  // busy excludes recompute forwards
};

// Earliest-feasible list scheduling over fixed stage orders (run_dispatch,
// pipeline.hpp:98-162).  Throws std::logic_error on a dependency deadlock.
// bwd_extra (optional, [stage][position]): time added to that stage's
// backward of that chunk — the just-in-time recompute of a chunk the stage
// checkpointed under a tape budget (zero / absent: the reference timing).
PpTrace pp_dispatch(const std::vector<std::vector<PpOp>>& orders, const std::vector<double>& fwd,
                    const std::vector<double>& bwd, double hop,
                    const std::vector<std::vector<double>>* bwd_extra = nullptr);

// Activation memory of one stage's op stream, replayed with the executor's
// rules (runtime/engine.cu StageRunner): a first-pass retain-forward keeps a
// tape unless that would leave no free slot under `tape_budget` (> 0), in
// which case it keeps only its stage input (nothing on the first stage) and
// is recomputed just before its backward; a K-plan discarded forward keeps
// its stage input until its F'.  Peaks are over the whole stream.
struct PpStageMem {
  int64_t peak_tapes = 0, peak_tape_tokens = 0, peak_kept_tokens = 0, checkpointed = 0;
  std::vector<uint8_t> ckpt;  // per position: checkpointed on this stage
};
PpStageMem pp_stage_memory(const PpChunks& c, const std::vector<PpOp>& order, const std::vector<int64_t>& tokens,
                           int64_t tape_budget, bool first_stage);
// bubble_ratio (pipeline.hpp:325-331): recompute counts as bubble.
double pp_bubble(const PpTrace& t);

// Layer range [begin, end) of a stage under the even split the executor
// uses (embedding on stage 0; final norm + head + loss on the last stage).
void pp_stage_layers(int64_t layers, int64_t stage, int64_t stages, int64_t* begin, int64_t* end);

}  // namespace cfb

namespace cfb {

// grid_search (tuner.hpp:39-112): for every (chunk_size, k) candidate, chunk
// the same sampled batches (sample_batch, dataset.hpp:242), time them with
// the state-aware 1F1B simulator and average the makespan; feasibility from
// the linear memory model at the longest sampled sequence (memory_model.hpp:
// 47).  k is forced to 1 with one stage.  Ties prefer larger chunk_size,
// then smaller k.
struct TuneRow {
  int64_t chunk_size = 0, k = 1;
  double mean_time = 0.0, predicted_peak_gib = 0.0;
  bool feasible = false;
};
struct TuneResult {
  bool has_best = false;
  int64_t best_chunk_size = 0, best_k = 0, evaluations = 0;
  std::vector<TuneRow> table;
};
struct MemCoeffs;
TuneResult grid_search(const std::vector<int64_t>& ids, const std::vector<int64_t>& lengths,
                       const std::vector<int64_t>& chunk_sizes, const std::vector<int64_t>& ks, int64_t stages,
                       const PpCost& cost, const MemCoeffs& mem, double budget_gib, int64_t global_batch_size,
                       int64_t batches_to_sample, uint64_t seed);
// grid_search for a pipeline (new; the reference's memory feasibility counts
// k * chunk_size retained tokens, which a 1F1B stage exceeds: its warm-up
// keeps min(P - s, M) chunks in flight).  Per sampled batch and stage the
// op stream is replayed (pp_stage_memory) under `tape_budget`; a candidate is
// feasible when every stage's base + per_chunk_token * peak tape tokens +
// kept_token_gib * peak kept-input tokens + per_context_token * gqa *
// max_len fits the budget; the reported peak is the worst stage's.  Timing
// adds each stage's checkpoint recomputes to its backwards.
TuneResult grid_search_pp(const std::vector<int64_t>& ids, const std::vector<int64_t>& lengths,
                          const std::vector<int64_t>& chunk_sizes, const std::vector<int64_t>& ks, int64_t stages,
                          const PpCost& cost, const MemCoeffs& mem, double kept_token_gib, int64_t tape_budget,
                          double budget_gib, int64_t global_batch_size, int64_t batches_to_sample, uint64_t seed);
std::string tuner_table_csv(const TuneResult& r);  // tuner.hpp:114-124
std::string tuner_report(const TuneResult& r);     // tuner.hpp:126-150

}  // namespace cfb
