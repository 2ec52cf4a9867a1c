// Host planning for the B200 ChunkFlow path: chunk construction (Alg. 1),
// state-aware scheduling (Alg. 2), replay validation and the data-parallel
// unit partition.  Integer output is bit-exact with the reference
// (/root/reference/proj/include/chunkflow/chunker.hpp, scheduler.hpp).
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace cfb {

struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {  // chunkflow::ParseError (common.hpp:20)
  using std::runtime_error::runtime_error;
};

enum : int64_t { kStandalone = 0, kDependent = 1 };
enum : int64_t { kFwdDiscard = 0, kFwdRetain = 1, kBackward = 2 };

struct Segment {
  int64_t seq, start, len;
};

struct Chunk {
  int64_t id = 0, kind = kStandalone, group = -1, index = -1, total = 0;
  int64_t seg_off = 0, seg_cnt = 0;
};

struct Event {
  int64_t kind, chunk, group, index;
  bool recompute, save_kv, read_prefix, acc_grad;
};

struct Plan {
  int64_t chunk_size = 0;
  int64_t k = 1;
  std::vector<Chunk> chunks;      // plan order; chunk id == position for
  std::vector<Segment> segments;  //   construct_chunks plans
  std::map<int64_t, std::vector<int64_t>> groups;  // group -> chunk ids
  std::map<int64_t, int64_t> chunk_tokens;         // chunk -> tokens
  std::vector<Event> events;
  int64_t peak_retained = 0, recompute_tokens = 0;
  std::vector<std::string> violations;

  const Chunk& chunk(int64_t id) const;
  std::map<int64_t, int64_t> index_of;  // chunk id -> position
};

// construct_chunks (chunker.hpp:177-227).
Plan construct_chunks(const int64_t* ids, const int64_t* lengths, int64_t n,
                      int64_t chunk_size);
// schedule_step (scheduler.hpp:132-171): fills plan.events, then replays.
void schedule_step(Plan& plan, int64_t k);
// schedule_group (scheduler.hpp:106-127).
Plan schedule_group(int64_t n, int64_t k, int64_t chunk_size);
// validate_plan (scheduler.hpp:182-271): fills diagnostics + violations.
void validate(Plan& plan);
// execution_plan_listing (scheduler.hpp:284-298).
std::string listing(const Plan& plan);

// Data-parallel unit partition: units are standalone chunks and
// whole dependent groups; deterministic LPT over cost
// alpha*tokens + beta*attention_pairs (+ recompute forwards at 1/3 weight).
// Returns rank -> sorted list of unit-first-chunk positions.
struct Unit {
  std::vector<int64_t> chunk_pos;  // positions in plan.chunks
  double cost = 0.0;
  int64_t tokens = 0;
};
std::vector<Unit> plan_units(const Plan& plan, double alpha, double beta);
std::vector<std::vector<int64_t>> lpt_assign(const std::vector<Unit>& units,
                                             int64_t world);
Plan sub_plan(const Plan& global, const std::vector<Unit>& units,
              const std::vector<int64_t>& mine, int64_t k);

uint64_t splitmix_next(uint64_t& state);

// synthesize (dataset.hpp:207-237): bucket by CDF inversion, then
// log-uniform within the bucket; bucket_low (:183-189).  Pure function of
// (spec, count, seed); bit-exact with the reference.
std::vector<int64_t> synthesize(const std::vector<int64_t>& bounds, const std::vector<double>& fracs,
                                int64_t max_length, int64_t count, uint64_t seed);
// sample_batch (dataset.hpp:242-268): seed-keyed Fisher-Yates permutation
// of [0, n) sliced into consecutive global batches; returns indices.
std::vector<int64_t> sample_batch(int64_t n, int64_t global_batch, int64_t step, uint64_t seed);

}  // namespace cfb
