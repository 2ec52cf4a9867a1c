#include "chunkflow_b200.hpp"
#include <cstdio>
int main() {
  namespace cf = chunkflow_b200;
  cf::Batch b;
  int64_t lens[] = {1, 1, 2, 4};
  for (int i = 0; i < 4; ++i) b.sequences.push_back({i, lens[i], {}});
  auto cp = cf::construct_chunks(b, 2);
  auto ep = cf::schedule_step(cp, 1);
  auto d = cf::validate_plan(ep);
  std::printf("chunks=%zu events=%zu peak=%lld recompute=%lld groups=%zu\n", cp.chunks.size(), ep.events.size(),
              (long long)d.peak_retained_tokens, (long long)d.recompute_token_count, cp.groups.size());
  // validate_plan replays the plan as held: edits are seen (test_scheduler.cpp:165-221)
  auto edited = ep;
  std::swap(edited.events[5], edited.events[6]);  // F+ chunk3 <-> B chunk3: backward without retain
  const auto de = cf::validate_plan(edited);
  std::printf("edited_violations=%zu first=%s\n", de.violations.size(),
              de.violations.empty() ? "-" : de.violations[0].c_str());
  cf::ExecutionPlan hand;  // hand-built: one backward, nothing retained
  hand.chunk_size = 4;
  cf::ExecEvent bw;
  bw.kind = cf::ExecKind::kBackward;
  hand.events.push_back(bw);
  std::printf("hand=%s\n", cf::validate_plan(hand).violations.at(0).c_str());
  try { cf::construct_chunks(b, 0); } catch (const cf::ValidationError& e) { std::printf("ValidationError: %s\n", e.what()); }
  // pipeline.hpp worked example (test_pipeline.cpp:141-211): 56 / 54 / 46 / 60 units
  cf::PipelineConfig pc;
  pc.num_stages = 4;
  const auto t1 = cf::simulate_1f1b({1, 1, 2, 4}, 4, cf::CostModel{});
  const auto t2 = cf::simulate_state_aware_1f1b(cp, pc, cf::CostModel{});
  pc.k = 2;
  const auto t3 = cf::simulate_state_aware_1f1b(cp, pc, cf::CostModel{});
  std::printf("makespans=%g,%g,%g bubble=%.2f stage0_ops=%zu\n", t1.makespan, t2.makespan, t3.makespan,
              100.0 * cf::bubble_ratio(t2), t2.stages[0].size());
  // memory model (test_memory_model.cpp Table 6) and tuner (test_tuner.cpp worked batch)
  const auto cal = cf::calibrate({{2048, 1, 32768, 41.6}, {2048, 1, 262144, 45.6}, {4096, 1, 32768, 47.5},
                                  {4096, 1, 262144, 50.8}, {8192, 1, 32768, 59.3}, {8192, 1, 262144, 63.8}});
  std::printf("base=%.4f resid=%.5f\n", cal.coefficients.base, cal.max_residual_gib);
  cf::PipelineConfig tc;
  tc.num_stages = 4;
  const auto tr = cf::grid_search(b.sequences, {2, 4}, {1, 2}, tc, cf::CostModel{}, cf::MemoryModelCoefficients{},
                                  1e9, 4, 1, 1);
  std::printf("tuner best=%lld,%lld evals=%lld\n", (long long)tr.best_chunk_size, (long long)tr.best_k,
              (long long)tr.evaluations);
  // wire formats
  const std::string js = cf::chunk_plan_json(ep);
  const auto set = cf::load_lengths("{\"id\": 7, \"length\": 3, \"tokens\": [1, 2, 3]}\n{\"length\": 2}\n");
  std::printf("json=%zu set=%zu,%lld,%zu\n", js.size() > 100 ? (size_t)1 : (size_t)0, set.size(),
              (long long)set[0].id, set[0].tokens.size());
  return 0;
}
