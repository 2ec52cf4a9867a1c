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
  return 0;
}
