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
  return 0;
}
