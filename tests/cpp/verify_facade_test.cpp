// verify_equivalence / compare_gradients / backward_full / run_plan through
// the C++ facade (GPU) with reference call sites (plan_runner.hpp:368-395,
// toy_model.hpp:575-596, :681-718).  Prints the report, a K-reordered but
// valid schedule's gradient difference (expected 0: K does not change the
// math), and the ValidationError of an invalid edited schedule.
#include <cstdio>

#include "chunkflow_b200.hpp"

int main() {
  namespace cf = chunkflow_b200;
  cf::Device dev(0);
  cf_model_cfg cfg{1, 0, 64, 128, 4, 2, 2, 256, 9, 10000.0, 1e-5};
  cf::Model model(dev, cfg);
  cf::SequenceSet batch;
  const int64_t lens[] = {150, 20, 9, 64, 33};
  uint64_t x = 7;
  for (int64_t i = 0; i < 5; ++i) {
    cf::SequenceRecord r{i, lens[i], {}};
    for (int64_t t = 0; t < lens[i]; ++t) {
      x = x * 6364136223846793005ULL + 1442695040888963407ULL;
      r.tokens.push_back(static_cast<int32_t>((x >> 33) % 64));
    }
    batch.push_back(r);
  }
  const cf::VerifyReport rep = cf::verify_equivalence(model, batch, 32, 1, 1e-4, 1e-2);
  std::printf("%s", rep.to_text().c_str());

  // compare_gradients of two identical runs: exactly 0
  cf::Batch b;
  b.sequences = batch;
  const auto cp = cf::construct_chunks(b, 32);
  const auto ep1 = cf::schedule_step(cp, 1);
  const auto r1 = cf::run_plan(model, cp, ep1, batch);
  const cf::GradientSet g1 = cf::read_gradients(model, r1.loss);
  const auto ep3 = cf::schedule_step(cp, 3);
  const auto r3 = cf::run_plan(model, cp, ep3, batch);
  const cf::GradientSet g3 = cf::read_gradients(model, r3.loss);
  const cf::GradComparison c = cf::compare_gradients(g1, g3);
  std::printf("k1_vs_k3 max_rel_err=%g loss_rel_err=%g\n", c.max_rel_err, c.loss_rel_err);

  // an edited schedule with a violation is refused (plan_runner.hpp:78-81)
  auto bad = ep1;
  bad.events.pop_back();
  try {
    cf::run_plan(model, cp, bad, batch);
    std::printf("invalid plan ran\n");
  } catch (const cf::ValidationError& e) {
    std::printf("ValidationError: %s\n", e.what());
  }
  const cf::GradientSet full = cf::backward_full(model, batch);
  std::printf("backward_full tensors=%zu loss=%.6f\n", full.tensors.size(), full.loss);
  return 0;
}
