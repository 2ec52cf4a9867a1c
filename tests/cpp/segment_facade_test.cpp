// Reference-style operator test through the C++ facade (GPU): a 3-token-
// chunk split of one sequence composed from detail::segment_forward /
// segment_backward the way plan_runner.hpp:128-156, 306-321 does, against
// run_plan on the same chunking.  Prints the loss difference and the max
// per-tensor gradient difference (expected: exactly 0, same kernels).
#include <cmath>
#include <cstdio>

#include "chunkflow_b200.hpp"

int main() {
  namespace cf = chunkflow_b200;
  cf::Device dev(0);
  cf_model_cfg cfg{0, 0, 64, 64, 4, 2, 2, 0, 5, 10000.0, 1e-5};
  cf::Model model(dev, cfg);
  const int64_t n = 150;
  std::vector<int32_t> tok(n);
  uint64_t x = 42;
  for (auto& t : tok) {
    x = x * 6364136223846793005ULL + 1442695040888963407ULL;
    t = static_cast<int32_t>((x >> 33) % 64);
  }
  std::vector<int64_t> tgt(n, -1);
  for (int64_t i = 0; i + 1 < n; ++i) tgt[i] = tok[i + 1];

  // run_plan: chunk 50, K = 3 (every chunk retained)
  cf::Batch b;
  b.sequences.push_back({0, n, tok});
  const auto cp = cf::construct_chunks(b, 50);
  const auto ep = cf::schedule_step(cp, 3);
  const cf_run_result r = cf::run_plan(model, cp, ep, b.sequences);
  const int64_t nt = cf_model_num_tensors(model.get());
  std::vector<std::vector<double>> g_plan;
  for (int64_t i = 0; i < nt; ++i) {
    char name[64];
    int64_t rows = 0, cols = 0;
    cf::check(cf_model_tensor_info(model.get(), i, name, sizeof name, &rows, &cols));
    g_plan.emplace_back(static_cast<size_t>(rows * cols));
    cf::check(cf_model_get_grad(model.get(), i, g_plan.back().data()));
  }

  // the same three segments through the operator API
  cf::check(cf_model_zero_grads(model.get()));
  const int64_t cut[4] = {0, 50, 100, 150};
  std::vector<cf::detail::SegmentTape> tapes;
  std::vector<std::vector<double>> pk(2), pv(2);  // running prefix per layer
  double loss_sum = 0;
  for (int s = 0; s < 3; ++s) {
    const int64_t a = cut[s], len = cut[s + 1] - cut[s];
    auto t = cf::detail::segment_forward(model, cfg, tok.data() + a, len, tgt.data() + a, a ? pk : decltype(pk){},
                                         a ? pv : decltype(pv){}, a, true);
    loss_sum += t.loss_sum;
    for (int l = 0; l < 2; ++l) {
      pk[l].insert(pk[l].end(), t.saved_k[l].begin(), t.saved_k[l].end());
      pv[l].insert(pv[l].end(), t.saved_v[l].begin(), t.saved_v[l].end());
    }
    tapes.push_back(std::move(t));
  }
  const size_t kvw = 2 * 16;
  std::vector<std::vector<double>> dk(2, std::vector<double>(n * kvw, 0.0)), dv = dk;
  for (int s = 2; s >= 0; --s) {
    const int64_t a = cut[s], len = cut[s + 1] - cut[s];
    std::vector<std::vector<double>> prek(2), prev(2), ink(2), inv(2), dpk, dpv;
    for (int l = 0; l < 2; ++l) {
      prek[l].assign(pk[l].begin(), pk[l].begin() + a * kvw);
      prev[l].assign(pv[l].begin(), pv[l].begin() + a * kvw);
      ink[l].assign(dk[l].begin() + a * kvw, dk[l].begin() + (a + len) * kvw);
      inv[l].assign(dv[l].begin() + a * kvw, dv[l].begin() + (a + len) * kvw);
    }
    cf::detail::segment_backward(model, cfg, tapes[s], a ? prek : decltype(prek){}, a ? prev : decltype(prev){}, &dpk,
                                 &dpv, &ink, &inv, static_cast<double>(n - 1));
    for (int l = 0; l < 2 && a > 0; ++l)
      for (size_t i = 0; i < static_cast<size_t>(a) * kvw; ++i) {
        dk[l][i] += dpk[l][i];
        dv[l][i] += dpv[l][i];
      }
  }
  double worst = 0;
  for (int64_t i = 0; i < nt; ++i) {
    std::vector<double> g(g_plan[static_cast<size_t>(i)].size());
    cf::check(cf_model_get_grad(model.get(), i, g.data()));
    for (size_t j = 0; j < g.size(); ++j) worst = std::fmax(worst, std::fabs(g[j] - g_plan[static_cast<size_t>(i)][j]));
  }
  std::printf("loss_diff=%g grad_diff=%g\n", loss_sum / (n - 1) - r.loss, worst);
  return 0;
}
