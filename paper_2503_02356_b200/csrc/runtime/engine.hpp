// Device runtime for the chunked training step: parameter/gradient storage,
// per-sequence KV state, retained-activation tapes and the event executor
// (the B200 counterpart of plan_runner.hpp:67-339).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "../../../include/chunkflow_b200.h"
#include "../host/plan.hpp"
#include "../kernels/attention.h"
#include "../kernels/ops.h"

namespace cfb {

using cfk::bf16;

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  cudaMemPool_t pool = nullptr;
  int64_t launches = 0;
  // data-parallel group (NCCL loaded at runtime)
  void* nccl_comm = nullptr;
  int rank = 0, world = 1;
  // per-launch CUDA-event timing (cf_ctx_set_profiling)
  bool profile = false;
  std::vector<cudaEvent_t> event_pool;
};

// One reference tensor (ToyModelParams::tensors order) and where it lives on
// the device: bf16 weights are stored [in,out] row-major exactly like the
// reference, q/k/v and gate/up column-fused into one matrix each.
struct Slot {
  std::string name;
  int64_t rows = 0, cols = 0;
  bool is_gain = false;  // fp32 RMSNorm gain (llama), initialised to 1
  void* w = nullptr;     // bf16* (weights) or float* (gains)
  float* g = nullptr;    // fp32 gradient (same layout)
  int64_t ld = 0;        // row pitch of the (fused) storage, elements
  int64_t draw_base = 0; // first SplitMix64 draw of this tensor
};

struct Layer {
  bf16* wqkv;  // [d, d+2kvw]
  bf16* wo;    // [d, d]
  bf16* w1;    // [d, gu_w]   llama: gate|up, toy: w1
  bf16* w2;    // [ffn, d]
  float* g1;   // [d] (llama)
  float* g2;
  float *d_wqkv, *d_wo, *d_w1, *d_w2, *d_g1, *d_g2;
};

struct Model {
  Ctx* ctx = nullptr;
  cf_model_cfg cfg{};
  bool llama = false;
  int64_t V, d, H, KVH, dh, kvw, ffn, L, qkv_w, gu_w;
  bf16* emb = nullptr;
  bf16* head = nullptr;
  float* gf = nullptr;
  float *d_emb = nullptr, *d_head = nullptr, *d_gf = nullptr;
  std::vector<Layer> layers;
  std::vector<Slot> slots;
  void* wbuf = nullptr;   // all weights (bf16) + gains (fp32)
  float* grads = nullptr; // all gradients, flat fp32
  int64_t grad_numel = 0, wbytes = 0, num_params = 0;
};

Model* model_create(Ctx* ctx, const cf_model_cfg& cfg);
void model_destroy(Model* m);
void model_get_param(Model* m, int64_t idx, double* host);
void model_set_param(Model* m, int64_t idx, const double* host);
void model_get_grad(Model* m, int64_t idx, double* host);

struct Batch {
  const int64_t* ids;
  const int64_t* lengths;
  const int32_t* tokens_host;  // may be null if tokens_dev given
  const int32_t* tokens_dev;
  int64_t n;
};

void run_plan(Ctx* ctx, Model* m, const Plan& plan, const Batch& b, const cf_run_opts& opts, cf_run_result* res);
cf_step* step_prepare(Ctx* ctx, Model* m, const Plan& plan, const Batch& b);
void step_run(Ctx* ctx, Model* m, cf_step* st, const cf_run_opts& opts, cf_run_result* res);
void step_destroy(cf_step* st);

void dp_init(Ctx* ctx, int rank, int world, const uint8_t* id128);
void dp_unique_id(uint8_t* out128);

}  // namespace cfb
