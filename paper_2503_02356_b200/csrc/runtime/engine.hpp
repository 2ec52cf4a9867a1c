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
#include "../kernels/optim.h"

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
  void* world_comm = nullptr;  // PP x DP: the communicator the groups are split from
  int rank = 0, world = 1;
  // pipeline-parallel links (cf_ctx_init_pp): one 2-rank communicator per
  // direction per neighbouring stage, each driven from its own stream, so
  // activation and gradient traffic never queue behind each other.
  int stage = 0, stages = 1;
  void* act_up = nullptr;    // send activations to stage+1
  void* grad_up = nullptr;   // receive gradients from stage+1
  void* act_down = nullptr;  // receive activations from stage-1
  void* grad_down = nullptr; // send gradients to stage-1
  cudaStream_t link_stream[4] = {nullptr, nullptr, nullptr, nullptr};
  // in-process pipeline (test transport): stages are contexts in one process
  // exchanging stage-boundary buffers through host mailboxes + CUDA events
  struct LocalPipe* local = nullptr;
  // per-launch CUDA-event timing (cf_ctx_set_profiling)
  bool profile = false;
  std::vector<cudaEvent_t> event_pool;
  // KV offload: host<->device copies of offloaded group state run here, and
  // the pinned host blocks are cached across steps
  cudaStream_t copy_stream = nullptr;
  // data-parallel gradient all-reduces overlapped with the last backward
  // (created on first use, released by cf_ctx_destroy)
  cudaStream_t dp_stream = nullptr;
  struct HostBlock {
    void* ptr;
    size_t bytes;
    bool busy;
  };
  std::vector<HostBlock> host_blocks;
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
  // pipeline stage slice: global layers [l_begin, l_end); embedding on the
  // first stage, final norm + head + loss on the last (L = local count)
  int64_t l_begin = 0, l_end = 0;
  bool has_embed = true, has_head = true;
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
  // gradient element ranges: layer l is [layer_goff[l], layer_goff[l+1]),
  // the embedding [0, layer_goff[0]), final norm + head [layer_goff[L], grad_numel)
  std::vector<int64_t> layer_goff;
  // AdamW state (cf_model_adamw_init): fp32 master weights and both moments in
  // the gradient buffer's layout, the storage-piece table the fused kernel
  // walks, and the step counter t
  std::vector<cfk::AdamPiece> pieces;
  void* opt_mem = nullptr;
  float *master = nullptr, *adam_m = nullptr, *adam_v = nullptr, *opt_scratch = nullptr, *clip_coef = nullptr;
  double* grad_norm = nullptr;
  cfk::AdamPiece* pieces_dev = nullptr;
  int64_t* block_start_dev = nullptr;
  int64_t opt_blocks = 0, opt_step = 0;
};

Model* model_create(Ctx* ctx, const cf_model_cfg& cfg, int64_t stage = 0, int64_t stages = 1);
void model_destroy(Model* m);
void model_get_param(Model* m, int64_t idx, double* host);
void model_set_param(Model* m, int64_t idx, const double* host);
void model_get_grad(Model* m, int64_t idx, double* host);
// AdamW (cf_model_adamw_*): state init from the current weights, one fused
// step over the flat gradient buffer, master-weight read-back.
void model_adamw_init(Model* m);
void model_adamw_step(Model* m, const cf_adamw_cfg& cfg, double* grad_norm);
void model_get_master(Model* m, int64_t idx, double* host);

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
// Operator level (detail::segment_forward / segment_backward,
// toy_model.hpp:206, :341): one segment of one sequence with a caller-held
// prefix.  K/V and their gradients are host fp64 [L][rows][kv_width].
struct SegmentState;
SegmentState* segment_forward(Ctx* ctx, Model* m, const int32_t* tokens, int64_t len, const int64_t* targets,
                              const double* prefix_k, const double* prefix_v, int64_t prefix_len, bool keep_tape,
                              double* loss_sum, double* saved_k, double* saved_v);
void segment_backward(Ctx* ctx, Model* m, SegmentState* sg, const double* prefix_k, const double* prefix_v,
                      double* d_prefix_k, double* d_prefix_v, const double* incoming_dk, const double* incoming_dv,
                      double normalizer);
void segment_destroy(SegmentState* sg);
void step_op_times(const cf_step* st, int64_t* n, int64_t* kinds, int64_t* ids, double* ms);
int64_t step_input_bytes(const cf_step* st);
// Pipeline-parallel step of one stage on this rank (ctx has PP links): the
// stage's chunk-aware 1F1B op stream (host/pp.hpp) with NCCL send/recv of
// fp32 [T, d] activations and gradients.
void pp_step_run(Ctx* ctx, Model* m, cf_step* st, int64_t k, const cf_run_opts& opts, cf_run_result* res);
// All stages of one pipeline in this process on one device (stage i uses
// models[i]): the same per-stage op streams, executed in dispatch order with
// in-memory hand-over between stages.  Results are summed over stages (loss
// and loss checks come from the last stage).
void pp_step_run_local(Ctx* ctx, Model* const* models, int64_t stages, cf_step* st, int64_t k,
                       const cf_run_opts& opts, cf_run_result* res);
void pp_init(Ctx* ctx, int rank, int world, int stages, const uint8_t* id128);
// In-process links for cf_pp_step_run: every stage's context (one host thread
// each) attaches to one LocalPipe; same op streams and buffer life cycle as
// the NCCL links, with device-to-device copies instead of ncclSend/Recv.
struct LocalPipe;
LocalPipe* local_pipe_create(int stages);
void local_pipe_destroy(LocalPipe* p);
void pp_init_local(Ctx* ctx, LocalPipe* p, int stage);

void dp_init(Ctx* ctx, int rank, int world, const uint8_t* id128);
void ctx_release(Ctx* ctx);
void dp_unique_id(uint8_t* out128);

}  // namespace cfb
