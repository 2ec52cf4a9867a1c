// C-ABI: device context, model, execution and operator-level entry points.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "../../../include/chunkflow_b200.h"
#include "../kernels/attention_tc.h"
#include "../kernels/gemm.h"
#include "../runtime/engine.hpp"
#include "capi_util.hpp"

struct cf_ctx {
  cfb::Ctx c;
};
struct cf_model {
  cfb::Model* m = nullptr;
  cf_ctx* ctx = nullptr;
};
struct cf_segment {
  cfb::SegmentState* s = nullptr;
};
namespace {
void need(const void* p, const char* what) {
  if (!p) throw cfb::ValidationError(std::string(what) + " is null");
}
// Every entry point that touches a context makes its device current, so two
// contexts on different GPUs can be driven from one host thread.
void need(const cf_ctx* c, const char* what) {
  need(static_cast<const void*>(c), what);
  cfb::cuda_check(cudaSetDevice(c->c.device), "cudaSetDevice");
}
void need(const cf_model* m, const char* what) {
  need(static_cast<const void*>(m), what);
  if (m->ctx) cfb::cuda_check(cudaSetDevice(m->ctx->c.device), "cudaSetDevice");
}
}  // namespace

extern "C" {

int cf_ctx_create(int device, cf_ctx** out) {
  return cfb::guard([&] {
    need(out, "out");
    int n = 0;
    cfb::cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) throw cfb::ValidationError("no CUDA device " + std::to_string(device));
    cfb::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    cfb::cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10) throw cfb::ValidationError("chunkflow_b200 requires an sm_100 (B200) device");
    auto h = std::make_unique<cf_ctx>();
    h->c.device = device;
    h->c.num_sms = prop.multiProcessorCount;
    cfb::cuda_check(cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cfb::cuda_check(cudaDeviceGetDefaultMemPool(&h->c.pool, device), "cudaDeviceGetDefaultMemPool");
    uint64_t keep = UINT64_MAX;  // keep freed blocks cached across chunks/steps
    cfb::cuda_check(cudaMemPoolSetAttribute(h->c.pool, cudaMemPoolAttrReleaseThreshold, &keep), "pool attr");
    *out = h.release();
  });
}

void cf_ctx_destroy(cf_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  cfb::ctx_release(&ctx->c);  // NCCL communicators, link streams, timing events
  cudaStreamDestroy(ctx->c.stream);
  delete ctx;
}

void* cf_ctx_stream(cf_ctx* ctx) { return ctx ? static_cast<void*>(ctx->c.stream) : nullptr; }

int cf_ctx_set_profiling(cf_ctx* ctx, int on) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    ctx->c.profile = on != 0;
  });
}

int cf_ctx_synchronize(cf_ctx* ctx) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    cfb::cuda_check(cudaStreamSynchronize(ctx->c.stream), "cudaStreamSynchronize");
  });
}

int cf_nccl_unique_id(uint8_t* out128) {
  return cfb::guard([&] {
    need(out128, "out");
    cfb::dp_unique_id(out128);
  });
}

int cf_ctx_init_dp(cf_ctx* ctx, int rank, int world, const uint8_t* id128) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    if (world < 1 || rank < 0 || rank >= world) throw cfb::ValidationError("bad rank/world");
    if (world > 1) need(id128, "nccl id");
    cfb::dp_init(&ctx->c, rank, world, id128);
  });
}

int cf_model_create(cf_ctx* ctx, const cf_model_cfg* cfg, cf_model** out) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(cfg, "cfg");
    auto h = std::make_unique<cf_model>();
    h->ctx = ctx;
    h->m = cfb::model_create(&ctx->c, *cfg);
    *out = h.release();
  });
}

int cf_model_create_stage(cf_ctx* ctx, const cf_model_cfg* cfg, int64_t stage, int64_t num_stages, cf_model** out) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(cfg, "cfg");
    need(out, "out");
    auto h = std::make_unique<cf_model>();
    h->ctx = ctx;
    h->m = cfb::model_create(&ctx->c, *cfg, stage, num_stages);
    *out = h.release();
  });
}

int cf_ctx_init_pp(cf_ctx* ctx, int rank, int world, int num_stages, const uint8_t* id128) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(id128, "nccl id");
    cfb::pp_init(&ctx->c, rank, world, num_stages, id128);
  });
}

struct cf_pp_local {
  cfb::LocalPipe* p = nullptr;
};

int cf_pp_local_create(int num_stages, cf_pp_local** out) {
  return cfb::guard([&] {
    need(out, "out");
    auto h = std::make_unique<cf_pp_local>();
    h->p = cfb::local_pipe_create(num_stages);
    *out = h.release();
  });
}

void cf_pp_local_destroy(cf_pp_local* pipe) {
  if (!pipe) return;
  cfb::local_pipe_destroy(pipe->p);
  delete pipe;
}

int cf_ctx_init_pp_local(cf_ctx* ctx, cf_pp_local* pipe, int stage) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(pipe, "pipe");
    cfb::pp_init_local(&ctx->c, pipe->p, stage);
  });
}

int cf_pp_step_run(cf_ctx* ctx, cf_model* model, cf_step* step, int64_t k, const cf_run_opts* opts,
                   cf_run_result* result) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(model, "model");
    need(step, "step");
    cf_run_opts o{};
    if (opts) o = *opts;
    cfb::pp_step_run(&ctx->c, model->m, step, k, o, result);
  });
}

int cf_pp_run_local(cf_ctx* ctx, cf_model* const* models, int64_t num_stages, cf_step* step, int64_t k,
                    const cf_run_opts* opts, cf_run_result* result) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(models, "models");
    need(step, "step");
    if (num_stages < 1) throw cfb::ValidationError("num_stages must be at least 1");
    std::vector<cfb::Model*> ms;
    for (int64_t s = 0; s < num_stages; ++s) {
      need(models[s], "models[i]");
      ms.push_back(models[s]->m);
    }
    cf_run_opts o{};
    if (opts) o = *opts;
    cfb::pp_step_run_local(&ctx->c, ms.data(), num_stages, step, k, o, result);
  });
}

void cf_model_destroy(cf_model* model) {
  if (!model) return;
  cfb::model_destroy(model->m);
  delete model;
}

int64_t cf_model_num_tensors(const cf_model* model) {
  return model ? static_cast<int64_t>(model->m->slots.size()) : -1;
}
int64_t cf_model_num_params(const cf_model* model) { return model ? model->m->num_params : -1; }

int cf_model_tensor_info(const cf_model* model, int64_t idx, char* name, size_t cap, int64_t* rows, int64_t* cols) {
  return cfb::guard([&] {
    need(model, "model");
    if (idx < 0 || idx >= static_cast<int64_t>(model->m->slots.size()))
      throw cfb::ValidationError("tensor index out of range");
    const cfb::Slot& s = model->m->slots[static_cast<size_t>(idx)];
    if (rows) *rows = s.rows;
    if (cols) *cols = s.cols;
    if (name && cap) {
      const size_t n = std::min(cap - 1, s.name.size());
      std::memcpy(name, s.name.data(), n);
      name[n] = 0;
    }
  });
}

int cf_model_get_param(cf_model* model, int64_t idx, double* host) {
  return cfb::guard([&] {
    need(model, "model");
    need(host, "host");
    cfb::model_get_param(model->m, idx, host);
  });
}
int cf_model_set_param(cf_model* model, int64_t idx, const double* host) {
  return cfb::guard([&] {
    need(model, "model");
    need(host, "host");
    cfb::model_set_param(model->m, idx, host);
  });
}
int cf_model_get_grad(cf_model* model, int64_t idx, double* host) {
  return cfb::guard([&] {
    need(model, "model");
    need(host, "host");
    cfb::model_get_grad(model->m, idx, host);
  });
}
int cf_model_adamw_init(cf_model* model) {
  return cfb::guard([&] {
    need(model, "model");
    cfb::model_adamw_init(model->m);
  });
}
int cf_model_adamw_step(cf_model* model, const cf_adamw_cfg* cfg, double* grad_norm) {
  return cfb::guard([&] {
    need(model, "model");
    need(cfg, "cfg");
    cfb::model_adamw_step(model->m, *cfg, grad_norm);
  });
}
int cf_model_get_master(cf_model* model, int64_t idx, double* host) {
  return cfb::guard([&] {
    need(model, "model");
    need(host, "host");
    cfb::model_get_master(model->m, idx, host);
  });
}
int cf_model_zero_grads(cf_model* model) {
  return cfb::guard([&] {
    need(model, "model");
    cfb::cuda_check(cudaMemsetAsync(model->m->grads, 0, static_cast<size_t>(model->m->grad_numel) * 4,
                                    model->ctx->c.stream),
                    "memset");
  });
}
int cf_model_grad_buffer(cf_model* model, void** dev_ptr, int64_t* numel) {
  return cfb::guard([&] {
    need(model, "model");
    if (dev_ptr) *dev_ptr = model->m->grads;
    if (numel) *numel = model->m->grad_numel;
  });
}

int cf_run_plan(cf_ctx* ctx, cf_model* model, const cf_plan* plan, const int64_t* seq_ids, const int64_t* lengths,
                const int32_t* tokens, int64_t n, const cf_run_opts* opts, cf_run_result* result) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(model, "model");
    need(plan, "plan");
    cf_run_opts o{};
    if (opts) o = *opts;
    cfb::Batch b{seq_ids, lengths, tokens, nullptr, n};
    cfb::run_plan(&ctx->c, model->m, plan->p, b, o, result);
  });
}

int cf_step_prepare(cf_ctx* ctx, cf_model* model, const cf_plan* plan, const int64_t* seq_ids,
                    const int64_t* lengths, const int32_t* tokens, int64_t n, cf_step** out) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(model, "model");
    need(plan, "plan");
    cfb::Batch b{seq_ids, lengths, tokens, nullptr, n};
    *out = cfb::step_prepare(&ctx->c, model->m, plan->p, b);
  });
}

int cf_step_run(cf_ctx* ctx, cf_model* model, cf_step* step, const cf_run_opts* opts, cf_run_result* result) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(model, "model");
    need(step, "step");
    cf_run_opts o{};
    if (opts) o = *opts;
    cfb::step_run(&ctx->c, model->m, step, o, result);
  });
}

void cf_step_destroy(cf_step* step) { cfb::step_destroy(step); }

int cf_step_input_bytes(const cf_step* step, int64_t* bytes) {
  return cfb::guard([&] {
    need(step, "step");
    need(bytes, "bytes");
    *bytes = cfb::step_input_bytes(step);
  });
}

int cf_step_op_times(const cf_step* step, int64_t* n, int64_t* kinds, int64_t* chunk_ids, double* ms) {
  return cfb::guard([&] {
    need(step, "step");
    need(n, "n");
    cfb::step_op_times(step, n, kinds, chunk_ids, ms);
  });
}

int cf_backward_full(cf_ctx* ctx, cf_model* model, const int64_t* seq_ids, const int64_t* lengths,
                     const int32_t* tokens, int64_t n, double normalizer_override, cf_run_result* result) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(model, "model");
    // backward_full: each sequence is its own standalone chunk of one
    // segment (no packing, no prefix), forward then backward.
    cfb::Plan p;
    p.chunk_size = 0;
    for (int64_t i = 0; i < n; ++i) {
      cfb::Chunk c;
      c.id = i;
      c.kind = cfb::kStandalone;
      c.total = lengths[i];
      c.seg_off = i;
      c.seg_cnt = 1;
      p.segments.push_back({seq_ids[i], 0, lengths[i]});
      p.index_of[i] = i;
      p.chunk_tokens[i] = lengths[i];
      p.chunk_size = std::max(p.chunk_size, lengths[i]);
      p.chunks.push_back(c);
    }
    cfb::schedule_step(p, 1);
    cf_run_opts o{};
    o.normalizer_override = normalizer_override;
    cfb::Batch b{seq_ids, lengths, tokens, nullptr, n};
    cfb::run_plan(&ctx->c, model->m, p, b, o, result);
  });
}

int cf_segment_forward(cf_ctx* ctx, cf_model* model, const int32_t* tokens, int64_t len, const int64_t* targets,
                       const double* prefix_k, const double* prefix_v, int64_t prefix_len, int keep_tape,
                       double* loss_sum, double* saved_k, double* saved_v, cf_segment** tape) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(model, "model");
    if (tape) *tape = nullptr;
    if (keep_tape && !tape) throw cfb::ValidationError("tape out-pointer required when keep_tape is set");
    cfb::SegmentState* s = cfb::segment_forward(&ctx->c, model->m, tokens, len, targets, prefix_k, prefix_v,
                                                prefix_len, keep_tape != 0, loss_sum, saved_k, saved_v);
    if (s) {
      auto h = std::make_unique<cf_segment>();
      h->s = s;
      *tape = h.release();
    }
  });
}

int cf_segment_backward(cf_ctx* ctx, cf_model* model, const cf_segment* tape, const double* prefix_k,
                        const double* prefix_v, double* d_prefix_k, double* d_prefix_v, const double* incoming_dk,
                        const double* incoming_dv, double normalizer) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    need(model, "model");
    if (!tape) throw cfb::ValidationError("segment backward requires a retained tape");
    cfb::segment_backward(&ctx->c, model->m, tape->s, prefix_k, prefix_v, d_prefix_k, d_prefix_v, incoming_dk,
                          incoming_dv, normalizer);
  });
}

void cf_segment_destroy(cf_segment* tape) {
  if (!tape) return;
  cfb::segment_destroy(tape->s);
  delete tape;
}

int cf_op_attention(cf_ctx* ctx, int impl, int backward, const void* q, int64_t q_stride, const void* k,
                    const void* v, int64_t kv_stride, int64_t kv_rows, void* o, float* lse, const void* dout,
                    void* dq, float* dk_acc, float* dv_acc, int64_t acc_stride, const int32_t* segs, int64_t nseg,
                    int64_t T, int64_t H, int64_t KVH, int64_t dh) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    std::vector<int32_t> meta(segs, segs + 4 * nseg);
    auto tiles = [&](int rows, bool keys) {
      const int64_t off = static_cast<int64_t>(meta.size());
      int64_t n = 0;
      for (int64_t s = 0; s < nseg; ++s) {
        const int32_t len = segs[4 * s + 1], prefix = segs[4 * s + 3];
        const int32_t total = keys ? prefix + len : len;
        for (int32_t f = 0; f < total; f += rows) {
          meta.insert(meta.end(), {static_cast<int32_t>(s), f, std::min(rows, total - f), 0});
          ++n;
        }
      }
      return std::make_pair(off, n);
    };
    const auto q64 = tiles(64, false), k64 = tiles(64, true), q128 = tiles(128, false), k128 = tiles(128, true);
    int32_t* dmeta = nullptr;
    cudaStream_t st = ctx->c.stream;
    cfb::cuda_check(cudaMallocAsync(&dmeta, meta.size() * 4, st), "malloc");
    cfb::cuda_check(cudaMemcpyAsync(dmeta, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice, st), "h2d");
    cfk::AttnParams p{};
    p.q = static_cast<const cfk::bf16*>(q);
    p.q_stride = q_stride;
    p.k = static_cast<const cfk::bf16*>(k);
    p.v = static_cast<const cfk::bf16*>(v);
    p.kv_stride = kv_stride;
    p.o = static_cast<cfk::bf16*>(o);
    p.o_stride = H * dh;
    p.lse = lse;
    p.dout = static_cast<const cfk::bf16*>(dout);
    p.dout_stride = H * dh;
    p.dq = static_cast<cfk::bf16*>(dq);
    p.dq_stride = H * dh;
    p.dk_acc = dk_acc;
    p.dv_acc = dv_acc;
    p.acc_stride = acc_stride;
    p.segs = reinterpret_cast<const cfk::AttnSeg*>(dmeta);
    p.tiles = reinterpret_cast<const cfk::AttnTile*>(dmeta + q64.first);
    p.num_tiles = static_cast<int32_t>(q64.second);
    p.T = static_cast<int32_t>(T);
    p.H = static_cast<int32_t>(H);
    p.KVH = static_cast<int32_t>(KVH);
    p.dh = static_cast<int32_t>(dh);
    p.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(dh)));
    float* dsum = nullptr;
    cfb::cuda_check(cudaMallocAsync(&dsum, static_cast<size_t>(T * H) * 4, st), "malloc");
    p.dsum = dsum;
    cudaError_t e;
    if (!backward) {
      if (impl == 3) {
        if (!cfk::attn_fwd_pp_supported(p))
          throw cfb::ValidationError("ping-pong attention needs head_dim 128 and an even GQA group");
        e = cfk::attn_forward_tc_pp(p, reinterpret_cast<const cfk::AttnTile*>(dmeta + q128.first),
                                    static_cast<int32_t>(q128.second), kv_rows, st);
      } else if (impl == 1) {
        if (!cfk::attn_tc_supported(p)) throw cfb::ValidationError("tcgen05 attention needs head_dim 128");
        e = cfk::attn_forward_tc(p, reinterpret_cast<const cfk::AttnTile*>(dmeta + q128.first),
                                 static_cast<int32_t>(q128.second), kv_rows, st);
      } else {
        e = cfk::attn_forward(p, st);
      }
    } else if (impl == 1 || impl == 2) {
      if (!cfk::attn_tc_supported(p)) throw cfb::ValidationError("tcgen05 attention needs head_dim 128");
      auto fn = impl == 1 ? cfk::attn_backward_tc : cfk::attn_backward_tc_v1;
      e = fn(p, reinterpret_cast<const cfk::AttnTile*>(dmeta + q128.first), static_cast<int32_t>(q128.second),
             reinterpret_cast<const cfk::AttnTile*>(dmeta + k128.first), static_cast<int32_t>(k128.second), kv_rows,
             st);
    } else {
      e = cfk::attn_backward(p, reinterpret_cast<const cfk::AttnTile*>(dmeta + k64.first),
                             static_cast<int32_t>(k64.second), st);
    }
    cfb::cuda_check(e, "attention");
    cudaFreeAsync(dsum, st);
    cudaFreeAsync(dmeta, st);
    cfb::cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

int cf_op_gemm(cf_ctx* ctx, const void* a, int a_kmajor, int64_t lda, const void* b, int b_kmajor, int64_t ldb,
               void* c, int64_t ldc, int64_t m, int64_t n, int64_t k, int epi, const void* residual, int64_t ld_res) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    cfk::GemmDesc d{a, lda, a_kmajor, b, ldb, b_kmajor, c, ldc, residual, ld_res, m, n, k, epi};
    cfb::cuda_check(cfk::gemm(d, ctx->c.stream), "gemm");
    ctx->c.launches += 1;
  });
}

int cf_op_lm_head_ce(cf_ctx* ctx, const void* x, const void* head, int64_t ldh, int64_t T, int64_t V, int64_t d,
                     const int32_t* targets, float inv_norm, float* lse, float* row_loss, void* dlogits) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    if (!x || !head || !targets || !lse || !row_loss) throw cfb::ValidationError("null operand");
    cudaStream_t st = ctx->c.stream;
    const int64_t np = cfk::ce_nparts(V);
    float* buf = nullptr;
    cfb::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&buf), static_cast<size_t>(T * np * 8 + T * 4 + 256), st),
                    "cudaMallocAsync");
    cfk::GemmDesc g{x, d, 1, head, ldh, 0, nullptr, 0, nullptr, 0, T, V, d, cfk::EPI_CE_STATS};
    g.ce_tgt = targets;
    g.ce_part = buf;
    g.ce_tlogit = buf + T * np * 2;
    cudaError_t e = cfk::gemm(g, st);
    if (e == cudaSuccess) e = cfk::ce_finish(buf, np, buf + T * np * 2, targets, T, lse, row_loss, st);
    if (e == cudaSuccess && dlogits) {
      cfk::GemmDesc b{x, d, 1, head, ldh, 0, dlogits, ldh, nullptr, 0, T, V, d, cfk::EPI_CE_GRAD};
      b.ce_tgt = targets;
      b.ce_lse = lse;
      b.ce_scale = inv_norm;
      e = cfk::gemm(b, st);
    }
    cudaFreeAsync(buf, st);
    cfb::cuda_check(e, "lm_head_ce");
    ctx->c.launches += dlogits ? 3 : 2;
  });
}

int cf_op_gemm_rope(cf_ctx* ctx, const void* a, int64_t lda, const void* w, int64_t ldw, void* c, int64_t m,
                    int64_t n, int64_t k, const void* tab, int64_t col_k, int64_t col_v, void* kc, void* vc,
                    int64_t cache_ld) {
  return cfb::guard([&] {
    need(ctx, "ctx");
    cfk::GemmDesc d{a, lda, 1, w, ldw, 0, c, n, tab, 64, m, n, k, cfk::EPI_BF16_ROPE};
    d.col_k = col_k;
    d.col_v = col_v;
    d.kc = kc;
    d.vc = vc;
    d.cache_ld = cache_ld;
    cfb::cuda_check(cfk::gemm(d, ctx->c.stream), "gemm_rope");
    ctx->c.launches += 1;
  });
}

}  // extern "C"

extern "C" int cf_debug_set_attn_stress(int on) {
  return cfb::guard([&] { cfk::set_attn_stress(on); });
}

extern "C" int cf_debug_set_gemm_mode(int mode) {
  return cfb::guard([&] {
    if (mode < 0 || mode > 2) throw cfb::ValidationError("gemm mode must be 0, 1 or 2");
    cfk::set_gemm_mode(mode);
  });
}
