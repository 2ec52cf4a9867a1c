// Device runtime: model storage + the chunk event executor.
//
// Mirrors run_plan (reference plan_runner.hpp:67-339) event by event, but
// with B200 data structures instead of the reference's StateStore copies:
//  * per dependent group, one contiguous KV cache [L][S][kvw] (bf16 K, V)
//    and one fp32 KV-gradient store [L][S][2*kvw] (dK | dV) for the whole
//    sequence.  A forward writes its own K/V rows in place (replaces
//    save_kv + assemble_prefix, plan_runner.hpp:128-156/206-217); attention
//    reads the prefix straight from the cache; a backward adds dK/dV for
//    every key row [0, start+T) in place (replaces the dKV scatter,
//    :306-321) and then consumes its own rows (incoming from later chunks +
//    its own contribution, :488-495).
//  * retained activations ("tapes") live in stream-ordered pool memory from a
//    retain-forward until the chunk's backward, so at most K chunks' tapes
//    are resident (Alg. 2).
//  * losses are reduced on the device in a fixed order into per-event slots,
//    read back once per step; recompute-loss equality is checked bitwise.
#include <algorithm>
#include <functional>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <memory>
#include <numeric>
#include <set>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <tuple>

#include "../capi/capi_util.hpp"
#include "../kernels/attention_tc.h"
#include "../kernels/gemm.h"
#include "../host/pp.hpp"
#include "engine.hpp"

namespace cfb {

using cfk::AttnParams;
using cfk::AttnSeg;
using cfk::AttnTile;
using cfk::bf16;

#define CK(expr) cuda_check((expr), #expr)

namespace {

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Bump allocator over one pool allocation.
struct Arena {
  char* base = nullptr;
  int64_t off = 0;
  template <class T>
  T* take(int64_t count) {
    off = align_up(off, 256);
    T* p = reinterpret_cast<T*>(base + off);
    off += count * static_cast<int64_t>(sizeof(T));
    return p;
  }
};

// Stream-ordered pool allocation.  The pool keeps freed blocks (release
// threshold = max) so per-chunk scratch is a lookup; when a request does not
// fit next to the cached blocks of other sizes, the cache is released
// (after the stream drains) and the request retried once.
void* pool_alloc(Ctx* c, int64_t bytes) {
  void* p = nullptr;
  const size_t n = static_cast<size_t>(std::max<int64_t>(bytes, 256));
  cudaError_t e = cudaMallocAsync(&p, n, c->stream);
  if (e == cudaErrorMemoryAllocation && c->pool) {
    (void)cudaGetLastError();
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemPoolTrimTo(c->pool, 0));
    e = cudaMallocAsync(&p, n, c->stream);
  }
  CK(e);
  return p;
}
void pool_free(Ctx* c, void* p) {
  if (p) CK(cudaFreeAsync(p, c->stream));
}

// Pinned host blocks for offloaded KV state, cached on the context across
// steps (page-locking tens of GB costs seconds; a block is reused by any
// later group that fits).
void* host_acquire(Ctx* c, size_t bytes) {
  for (auto& b : c->host_blocks)
    if (!b.busy && b.bytes >= bytes) {
      b.busy = true;
      return b.ptr;
    }
  void* p = nullptr;
  CK(cudaMallocHost(&p, bytes));
  c->host_blocks.push_back({p, bytes, true});
  return p;
}
void host_release(Ctx* c, void* p) {
  for (auto& b : c->host_blocks)
    if (b.ptr == p) b.busy = false;
}
cudaEvent_t new_timing_free_event() {
  cudaEvent_t e;
  CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

// --------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  void* h = nullptr;
  int (*get_id)(void*) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*err)(int) = nullptr;
  void* init_rank = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*split)(void*, int, int, void**, void*) = nullptr;  // ncclCommSplit (NCCL >= 2.18)
  int (*destroy)(void*) = nullptr;                          // ncclCommDestroy
};
struct Id128 {
  char b[128];
};
Nccl& nccl() {
  static Nccl n;
  if (!n.h) {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) throw NcclError("libnccl.so.2 not loadable");
    n.get_id = reinterpret_cast<int (*)(void*)>(dlsym(n.h, "ncclGetUniqueId"));
    n.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(n.h, "ncclAllReduce"));
    n.err = reinterpret_cast<const char* (*)(int)>(dlsym(n.h, "ncclGetErrorString"));
    n.init_rank = dlsym(n.h, "ncclCommInitRank");
    n.send = reinterpret_cast<int (*)(const void*, size_t, int, int, void*, cudaStream_t)>(dlsym(n.h, "ncclSend"));
    n.recv = reinterpret_cast<int (*)(void*, size_t, int, int, void*, cudaStream_t)>(dlsym(n.h, "ncclRecv"));
    n.split = reinterpret_cast<int (*)(void*, int, int, void**, void*)>(dlsym(n.h, "ncclCommSplit"));
    n.destroy = reinterpret_cast<int (*)(void*)>(dlsym(n.h, "ncclCommDestroy"));
    if (!n.get_id || !n.all_reduce || !n.init_rank) throw NcclError("NCCL symbols missing");
  }
  return n;
}
void nccl_check(int r, const char* what) {
  if (r != 0) throw NcclError(std::string(what) + ": " + (nccl().err ? nccl().err(r) : "error"));
}
constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0, kNcclNoColor = -1;

}  // namespace

void dp_unique_id(uint8_t* out) { nccl_check(nccl().get_id(out), "ncclGetUniqueId"); }

// Releases what a context acquired beyond its stream (cf_ctx_destroy): every
// NCCL communicator (world, DP group, the four stage links), the link
// streams and the profiling events.  Never throws.
void ctx_release(Ctx* ctx) {
  void* comms[] = {ctx->nccl_comm, ctx->world_comm, ctx->act_up, ctx->grad_up, ctx->act_down, ctx->grad_down};
  std::set<void*> seen;
  for (void* c : comms)
    if (c && seen.insert(c).second && nccl().destroy) nccl().destroy(c);
  ctx->nccl_comm = ctx->world_comm = ctx->act_up = ctx->grad_up = ctx->act_down = ctx->grad_down = nullptr;
  for (auto& ls : ctx->link_stream)
    if (ls) {
      cudaStreamSynchronize(ls);
      cudaStreamDestroy(ls);
      ls = nullptr;
    }
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  ctx->event_pool.clear();
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
    ctx->copy_stream = nullptr;
  }
  if (ctx->dp_stream) {
    cudaStreamSynchronize(ctx->dp_stream);
    cudaStreamDestroy(ctx->dp_stream);
    ctx->dp_stream = nullptr;
  }
  for (auto& b : ctx->host_blocks) cudaFreeHost(b.ptr);
  ctx->host_blocks.clear();
}

void dp_init(Ctx* ctx, int rank, int world, const uint8_t* id) {
  // world == 1 without an id: no communicator.  With an id, a 1-rank NCCL
  // communicator is created (exercises the full DP path on one GPU).
  if (world <= 1 && !id) return;
  Id128 u;
  std::memcpy(u.b, id, 128);
  auto init = reinterpret_cast<int (*)(void**, int, Id128, int)>(nccl().init_rank);
  CK(cudaSetDevice(ctx->device));
  nccl_check(init(&ctx->nccl_comm, world, u, rank), "ncclCommInitRank");
  ctx->rank = rank;
  ctx->world = world;
}

// Pipeline x data parallel layout (config C5): rank = replica * stages +
// stage.  From one world communicator: the DP group of each stage (same
// stage across replicas) and, for every neighbouring stage pair of a
// replica, two 2-rank links (activations up, gradients down), each used by
// exactly one sender and one receiver in the same op order on both sides —
// forwards in plan order, backwards in backward-queue order — so the
// streams of different links can never wait on each other in a cycle.
void pp_init(Ctx* ctx, int rank, int world, int stages, const uint8_t* id) {
  if (stages < 1 || world % stages) throw ValidationError("world size must be a multiple of the stage count");
  if (rank < 0 || rank >= world) throw ValidationError("bad rank");
  Nccl& n = nccl();
  if (!n.split || !n.send || !n.recv) throw NcclError("NCCL without ncclCommSplit/ncclSend/ncclRecv");
  Id128 u;
  std::memcpy(u.b, id, 128);
  auto init = reinterpret_cast<int (*)(void**, int, Id128, int)>(n.init_rank);
  CK(cudaSetDevice(ctx->device));
  void* world_comm = nullptr;
  nccl_check(init(&world_comm, world, u, rank), "ncclCommInitRank");
  ctx->world_comm = world_comm;  // kept so cf_ctx_destroy can release it
  const int s = rank % stages, rep = rank / stages, dp = world / stages;
  ctx->stage = s;
  ctx->stages = stages;
  void* dpc = nullptr;
  nccl_check(n.split(world_comm, s, rep, &dpc, nullptr), "ncclCommSplit(dp)");
  if (dp > 1) {
    ctx->nccl_comm = dpc;
    ctx->rank = rep;
    ctx->world = dp;
  } else if (dpc && n.destroy) {
    n.destroy(dpc);  // a 1-rank DP group is not used
  }
  // link j joins stages j and j+1 of a replica; even links first, then odd
  auto link_color = [&](int parity) {
    if (s % 2 == parity && s + 1 < stages) return rep * stages + s;  // lower end of link s
    if (s % 2 != parity && s > 0) return rep * stages + s - 1;       // upper end of link s-1
    return kNcclNoColor;
  };
  for (int parity = 0; parity < 2; ++parity)
    for (int dir = 0; dir < 2; ++dir) {
      void* c = nullptr;
      nccl_check(n.split(world_comm, link_color(parity), s, &c, nullptr), "ncclCommSplit(link)");
      if (!c) continue;
      const bool up = s % 2 == parity;  // this link goes to stage s+1
      if (up)
        (dir == 0 ? ctx->act_up : ctx->grad_up) = c;
      else
        (dir == 0 ? ctx->act_down : ctx->grad_down) = c;
    }
  for (auto& ls : ctx->link_stream)
    if (!ls) CK(cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking));
}

// ------------------------------------------------------------------ model
Model* model_create(Ctx* ctx, const cf_model_cfg& cfg, int64_t stage, int64_t stages) {
  auto m = std::make_unique<Model>();
  m->ctx = ctx;
  m->cfg = cfg;
  m->llama = cfg.arch == CF_ARCH_LLAMA;
  if (cfg.arch != CF_ARCH_TOY && cfg.arch != CF_ARCH_LLAMA) throw ValidationError("unknown arch");
  if (cfg.vocab_size < 1 || cfg.d_model < 1 || cfg.num_heads < 1 || cfg.num_kv_heads < 1 || cfg.num_layers < 1)
    throw ValidationError("model dimensions must be positive");
  if (cfg.d_model % cfg.num_heads) throw ValidationError("d_model must be divisible by num_heads");
  if (cfg.num_heads % cfg.num_kv_heads) throw ValidationError("num_heads must be divisible by num_kv_heads");
  m->V = cfg.vocab_size;
  m->d = cfg.d_model;
  m->H = cfg.num_heads;
  m->KVH = cfg.num_kv_heads;
  m->dh = m->d / m->H;
  m->kvw = m->KVH * m->dh;
  pp_stage_layers(cfg.num_layers, stage, stages, &m->l_begin, &m->l_end);
  m->L = m->l_end - m->l_begin;
  m->has_embed = stage == 0;
  m->has_head = stage == stages - 1;
  m->ffn = m->llama ? cfg.ffn_width : 2 * m->d;
  if (m->ffn < 1) throw ValidationError("llama arch needs ffn_width");
  if (m->llama && (m->dh % 2)) throw ValidationError("RoPE needs an even head dim");
  if (m->dh > 128) throw ValidationError("head_dim > 128 not supported");
  if (m->d % 8 || m->kvw % 8 || m->ffn % 8)
    throw ValidationError("d_model, kv width and ffn width must be multiples of 8 (16-byte TMA rows)");
  m->qkv_w = m->d + 2 * m->kvw;
  m->gu_w = m->llama ? 2 * m->ffn : m->ffn;
  const int64_t Vp = align_up(m->V, 8);

  // Storage plan: weights (bf16) then gains (fp32), each 256-byte aligned;
  // gradients (fp32) mirror the weight layout in one flat buffer.
  struct Piece {
    int64_t elems;
    bool f32;
  };
  std::vector<Piece> pieces;
  if (m->has_embed) pieces.push_back({m->V * m->d, false});  // emb
  for (int64_t l = 0; l < m->L; ++l) {
    pieces.push_back({m->d * m->qkv_w, false});
    pieces.push_back({m->d * m->d, false});
    pieces.push_back({m->d * m->gu_w, false});
    pieces.push_back({m->ffn * m->d, false});
    if (m->llama) {
      pieces.push_back({m->d, true});
      pieces.push_back({m->d, true});
    }
  }
  if (m->has_head) {
    if (m->llama) pieces.push_back({m->d, true});
    pieces.push_back({m->d * Vp, false});  // head [d, Vp]
  }
  int64_t wbytes = 0, gelems = 0;
  std::vector<int64_t> woff, goff;
  for (const Piece& p : pieces) {
    wbytes = align_up(wbytes, 256);
    woff.push_back(wbytes);
    wbytes += p.elems * (p.f32 ? 4 : 2);
    gelems = align_up(gelems, 64);
    goff.push_back(gelems);
    gelems += p.elems;
  }
  CK(cudaMalloc(&m->wbuf, static_cast<size_t>(wbytes)));
  CK(cudaMalloc(&m->grads, static_cast<size_t>(gelems) * 4));
  CK(cudaMemsetAsync(m->grads, 0, static_cast<size_t>(gelems) * 4, ctx->stream));
  m->wbytes = wbytes;
  m->grad_numel = gelems;
  char* wb = static_cast<char*>(m->wbuf);
  size_t pi = 0;
  auto wptr = [&](size_t i) { return wb + woff[i]; };
  auto gptr = [&](size_t i) { return m->grads + goff[i]; };
  if (m->has_embed) {
    m->emb = reinterpret_cast<bf16*>(wptr(pi));
    m->d_emb = gptr(pi++);
  }
  m->layers.resize(static_cast<size_t>(m->L));
  m->layer_goff.clear();
  for (auto& ly : m->layers) {
    m->layer_goff.push_back(goff[pi]);
    ly.wqkv = reinterpret_cast<bf16*>(wptr(pi));
    ly.d_wqkv = gptr(pi++);
    ly.wo = reinterpret_cast<bf16*>(wptr(pi));
    ly.d_wo = gptr(pi++);
    ly.w1 = reinterpret_cast<bf16*>(wptr(pi));
    ly.d_w1 = gptr(pi++);
    ly.w2 = reinterpret_cast<bf16*>(wptr(pi));
    ly.d_w2 = gptr(pi++);
    ly.g1 = ly.g2 = ly.d_g1 = ly.d_g2 = nullptr;
    if (m->llama) {
      ly.g1 = reinterpret_cast<float*>(wptr(pi));
      ly.d_g1 = gptr(pi++);
      ly.g2 = reinterpret_cast<float*>(wptr(pi));
      ly.d_g2 = gptr(pi++);
    }
  }
  m->layer_goff.push_back(pi < goff.size() ? goff[pi] : gelems);
  if (m->has_head) {
    if (m->llama) {
      m->gf = reinterpret_cast<float*>(wptr(pi));
      m->d_gf = gptr(pi++);
    }
    m->head = reinterpret_cast<bf16*>(wptr(pi));
    m->d_head = gptr(pi++);
  }

  // Reference tensor order (toy_model.hpp:116-126; llama extension).
  auto add = [&](std::string name, int64_t r, int64_t c, void* w, float* g, int64_t ld, bool gain) {
    Slot s;
    s.name = std::move(name);
    s.rows = r;
    s.cols = c;
    s.w = w;
    s.g = g;
    s.ld = ld;
    s.is_gain = gain;
    m->slots.push_back(s);
  };
  if (m->has_embed) add("embedding", m->V, m->d, m->emb, m->d_emb, m->d, false);
  for (int64_t l = 0; l < m->L; ++l) {
    Layer& ly = m->layers[static_cast<size_t>(l)];
    const std::string p = "layer" + std::to_string(m->l_begin + l) + ".";
    if (m->llama) add(p + "attn_norm", 1, m->d, ly.g1, ly.d_g1, m->d, true);
    add(p + "wq", m->d, m->d, ly.wqkv, ly.d_wqkv, m->qkv_w, false);
    add(p + "wk", m->d, m->kvw, ly.wqkv + m->d, ly.d_wqkv + m->d, m->qkv_w, false);
    add(p + "wv", m->d, m->kvw, ly.wqkv + m->d + m->kvw, ly.d_wqkv + m->d + m->kvw, m->qkv_w, false);
    add(p + "wo", m->d, m->d, ly.wo, ly.d_wo, m->d, false);
    if (m->llama) {
      add(p + "ffn_norm", 1, m->d, ly.g2, ly.d_g2, m->d, true);
      add(p + "w_gate", m->d, m->ffn, ly.w1, ly.d_w1, m->gu_w, false);
      add(p + "w_up", m->d, m->ffn, ly.w1 + m->ffn, ly.d_w1 + m->ffn, m->gu_w, false);
      add(p + "w_down", m->ffn, m->d, ly.w2, ly.d_w2, m->d, false);
    } else {
      add(p + "w1", m->d, m->ffn, ly.w1, ly.d_w1, m->gu_w, false);
      add(p + "w2", m->ffn, m->d, ly.w2, ly.d_w2, m->d, false);
    }
  }
  if (m->has_head) {
    if (m->llama) add("final_norm", 1, m->d, m->gf, m->d_gf, m->d, true);
    add("head", m->d, m->V, m->head, m->d_head, Vp, false);
  }

  // init_model (toy_model.hpp:128-132): one SplitMix64 stream in tensor
  // order, regenerated per element on the device (every rank identical).
  // A pipeline stage starts at the draw its first tensor has in the full
  // model, so stage slices hold exactly the full model's values.
  const double scale = 1.0 / std::sqrt(static_cast<double>(m->d));
  const int64_t per_layer = 2 * m->d * m->d + 2 * m->d * m->kvw + m->d * m->gu_w + m->ffn * m->d;
  int64_t draw = m->has_embed ? 0 : m->V * m->d + m->l_begin * per_layer;
  for (Slot& s : m->slots) {
    m->num_params += s.rows * s.cols;
    if (s.is_gain) {
      CK(cfk::fill_f32(static_cast<float*>(s.w), s.cols, 1.0f, ctx->stream));
      continue;
    }
    s.draw_base = draw;
    CK(cfk::init_uniform_bf16(static_cast<bf16*>(s.w), s.ld, s.rows, s.cols, static_cast<uint64_t>(draw), cfg.seed,
                              scale, ctx->stream));
    draw += s.rows * s.cols;
  }
  // storage pieces for the fused AdamW (weights and gradients share the
  // element order piece by piece; RMSNorm gains are fp32 and not decayed)
  for (size_t i = 0; i < pieces.size(); ++i) {
    cfk::AdamPiece ap;
    ap.goff = goff[i];
    ap.n = pieces[i].elems;
    ap.w = wb + woff[i];
    ap.f32 = pieces[i].f32 ? 1 : 0;
    ap.decay = pieces[i].f32 ? 0 : 1;
    m->pieces.push_back(ap);
  }
  if (m->has_head && Vp != m->V)  // zero the head's pad columns
    CK(cudaMemset2DAsync(m->head + m->V, static_cast<size_t>(Vp) * 2, 0, static_cast<size_t>(Vp - m->V) * 2,
                         static_cast<size_t>(m->d), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return m.release();
}

static const Slot& slot_at(Model* m, int64_t idx) {
  if (idx < 0 || idx >= static_cast<int64_t>(m->slots.size())) throw ValidationError("tensor index out of range");
  return m->slots[static_cast<size_t>(idx)];
}

void model_destroy(Model* m) {
  if (!m) return;
  cudaFree(m->wbuf);
  cudaFree(m->grads);
  if (m->opt_mem) cudaFree(m->opt_mem);
  delete m;
}

void model_adamw_init(Model* m) {
  cudaStream_t st = m->ctx->stream;
  if (!m->opt_mem) {
    const int np = static_cast<int>(m->pieces.size());
    std::vector<int64_t> bs(static_cast<size_t>(np) + 1, 0);
    for (int i = 0; i < np; ++i) bs[static_cast<size_t>(i) + 1] = bs[static_cast<size_t>(i)] + cfk::adam_blocks(m->pieces[i].n);
    m->opt_blocks = bs.back();
    const int64_t nb_all = cfk::adam_blocks(m->grad_numel);
    Arena measure{nullptr, 0};
    auto carve = [&](Arena& a) {
      m->master = a.take<float>(m->grad_numel);
      m->adam_m = a.take<float>(m->grad_numel);
      m->adam_v = a.take<float>(m->grad_numel);
      m->opt_scratch = a.take<float>(nb_all + 1);
      m->clip_coef = a.take<float>(1);
      m->grad_norm = a.take<double>(1);
      m->pieces_dev = a.take<cfk::AdamPiece>(np);
      m->block_start_dev = a.take<int64_t>(np + 1);
    };
    carve(measure);
    CK(cudaMalloc(&m->opt_mem, static_cast<size_t>(measure.off + 256)));
    Arena a{static_cast<char*>(m->opt_mem), 0};
    carve(a);
    CK(cudaMemcpyAsync(m->pieces_dev, m->pieces.data(), sizeof(cfk::AdamPiece) * m->pieces.size(),
                       cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(m->block_start_dev, bs.data(), sizeof(int64_t) * bs.size(), cudaMemcpyHostToDevice, st));
  }
  // padding between pieces stays 0 in every buffer
  CK(cudaMemsetAsync(m->master, 0, static_cast<size_t>(m->grad_numel) * 4, st));
  CK(cudaMemsetAsync(m->adam_m, 0, static_cast<size_t>(m->grad_numel) * 4, st));
  CK(cudaMemsetAsync(m->adam_v, 0, static_cast<size_t>(m->grad_numel) * 4, st));
  CK(cfk::master_from_weights(m->pieces_dev, static_cast<int>(m->pieces.size()), m->block_start_dev, m->opt_blocks,
                              m->master, st));
  m->opt_step = 0;
  CK(cudaStreamSynchronize(st));
}

// One AdamW step (torch.optim.AdamW semantics) on the gradients of the last
// run: optional global-norm clipping, then the fused update of master,
// moments and working weights.
void model_adamw_step(Model* m, const cf_adamw_cfg& c, double* grad_norm) {
  if (!m->opt_mem) throw ValidationError("AdamW state not initialised (cf_model_adamw_init)");
  if (!(c.lr >= 0) || !(c.beta1 >= 0 && c.beta1 < 1) || !(c.beta2 >= 0 && c.beta2 < 1) || !(c.eps > 0) ||
      !(c.weight_decay >= 0))
    throw ValidationError("invalid AdamW hyper-parameters");
  cudaStream_t st = m->ctx->stream;
  const bool clip = c.max_grad_norm > 0 || grad_norm;
  if (clip)
    CK(cfk::grad_clip_coef(m->grads, m->grad_numel, static_cast<float>(c.max_grad_norm), m->opt_scratch, m->clip_coef,
                           m->grad_norm, st));
  ++m->opt_step;
  const double t = static_cast<double>(m->opt_step);
  cfk::AdamHyper h;
  h.lr = static_cast<float>(c.lr);
  h.b1 = static_cast<float>(c.beta1);
  h.b2 = static_cast<float>(c.beta2);
  h.eps = static_cast<float>(c.eps);
  h.wd = static_cast<float>(c.weight_decay);
  h.step_size = static_cast<float>(c.lr / (1.0 - std::pow(c.beta1, t)));
  h.sqrt_bc2 = static_cast<float>(std::sqrt(1.0 - std::pow(c.beta2, t)));
  std::vector<cfk::AdamPiece> pcs = m->pieces;
  if (c.decay_gains) {
    for (auto& p : pcs) p.decay = 1;
    CK(cudaMemcpyAsync(m->pieces_dev, pcs.data(), sizeof(cfk::AdamPiece) * pcs.size(), cudaMemcpyHostToDevice, st));
  }
  CK(cfk::adamw_step(m->pieces_dev, static_cast<int>(pcs.size()), m->block_start_dev, m->opt_blocks, m->grads,
                     m->master, m->adam_m, m->adam_v, c.max_grad_norm > 0 ? m->clip_coef : nullptr, h, st));
  if (c.decay_gains)  // restore the default table
    CK(cudaMemcpyAsync(m->pieces_dev, m->pieces.data(), sizeof(cfk::AdamPiece) * m->pieces.size(),
                       cudaMemcpyHostToDevice, st));
  m->ctx->launches += clip ? 3 : 1;
  if (grad_norm) {
    CK(cudaMemcpyAsync(grad_norm, m->grad_norm, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
}

void model_get_master(Model* m, int64_t idx, double* host) {
  if (!m->opt_mem) throw ValidationError("AdamW state not initialised (cf_model_adamw_init)");
  const Slot& s = slot_at(m, idx);
  cudaStream_t st = m->ctx->stream;
  double* tmp = static_cast<double*>(pool_alloc(m->ctx, s.rows * s.cols * 8));
  CK(cfk::f32_to_f64(m->master + (s.g - m->grads), s.ld, s.rows, s.cols, tmp, st));
  CK(cudaMemcpyAsync(host, tmp, static_cast<size_t>(s.rows * s.cols) * 8, cudaMemcpyDeviceToHost, st));
  pool_free(m->ctx, tmp);
  CK(cudaStreamSynchronize(st));
}


void model_get_param(Model* m, int64_t idx, double* host) {
  const Slot& s = slot_at(m, idx);
  cudaStream_t st = m->ctx->stream;
  double* tmp = static_cast<double*>(pool_alloc(m->ctx, s.rows * s.cols * 8));
  if (s.is_gain)
    CK(cfk::f32_to_f64(static_cast<float*>(s.w), s.ld, s.rows, s.cols, tmp, st));
  else
    CK(cfk::bf16_to_f64(static_cast<bf16*>(s.w), s.ld, s.rows, s.cols, tmp, st));
  CK(cudaMemcpyAsync(host, tmp, static_cast<size_t>(s.rows * s.cols) * 8, cudaMemcpyDeviceToHost, st));
  pool_free(m->ctx, tmp);
  CK(cudaStreamSynchronize(st));
}

void model_set_param(Model* m, int64_t idx, const double* host) {
  const Slot& s = slot_at(m, idx);
  cudaStream_t st = m->ctx->stream;
  double* tmp = static_cast<double*>(pool_alloc(m->ctx, s.rows * s.cols * 8));
  CK(cudaMemcpyAsync(tmp, host, static_cast<size_t>(s.rows * s.cols) * 8, cudaMemcpyHostToDevice, st));
  if (s.is_gain)
    CK(cfk::f64_to_f32(tmp, s.rows, s.cols, static_cast<float*>(s.w), s.ld, st));
  else
    CK(cfk::f64_to_bf16(tmp, s.rows, s.cols, static_cast<bf16*>(s.w), s.ld, st));
  // keep the AdamW master copy in step with a caller-set weight (the fp32
  // value the caller gave, not its bf16 rounding)
  if (m->master) CK(cfk::f64_to_f32(tmp, s.rows, s.cols, m->master + (s.g - m->grads), s.ld, st));
  pool_free(m->ctx, tmp);
  CK(cudaStreamSynchronize(st));
}

void model_get_grad(Model* m, int64_t idx, double* host) {
  const Slot& s = slot_at(m, idx);
  cudaStream_t st = m->ctx->stream;
  double* tmp = static_cast<double*>(pool_alloc(m->ctx, s.rows * s.cols * 8));
  CK(cfk::f32_to_f64(s.g, s.ld, s.rows, s.cols, tmp, st));
  CK(cudaMemcpyAsync(host, tmp, static_cast<size_t>(s.rows * s.cols) * 8, cudaMemcpyDeviceToHost, st));
  pool_free(m->ctx, tmp);
  CK(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------- executor
namespace {

// Per-chunk index metadata (built on the host from the plan + token payload;
// uploaded once per step).  Offsets are in int32 units into the meta buffer.
struct ChunkMeta {
  int64_t id = 0, T = 0;
  bool dependent = false;
  int64_t seq = -1, start = 0, seq_len = 0, group = -1, index = -1;
  int64_t o_tok = 0, o_tgt = 0, o_pos = 0, o_segs = 0, nsegs = 0, o_qt = 0, nqt = 0, o_kt = 0, nkt = 0;
  int64_t o_qt128 = 0, nqt128 = 0, o_kt128 = 0, nkt128 = 0;  // 128-row tiles (tcgen05 kernels)
  int64_t o_order = 0, o_uniq = 0, o_uoff = 0, nuniq = 0;
  double pairs = 0;
};

struct GroupState {
  int64_t S = 0;
  bf16* kc = nullptr;   // [L][S][kvw]
  bf16* vc = nullptr;
  float* dkv = nullptr; // [L][S][2kvw]
  void* mem = nullptr;
  std::vector<int64_t> contributions;  // per chunk index
  std::vector<bool> saved;
  // KV offload (cf_run_opts.kv_offload; the paper's deferred "offloading
  // optimization"): the [L][S] state lives in pinned host
  // memory (hk / hv / hdkv) and the device holds two one-layer staging
  // buffers (sk / sv / sdkv [S] rows, by layer parity).  Layer l's rows are
  // loaded on the copy stream while layer l -/+ 1 computes; new K/V rows
  // (forward) and prefix dK/dV rows (backward) are written back after the
  // layer's attention.
  bool offload = false;
  bf16 *hk = nullptr, *hv = nullptr;
  float* hdkv = nullptr;
  void* hmem = nullptr;
  bf16* sk[2] = {nullptr, nullptr};
  bf16* sv[2] = {nullptr, nullptr};
  float* sdkv[2] = {nullptr, nullptr};
  cudaEvent_t used[2] = {nullptr, nullptr};    // compute done with staging b
  cudaEvent_t loaded[2] = {nullptr, nullptr};  // staging b holds the layer it was loaded for
  int64_t staged_layer[2] = {-1, -1};
  bool staged_bwd[2] = {false, false};
  int64_t dkv_valid = 0;                       // host dK/dV rows [0, dkv_valid) hold contributions
  std::vector<bool> on_host;                   // chunk index -> own K/V rows written back
  bf16* K(int64_t l, int64_t kvw) const { return offload ? sk[l & 1] : kc + l * S * kvw; }
  bf16* V(int64_t l, int64_t kvw) const { return offload ? sv[l & 1] : vc + l * S * kvw; }
  float* DKV(int64_t l, int64_t kvw) const { return offload ? sdkv[l & 1] : dkv + l * S * 2 * kvw; }
};

struct Tape {
  void* mem = nullptr;
  int64_t T = 0;
  float* x_in = nullptr;  // (L+1) x T x d
  bf16* qkv = nullptr;    // L x T x qkv_w
  bf16* o = nullptr;      // L x T x d
  float* lse = nullptr;   // L x H x T
  float* x_mid = nullptr; // L x T x d
  bf16* act = nullptr;    // L x T x gu_w
  float* lse_head = nullptr; // T   LM-head log-sum-exp (the backward rebuilds dlogits from it)
  float2* tab = nullptr;  // T x dh/2
  // llama, retained tapes only: the GEMM inputs the backward would
  // otherwise recompute — normed activations and the SwiGLU output
  bf16* xn1 = nullptr;    // L x T x d   rmsnorm(x_in)
  bf16* xn2 = nullptr;    // L x T x d   rmsnorm(x_mid)
  bf16* h = nullptr;      // L x T x ffn swiglu(gate, up)
  bf16* xnf = nullptr;    // T x d       final norm
  int64_t bytes = 0;
  // A discard forward keeps nothing past its own layer, so its transient tape
  // is one layer's working set (x_in a ring of 2, the rest 1 slot) instead of
  // L layers' — what makes in-flight chunks cheap on a pipeline stage.
  bool ring = false;
  int64_t sx = 0, sq = 0, sl = 0, sa = 0;  // per-layer strides of x / qkv / lse / act
  float* xin(int64_t l) const { return x_in + (ring ? (l & 1) : l) * sx; }
  float* xmid(int64_t l) const { return x_mid + (ring ? 0 : l) * sx; }
  bf16* qkvl(int64_t l) const { return qkv + (ring ? 0 : l) * sq; }
  bf16* ol(int64_t l) const { return o + (ring ? 0 : l) * (sx); }
  float* lsel(int64_t l) const { return lse + (ring ? 0 : l) * sl; }
  bf16* actl(int64_t l) const { return act + (ring ? 0 : l) * sa; }
};

}  // namespace
}  // namespace cfb

struct cf_step {
  std::vector<cfb::ChunkMeta> chunks;  // indexed by plan position
  std::map<int64_t, int64_t> pos_of;   // chunk id -> position
  const cfb::Plan* plan = nullptr;
  int32_t* meta_dev = nullptr;
  int32_t* meta_host = nullptr;  // pinned
  int64_t meta_len = 0;
  double normalizer = 0;
  std::string normalizer_error;  // batch_normalizer's ValidationError, if any
  int64_t tokens = 0;
  // algorithmic FLOPs split into one layer's share and the
  // LM head's, so a pipeline stage can report its own slice
  double mf_layer = 0, mf_head = 0, hw_layer = 0, hw_head = 0;
  std::map<int64_t, int64_t> group_len;  // group -> sequence length
  cfb::Plan plan_copy;
  // device time of every op of the last run when the context profiles
  // (cf_step_op_times): kind (CF_PP_*), chunk id, milliseconds
  std::vector<std::array<double, 3>> op_times;
};

namespace cfb {

// Appends one chunk's device metadata (tokens, targets, positions, attention
// segments and tiles, embedding-backward CSR) to `meta` and records the
// offsets in `cm`.  seg_ls: per segment (length, start position in its
// sequence); a dependent chunk's keys are its sequence's rows [0, start+len)
// of the group KV cache.
void append_chunk_meta(ChunkMeta& cm, std::vector<int32_t>& meta, const std::vector<int32_t>& tk_rows,
                       const std::vector<int32_t>& tg, const std::vector<int32_t>& ps,
                       const std::vector<std::pair<int64_t, int64_t>>& seg_ls) {
  auto put = [&](int32_t v) { meta.push_back(v); };
  auto here = [&]() { return static_cast<int64_t>(meta.size()); };
  cm.T = static_cast<int64_t>(tk_rows.size());
  cm.pairs = 0;
  for (const auto& [len, start] : seg_ls) {
    const double L_ = static_cast<double>(len), P_ = static_cast<double>(start);
    cm.pairs += L_ * P_ + L_ * (L_ + 1) / 2;
  }
  cm.o_tok = here();
  std::vector<std::pair<int32_t, int32_t>> tok_rows;
  for (size_t r = 0; r < tk_rows.size(); ++r) {
    put(tk_rows[r]);
    tok_rows.emplace_back(tk_rows[r], static_cast<int32_t>(r));
  }
  cm.o_tgt = here();
  for (int32_t v : tg) put(v);
  cm.o_pos = here();
  for (int32_t v : ps) put(v);
  // attention segments and tiles
  while (meta.size() % 4) put(0);
  cm.o_segs = here();
  std::vector<AttnSeg> segs;
  int32_t qs = 0;
  for (const auto& [len, start] : seg_ls) {
    AttnSeg a;
    a.q_start = qs;
    a.len = static_cast<int32_t>(len);
    a.prefix = static_cast<int32_t>(cm.dependent ? start : 0);
    a.kv_row0 = cm.dependent ? 0 : qs;
    segs.push_back(a);
    qs += a.len;
  }
  for (const AttnSeg& a : segs) {
    put(a.q_start);
    put(a.len);
    put(a.kv_row0);
    put(a.prefix);
  }
  cm.nsegs = static_cast<int64_t>(segs.size());
  cm.o_qt = here();
  for (size_t s = 0; s < segs.size(); ++s)
    for (int32_t f = 0; f < segs[s].len; f += 64) {
      put(static_cast<int32_t>(s));
      put(f);
      put(std::min(64, segs[s].len - f));
      put(0);
      ++cm.nqt;
    }
  cm.o_kt = here();
  for (size_t s = 0; s < segs.size(); ++s) {
    const int32_t nk = segs[s].prefix + segs[s].len;
    for (int32_t f = 0; f < nk; f += 64) {
      put(static_cast<int32_t>(s));
      put(f);
      put(std::min(64, nk - f));
      put(0);
      ++cm.nkt;
    }
  }
  // 128-query tiles, heaviest (most visible keys) first so the causal tail
  // of the grid is short; 128-key tiles likewise by number of queries.
  {
    std::vector<std::array<int32_t, 4>> qt, kt;
    for (size_t s = 0; s < segs.size(); ++s) {
      for (int32_t f = 0; f < segs[s].len; f += 128)
        qt.push_back({static_cast<int32_t>(s), f, std::min(128, segs[s].len - f), segs[s].prefix + f});
      const int32_t nk = segs[s].prefix + segs[s].len;
      for (int32_t f = 0; f < nk; f += 128)
        kt.push_back({static_cast<int32_t>(s), f, std::min(128, nk - f),
                      segs[s].len - std::max(0, f - segs[s].prefix)});
    }
    auto by_work = [](const std::array<int32_t, 4>& x, const std::array<int32_t, 4>& y) { return x[3] > y[3]; };
    std::stable_sort(qt.begin(), qt.end(), by_work);
    std::stable_sort(kt.begin(), kt.end(), by_work);
    cm.o_qt128 = here();
    for (auto& x : qt) {
      put(x[0]);
      put(x[1]);
      put(x[2]);
      put(0);
    }
    cm.nqt128 = static_cast<int64_t>(qt.size());
    cm.o_kt128 = here();
    for (auto& x : kt) {
      put(x[0]);
      put(x[1]);
      put(x[2]);
      put(0);
    }
    cm.nkt128 = static_cast<int64_t>(kt.size());
  }
  // embedding-backward CSR: rows grouped by token id, ascending rows
  std::sort(tok_rows.begin(), tok_rows.end());
  cm.o_order = here();
  for (const auto& tr : tok_rows) put(tr.second);
  std::vector<int32_t> uniq, uoff;
  for (size_t i = 0; i < tok_rows.size(); ++i) {
    if (i == 0 || tok_rows[i].first != tok_rows[i - 1].first) {
      uniq.push_back(tok_rows[i].first);
      uoff.push_back(static_cast<int32_t>(i));
    }
  }
  uoff.push_back(static_cast<int32_t>(tok_rows.size()));
  cm.o_uniq = here();
  for (int32_t v : uniq) put(v);
  cm.o_uoff = here();
  for (int32_t v : uoff) put(v);
  cm.nuniq = static_cast<int64_t>(uniq.size());
  while (meta.size() % 4) put(0);
}

// Builds metadata for every chunk of the plan.
cf_step* step_prepare(Ctx* ctx, Model* m, const Plan& plan, const Batch& b) {
  auto st = std::make_unique<cf_step>();
  st->plan_copy = plan;
  st->plan = &st->plan_copy;
  std::map<int64_t, int64_t> idx_of;
  std::vector<int64_t> tok_off(static_cast<size_t>(b.n) + 1, 0);
  for (int64_t i = 0; i < b.n; ++i) {
    if (!idx_of.emplace(b.ids[i], i).second) throw ValidationError("duplicate sequence id " + std::to_string(b.ids[i]));
    tok_off[i + 1] = tok_off[i] + b.lengths[i];
  }
  // normalizer: global target count (toy_model.hpp:533-541).  The reference
  // only computes (and so only validates) it when no normalizer override is
  // given (plan_runner.hpp:89-91): the error is kept and raised by a run
  // without an override.
  int64_t targets = 0;
  for (int64_t i = 0; i < b.n; ++i) {
    if (b.lengths[i] < 2 && st->normalizer_error.empty())
      st->normalizer_error = "sequence " + std::to_string(b.ids[i]) + " must have length >= 2";
    targets += b.lengths[i] - 1;
  }
  if (targets <= 0 && st->normalizer_error.empty()) st->normalizer_error = "batch has no prediction targets";
  st->normalizer = static_cast<double>(targets);
  if (!b.tokens_host) throw ValidationError("token payload required");
  for (int64_t i = 0; i < tok_off[b.n]; ++i)
    if (b.tokens_host[i] < 0 || b.tokens_host[i] >= m->V)
      throw ValidationError("token id " + std::to_string(b.tokens_host[i]) + " out of vocabulary range");

  const double Nlayer = static_cast<double>(m->d * m->qkv_w + m->d * m->d + m->d * m->gu_w + m->ffn * m->d);
  const double Nhead = static_cast<double>(m->d * m->V);
  const double attn_unit = static_cast<double>(m->H * m->dh);
  std::vector<int32_t> meta;
  for (size_t ci = 0; ci < plan.chunks.size(); ++ci) {
    const Chunk& c = plan.chunks[ci];
    ChunkMeta cm;
    cm.id = c.id;
    cm.dependent = c.kind == kDependent;
    cm.group = c.group;
    cm.index = c.index;
    st->pos_of[c.id] = static_cast<int64_t>(ci);
    // tokens / targets / positions (plan_runner.hpp:112-122)
    std::vector<int32_t> tk_rows, tg, ps;
    std::vector<std::pair<int64_t, int64_t>> seg_ls;
    for (int64_t s = 0; s < c.seg_cnt; ++s) {
      const Segment& sg = plan.segments[static_cast<size_t>(c.seg_off + s)];
      auto it = idx_of.find(sg.seq);
      if (it == idx_of.end()) throw ValidationError("chunk references unknown sequence " + std::to_string(sg.seq));
      const int64_t len = b.lengths[it->second];
      if (sg.start < 0 || sg.len < 1 || sg.start + sg.len > len)
        throw ValidationError("chunk segment exceeds sequence " + std::to_string(sg.seq));
      const int32_t* tk = b.tokens_host + tok_off[it->second];
      for (int64_t t = 0; t < sg.len; ++t) {
        const int64_t p = sg.start + t;
        tk_rows.push_back(tk[p]);
        tg.push_back(p + 1 < len ? tk[p + 1] : -1);
        ps.push_back(static_cast<int32_t>(p));
      }
      if (cm.dependent) {
        cm.seq = sg.seq;
        cm.start = sg.start;
        cm.seq_len = len;
        st->group_len[c.group] = len;
      }
      seg_ls.emplace_back(sg.len, sg.start);
    }
    append_chunk_meta(cm, meta, tk_rows, tg, ps, seg_ls);
    st->tokens += cm.T;
    st->mf_layer += 6.0 * Nlayer * static_cast<double>(cm.T) + 12.0 * attn_unit * cm.pairs;
    st->mf_head += 6.0 * Nhead * static_cast<double>(cm.T);
    st->chunks.push_back(cm);
  }
  // Dependent groups write K/V rows at their sequence's absolute positions of
  // one per-group cache, so the structure the reference's StateStore checks
  // lazily (assemble_prefix, plan_runner.hpp:128-156: "KV prefix does not
  // cover the segment start") is checked here up front for any plan — also
  // one loaded from chunk_plan.json: every member of a group is one segment
  // of the same sequence, members sit at their index_in_group, and member i
  // starts where members 0..i-1 end.
  for (const auto& [gid, members] : plan.groups) {
    int64_t seq = -1, next = 0;
    for (size_t i = 0; i < members.size(); ++i) {
      auto pit = st->pos_of.find(members[i]);
      if (pit == st->pos_of.end()) throw ValidationError("plan references unknown chunk " + std::to_string(members[i]));
      const Chunk& c = plan.chunks[static_cast<size_t>(pit->second)];
      ChunkMeta& cm = st->chunks[static_cast<size_t>(pit->second)];
      if (!cm.dependent || c.group != gid)
        throw ValidationError("chunk " + std::to_string(c.id) + " is listed in group " + std::to_string(gid) +
                              " but is not one of its dependent chunks");
      if (c.seg_cnt != 1)
        throw ValidationError("dependent chunk " + std::to_string(c.id) + " must have exactly one segment");
      if (c.index != static_cast<int64_t>(i))
        throw ValidationError("chunk " + std::to_string(c.id) + " has index_in_group " + std::to_string(c.index) +
                              " but is member " + std::to_string(i) + " of group " + std::to_string(gid));
      if (i == 0) seq = cm.seq;
      if (cm.seq != seq)
        throw ValidationError("group " + std::to_string(gid) + " spans sequences " + std::to_string(seq) + " and " +
                              std::to_string(cm.seq));
      if (cm.start != next)
        throw ValidationError("KV prefix does not cover the segment start of sequence " + std::to_string(cm.seq));
      next = cm.start + cm.T;
    }
  }
  for (const ChunkMeta& cm : st->chunks)
    if (cm.dependent && !plan.groups.count(cm.group))
      throw ValidationError("chunk plan has no group " + std::to_string(cm.group));
  st->hw_layer = st->mf_layer;
  st->hw_head = st->mf_head;
  // every backward recomputes the head GEMM to rebuild dlogits from the LSE
  for (const ChunkMeta& cm : st->chunks) st->hw_head += 2.0 * Nhead * static_cast<double>(cm.T);
  for (const Event& e : plan.events)
    if (e.recompute) {
      const ChunkMeta& cm = st->chunks[static_cast<size_t>(st->pos_of.at(e.chunk))];
      st->hw_layer += 2.0 * Nlayer * static_cast<double>(cm.T) + 4.0 * attn_unit * cm.pairs;
      st->hw_head += 2.0 * Nhead * static_cast<double>(cm.T);
    }
  st->meta_len = static_cast<int64_t>(meta.size());
  CK(cudaMallocHost(&st->meta_host, static_cast<size_t>(st->meta_len + 4) * 4));
  std::memcpy(st->meta_host, meta.data(), meta.size() * 4);
  CK(cudaMalloc(&st->meta_dev, static_cast<size_t>(st->meta_len + 4) * 4));
  CK(cudaMemcpyAsync(st->meta_dev, st->meta_host, static_cast<size_t>(st->meta_len) * 4, cudaMemcpyHostToDevice,
                     ctx->stream));
  return st.release();
}

void step_op_times(const cf_step* st, int64_t* n, int64_t* kinds, int64_t* ids, double* ms) {
  *n = static_cast<int64_t>(st->op_times.size());
  for (size_t i = 0; i < st->op_times.size(); ++i) {
    if (kinds) kinds[i] = static_cast<int64_t>(st->op_times[i][0]);
    if (ids) ids[i] = static_cast<int64_t>(st->op_times[i][1]);
    if (ms) ms[i] = st->op_times[i][2];
  }
}

int64_t step_input_bytes(const cf_step* st) { return st->meta_len * 4; }

void step_destroy(cf_step* st) {
  if (!st) return;
  cudaFree(st->meta_dev);
  cudaFreeHost(st->meta_host);
  delete st;
}

namespace {

struct Exec {
  Ctx* ctx;
  Model* m;
  cf_step* st;
  cudaStream_t s;
  bool corrupt = false;
  float inv_norm = 0;
  double* loss_slots = nullptr;  // device, one per event
  int64_t launches = 0;
  int64_t act_bytes = 0, act_peak = 0, kv_bytes = 0, kv_peak = 0;

  template <class T>
  T* meta(int64_t off) const {
    return reinterpret_cast<T*>(st->meta_dev + off);
  }
  void L(cudaError_t e, const char* what, int n = 1) {
    cuda_check(e, what);
    launches += n;
  }
  // --- optional per-launch timing (cf_ctx_set_profiling)
  struct Rec {
    cudaEvent_t a, b;
    int cls;  // 0 gemm, 1 attention forward, 2 attention backward
    double flops;
    int n;
    bool dep;  // attention of a dependent (split-sequence) chunk
  };
  std::vector<Rec> recs;
  size_t ev_used = 0;
  cudaEvent_t ev() {
    if (ev_used == ctx->event_pool.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ctx->event_pool.push_back(e);
    }
    return ctx->event_pool[ev_used++];
  }
  cudaEvent_t mark(cudaStream_t on = nullptr) {
    if (!ctx->profile) return nullptr;
    cudaEvent_t a = ev();
    CK(cudaEventRecord(a, on ? on : s));
    return a;
  }
  void close(cudaEvent_t a, int cls, double flops, int n, cudaStream_t on = nullptr, bool dep = false) {
    if (!ctx->profile) return;
    cudaEvent_t b = ev();
    CK(cudaEventRecord(b, on ? on : s));
    recs.push_back({a, b, cls, flops, n, dep});
  }
  void gemm(const void* a, int a_k, int64_t lda, const void* b, int b_k, int64_t ldb, void* c, int64_t ldc, int64_t M,
            int64_t N, int64_t K, int epi, const void* r = nullptr, int64_t ldr = 0) {
    cfk::GemmDesc d{a, lda, a_k, b, ldb, b_k, c, ldc, r, ldr, M, N, K, epi};
    cudaEvent_t t0 = mark();
    L(cfk::gemm(d, s), "gemm");
    close(t0, 0, 2.0 * static_cast<double>(M) * static_cast<double>(N) * static_cast<double>(K), 1);
  }

  // Two weight-gradient GEMMs (EPI_F32_ACC) in one CTA-pair launch when the
  // kernel can take both (cfk::gemm2), so their tiles share the last wave.
  void gemm_wgrad2(const cfk::GemmDesc& d0, const cfk::GemmDesc& d1) {
    cudaEvent_t t0 = mark();
    L(cfk::gemm2(d0, d1, s), "gemm2");
    close(t0, 0,
          2.0 * (static_cast<double>(d0.M) * static_cast<double>(d0.N) * static_cast<double>(d0.K) +
                 static_cast<double>(d1.M) * static_cast<double>(d1.N) * static_cast<double>(d1.K)),
          1);
  }

  void gemm_desc(const cfk::GemmDesc& d) {
    cudaEvent_t t0 = mark();
    L(cfk::gemm(d, s), "gemm");
    close(t0, 0, 2.0 * static_cast<double>(d.M) * static_cast<double>(d.N) * static_cast<double>(d.K), 1);
  }

  // LM head + cross-entropy forward (toy_model.hpp:320-331) fused into the
  // head GEMM: the epilogue reduces each row's 256-column slabs to (max, sum
  // exp) partials and picks the target logit, ce_finish() combines them into
  // the LSE (kept in the tape for the backward) and the row losses — the
  // [T, V] logits never reach HBM.
  void head_forward(const bf16* xnf, int64_t T, const int32_t* tgt, float* lse_out, double* loss_slot) {
    const int64_t Vp = align_up(m->V, 8), np = cfk::ce_nparts(m->V);
    float* buf = static_cast<float*>(pool_alloc(ctx, T * np * 8 + 2 * T * 4 + 256));
    float* part = buf;
    float* tlogit = buf + T * np * 2;
    float* row_loss = tlogit + T;
    cfk::GemmDesc g{xnf, m->d, 1, m->head, Vp, 0, nullptr, 0, nullptr, 0, T, m->V, m->d, cfk::EPI_CE_STATS};
    g.ce_tgt = tgt;
    g.ce_part = part;
    g.ce_tlogit = tlogit;
    gemm_desc(g);
    L(cfk::ce_finish(part, np, tlogit, tgt, T, lse_out, row_loss, s), "ce_finish");
    L(cfk::sum_f64(row_loss, T, loss_slot, s), "loss_sum");
    pool_free(ctx, buf);
  }

  // LM head backward (toy_model.hpp:369-388): dlogits are rebuilt from the
  // saved LSE by a recompute of the head GEMM (EPI_CE_GRAD) instead of being
  // kept from the forward, in row blocks of at most ~1 GiB of bf16 dlogits
  // (one block at C2; C5's 152K vocabulary takes a few), each followed by
  // its weight-gradient and input-gradient GEMMs.
  void head_backward(const bf16* xnf, int64_t T, const int32_t* tgt, const float* lse, float* dxf) {
    const int64_t Vp = align_up(m->V, 8), d = m->d;
    const int64_t cap = std::max<int64_t>(256, ((int64_t{1} << 30) / (Vp * 2)) / 256 * 256);
    const int64_t nblk = (T + cap - 1) / cap;
    const int64_t rb = std::min<int64_t>(T, align_up((T + nblk - 1) / nblk, 128));
    bf16* dl = static_cast<bf16*>(pool_alloc(ctx, rb * Vp * 2));
    for (int64_t r0 = 0; r0 < T; r0 += rb) {
      const int64_t n = std::min(rb, T - r0);
      cfk::GemmDesc g{xnf + r0 * d, d, 1, m->head, Vp, 0, dl, Vp, nullptr, 0, n, m->V, d, cfk::EPI_CE_GRAD};
      g.ce_tgt = tgt + r0;
      g.ce_lse = lse + r0;
      g.ce_scale = inv_norm;
      gemm_desc(g);
      gemm(xnf + r0 * d, 0, d, dl, 0, Vp, m->d_head, Vp, d, m->V, n, cfk::EPI_F32_ACC);
      gemm(dl, 1, Vp, m->head, 1, Vp, dxf + r0 * d, d, n, d, m->V, cfk::EPI_F32);
    }
    pool_free(ctx, dl);
  }

  // ---- KV offload: per-layer staging of an offloaded group's state.
  // Loads of layer l into staging buffer l & 1, on the copy stream.
  void kv_load(const ChunkMeta& cm, GroupState* gs, int64_t l, bool bwd) {
    const int b = static_cast<int>(l & 1);
    if (gs->staged_layer[b] == l && gs->staged_bwd[b] == bwd) return;
    cudaStream_t cs = ctx->copy_stream;
    const int64_t kvw = m->kvw, S = gs->S;
    const int64_t rows = bwd ? cm.start + cm.T : cm.start;  // backward: own rows too (incl. their incoming dK/dV)
    CK(cudaStreamWaitEvent(cs, gs->used[b], 0));
    if (rows > 0) {
      CK(cudaMemcpyAsync(gs->sk[b], gs->hk + l * S * kvw, static_cast<size_t>(rows * kvw) * 2, cudaMemcpyHostToDevice, cs));
      CK(cudaMemcpyAsync(gs->sv[b], gs->hv + l * S * kvw, static_cast<size_t>(rows * kvw) * 2, cudaMemcpyHostToDevice, cs));
    }
    if (bwd) {
      const int64_t valid = std::min(rows, gs->dkv_valid);
      if (valid > 0)
        CK(cudaMemcpyAsync(gs->sdkv[b], gs->hdkv + l * S * 2 * kvw, static_cast<size_t>(valid * 2 * kvw) * 4,
                           cudaMemcpyHostToDevice, cs));
      if (rows > valid)
        CK(cudaMemsetAsync(gs->sdkv[b] + valid * 2 * kvw, 0, static_cast<size_t>((rows - valid) * 2 * kvw) * 4, cs));
    }
    CK(cudaEventRecord(gs->loaded[b], cs));
    gs->staged_layer[b] = l;
    gs->staged_bwd[b] = bwd;
  }
  // Before layer l's use: its rows are staged (prefetching the next layer of
  // the pass into the other buffer so the copy overlaps this layer's math).
  void kv_stage(const ChunkMeta& cm, GroupState* gs, int64_t l, bool bwd) {
    kv_load(cm, gs, l, bwd);
    CK(cudaStreamWaitEvent(s, gs->loaded[l & 1], 0));
    const int64_t nxt = bwd ? l - 1 : l + 1;
    if (nxt >= 0 && nxt < m->L) kv_load(cm, gs, nxt, bwd);
  }
  // After layer l's attention: write back what changed, release the buffer.
  void kv_release(const ChunkMeta& cm, GroupState* gs, int64_t l, bool bwd) {
    const int b = static_cast<int>(l & 1);
    cudaStream_t cs = ctx->copy_stream;
    const int64_t kvw = m->kvw, S = gs->S;
    CK(cudaEventRecord(gs->used[b], s));
    CK(cudaStreamWaitEvent(cs, gs->used[b], 0));  // the copy stream now trails this layer's attention
    if (!bwd) {
      if (!gs->on_host[static_cast<size_t>(cm.index)]) {  // a recompute rewrites identical rows: skip
        const size_t off = static_cast<size_t>((l * S + cm.start) * kvw);
        CK(cudaMemcpyAsync(gs->hk + off, gs->sk[b] + cm.start * kvw, static_cast<size_t>(cm.T * kvw) * 2,
                           cudaMemcpyDeviceToHost, cs));
        CK(cudaMemcpyAsync(gs->hv + off, gs->sv[b] + cm.start * kvw, static_cast<size_t>(cm.T * kvw) * 2,
                           cudaMemcpyDeviceToHost, cs));
      }
    } else if (cm.start > 0) {  // prefix dK/dV now include this chunk's contribution; own rows are consumed
      CK(cudaMemcpyAsync(gs->hdkv + l * S * 2 * kvw, gs->sdkv[b], static_cast<size_t>(cm.start * 2 * kvw) * 4,
                         cudaMemcpyDeviceToHost, cs));
    }
    // the staged rows no longer match the host copy for the next pass
    gs->staged_layer[b] = -1;
    CK(cudaEventRecord(gs->used[b], cs));  // reuse only after the write-back
  }

  Tape alloc_tape(int64_t T, bool retain) {
    Tape t;
    t.T = T;
    const int64_t d = m->d;
    t.ring = !retain && m->L > 1;
    const int64_t L_ = t.ring ? 1 : m->L;
    t.sx = T * d;
    t.sq = T * m->qkv_w;
    t.sl = m->H * T;
    t.sa = T * m->gu_w;
    auto carve = [&](Arena& a) {
      t.x_in = a.take<float>((t.ring ? 2 : L_ + 1) * T * d);
      t.qkv = a.take<bf16>(L_ * T * m->qkv_w);
      t.o = a.take<bf16>(L_ * T * d);
      t.lse = a.take<float>(L_ * m->H * T);
      t.x_mid = a.take<float>(L_ * T * d);
      t.act = a.take<bf16>(L_ * T * m->gu_w);
      if (retain && m->has_head) t.lse_head = a.take<float>(T);
      t.tab = a.take<float2>(T * std::max<int64_t>(1, m->dh / 2));
      if (retain && m->llama) {
        t.xn1 = a.take<bf16>(L_ * T * d);
        t.xn2 = a.take<bf16>(L_ * T * d);
        t.h = a.take<bf16>(L_ * T * m->ffn);
        if (m->has_head) t.xnf = a.take<bf16>(T * d);
      }
    };
    Arena measure{nullptr, 0};
    carve(measure);
    const int64_t bytes = measure.off + 256;
    t.mem = pool_alloc(ctx, bytes);
    t.bytes = bytes;
    Arena a{static_cast<char*>(t.mem), 0};
    carve(a);
    act_bytes += bytes;
    act_peak = std::max(act_peak, act_bytes);
    return t;
  }
  void free_tape(Tape& t) {
    pool_free(ctx, t.mem);
    act_bytes -= t.bytes;
    t.mem = nullptr;
  }

  AttnParams attn_params(const ChunkMeta& cm, const Tape& t, int64_t l, GroupState* gs) {
    AttnParams p{};
    const int64_t T = cm.T;
    p.q = t.qkvl(l);
    p.q_stride = m->qkv_w;
    if (cm.dependent) {
      p.k = gs->K(l, m->kvw);
      p.v = gs->V(l, m->kvw);
      p.kv_stride = m->kvw;
      p.dk_acc = gs->DKV(l, m->kvw);
      p.dv_acc = p.dk_acc + m->kvw;
    } else {
      p.k = p.q + m->d;
      p.v = p.q + m->d + m->kvw;
      p.kv_stride = m->qkv_w;
    }
    p.acc_stride = 2 * m->kvw;
    p.o = t.ol(l);
    p.o_stride = m->d;
    p.lse = t.lsel(l);
    p.segs = meta<const AttnSeg>(cm.o_segs);
    p.tiles = meta<const AttnTile>(cm.o_qt);
    p.num_tiles = static_cast<int32_t>(cm.nqt);
    p.T = static_cast<int32_t>(T);
    p.H = static_cast<int32_t>(m->H);
    p.KVH = static_cast<int32_t>(m->KVH);
    p.dh = static_cast<int32_t>(m->dh);
    p.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(m->dh)));
    return p;
  }

  // Forward of one chunk (segment_forward per segment, toy_model.hpp:206-334).
  // A pipeline stage without the embedding finds its input already in
  // t.x_in[0]; one without the head leaves its output in t.x_in[L].
  void forward(const ChunkMeta& cm, Tape& t, GroupState* gs, int64_t slot, bool retain) {
    const int64_t T = cm.T, d = m->d;
    const int32_t* tok = meta<const int32_t>(cm.o_tok);
    const int32_t* tgt = meta<const int32_t>(cm.o_tgt);
    bf16* A = static_cast<bf16*>(pool_alloc(ctx, T * std::max(d, m->ffn) * 2));
    bf16* hscr = nullptr;  // SwiGLU output of a discard forward (fused epilogue)
    if (m->has_embed) L(cfk::embed_fwd(tok, m->emb, d, T, t.xin(0), s), "embed");
    if (m->llama)
      L(cfk::rope_table(meta<const int32_t>(cm.o_pos), T, static_cast<int>(m->dh), m->cfg.rope_theta, t.tab, s),
        "rope_table");
    for (int64_t l = 0; l < m->L; ++l) {
      const Layer& ly = m->layers[static_cast<size_t>(l)];
      float* x = t.xin(l);
      float* xm = t.xmid(l);
      bf16* qkv = t.qkvl(l);
      bf16* act = t.actl(l);
      bf16* xn1 = t.xn1 ? t.xn1 + l * T * d : A;
      if (m->llama)
        L(cfk::rmsnorm_fwd(x, ly.g1, T, d, static_cast<float>(m->cfg.rms_eps), xn1, s), "rmsnorm");
      else
        L(cfk::to_bf16(x, xn1, T * d, s), "to_bf16");
      if (cm.dependent && gs->offload) kv_stage(cm, gs, l, false);
      bf16* kc_rows = cm.dependent ? gs->K(l, m->kvw) + cm.start * m->kvw : nullptr;
      bf16* vc_rows = cm.dependent ? gs->V(l, m->kvw) + cm.start * m->kvw : nullptr;
      if (m->llama && cfk::gemm_rope_ok(T, m->qkv_w, d, m->dh, d, d + m->kvw)) {
        // RoPE and the KV-cache copy in the q|k|v GEMM's epilogue
        cfk::GemmDesc g{xn1, d, 1, ly.wqkv, m->qkv_w, 0, qkv, m->qkv_w, t.tab, m->dh / 2, T, m->qkv_w, d,
                        cfk::EPI_BF16_ROPE};
        g.col_k = d;
        g.col_v = d + m->kvw;
        g.kc = kc_rows;
        g.vc = vc_rows;
        g.cache_ld = m->kvw;
        cudaEvent_t g0 = mark();
        L(cfk::gemm(g, s), "gemm_rope");
        close(g0, 0, 2.0 * static_cast<double>(T) * static_cast<double>(m->qkv_w) * static_cast<double>(d), 1);
      } else {
        gemm(xn1, 1, d, ly.wqkv, 0, m->qkv_w, qkv, m->qkv_w, T, m->qkv_w, d, cfk::EPI_BF16);
        if (m->llama)
          L(cfk::rope_qk(qkv, m->qkv_w, T, static_cast<int>(m->H), static_cast<int>(m->KVH),
                         static_cast<int>(m->dh), d, t.tab, s),
            "rope");
        if (cm.dependent)
          L(cfk::kv_store(qkv, m->qkv_w, T, m->kvw, d, d + m->kvw, kc_rows, vc_rows, m->kvw, s), "kv_store");
      }
      AttnParams p = attn_params(cm, t, l, gs);
      cudaEvent_t t0 = mark();
      if (cfk::attn_fwd_pp_supported(p))
        L(cfk::attn_forward_tc_pp(p, meta<const AttnTile>(cm.o_qt128), static_cast<int32_t>(cm.nqt128),
                                  cm.dependent ? gs->S : T, s),
          "attn_fwd_tc_pp");
      else if (cfk::attn_tc_supported(p))
        L(cfk::attn_forward_tc(p, meta<const AttnTile>(cm.o_qt128), static_cast<int32_t>(cm.nqt128),
                               cm.dependent ? gs->S : T, s),
          "attn_fwd_tc");
      else
        L(cfk::attn_forward(p, s), "attn_fwd");
      close(t0, 1, 4.0 * static_cast<double>(m->H * m->dh) * cm.pairs, 1, nullptr, cm.dependent);
      if (cm.dependent && gs->offload) kv_release(cm, gs, l, false);
      gemm(t.ol(l), 1, d, ly.wo, 0, d, xm, d, T, d, d, cfk::EPI_F32_RES, x, d);
      float* xn = t.xin(l + 1);
      if (m->llama) {
        bf16* xn2 = t.xn2 ? t.xn2 + l * T * d : A;
        L(cfk::rmsnorm_fwd(xm, ly.g2, T, d, static_cast<float>(m->cfg.rms_eps), xn2, s), "rmsnorm");
        bf16* hl = t.h ? t.h + l * T * m->ffn : A;
        if (cfk::gemm_swiglu_ok(T, m->gu_w, d)) {  // h written by the gate|up GEMM's epilogue
          // the epilogue writes h while later tiles still load xn2: on a
          // discard forward both would live in A, so h gets its own scratch
          if (!t.h) {
            if (!hscr) hscr = static_cast<bf16*>(pool_alloc(ctx, T * m->ffn * 2));
            hl = hscr;
          }
          gemm(xn2, 1, d, ly.w1, 0, m->gu_w, act, m->gu_w, T, m->gu_w, d, cfk::EPI_BF16_SWIGLU, hl, m->ffn);
        } else {
          gemm(xn2, 1, d, ly.w1, 0, m->gu_w, act, m->gu_w, T, m->gu_w, d, cfk::EPI_BF16);
          L(cfk::swiglu_fwd(act, T, m->ffn, hl, s), "swiglu");
        }
        gemm(hl, 1, m->ffn, ly.w2, 0, d, xn, d, T, d, m->ffn, cfk::EPI_F32_RES, xm, d);
      } else {
        L(cfk::to_bf16(xm, A, T * d, s), "to_bf16");
        gemm(A, 1, d, ly.w1, 0, m->gu_w, act, m->gu_w, T, m->ffn, d, cfk::EPI_BF16_TANH);
        gemm(act, 1, m->ffn, ly.w2, 0, d, xn, d, T, d, m->ffn, cfk::EPI_F32_RES, xm, d);
      }
    }
    if (m->has_head) {
      const float* xL = t.xin(m->L);
      bf16* xnf = t.xnf ? t.xnf : A;
      if (m->llama)
        L(cfk::rmsnorm_fwd(xL, m->gf, T, d, static_cast<float>(m->cfg.rms_eps), xnf, s), "rmsnorm");
      else
        L(cfk::to_bf16(xL, xnf, T * d, s), "to_bf16");
      head_forward(xnf, T, tgt, retain ? t.lse_head : nullptr, loss_slots + slot);
    }
    if (hscr) pool_free(ctx, hscr);
    pool_free(ctx, A);
  }

  // Backward of one chunk (segment_backward, toy_model.hpp:341-520).  A
  // pipeline stage without the head passes the gradient of its output in
  // dx_io; a stage without the embedding gets its input gradient back there.
  // Called (when set) as each gradient range becomes final in this
  // backward: -1 final norm + head, l for layer l, -2 the embedding.
  std::function<void(int64_t)> on_grads_final;
  void backward(const ChunkMeta& cm, Tape& t, GroupState* gs, float* dx_io = nullptr) {
    const int64_t T = cm.T, d = m->d, qw = m->qkv_w, kvw = m->kvw;
    const float eps = static_cast<float>(m->cfg.rms_eps);
    float *dx, *dmid, *da, *dsum, *rstd, *dkv_local = nullptr;
    bf16 *A, *xb, *dh, *dgu, *dqkv;
    auto carve = [&](Arena& a) {
      dx = dx_io ? dx_io : a.take<float>(T * d);
      dmid = a.take<float>(T * d);
      da = a.take<float>(T * d);
      A = a.take<bf16>(T * std::max(d, m->ffn));  // bf16 activations (recomputed)
      xb = a.take<bf16>(T * d);                    // bf16 of a gradient
      dh = a.take<bf16>(T * m->ffn);
      dgu = a.take<bf16>(T * m->gu_w);
      dqkv = a.take<bf16>(T * qw);
      dsum = a.take<float>(m->H * T);
      rstd = a.take<float>(T);
      if (!cm.dependent) dkv_local = a.take<float>(T * 2 * kvw);
    };
    Arena measure{nullptr, 0};
    carve(measure);
    Arena a{static_cast<char*>(pool_alloc(ctx, measure.off + 256)), 0};
    carve(a);
    void* scratch = a.base;

    // Output head + CE (toy_model.hpp:369-388): dHead += xf^T dlogits, dxf = dlogits head^T.
    // RMSNorm backward; the fused kernel also leaves bf16(out) in xb (the
    // next dgrad/wgrad GEMM input) and accumulates the gain gradient
    const bool fused = m->llama && cfk::rmsnorm_bwd_fused_ok(d);
    auto norm_bwd = [&](const float* xin, const float* gain, const float* dres, float* out, float* dgain) {
      if (fused) {
        L(cfk::rmsnorm_bwd_fused(xin, gain, da, dres, T, d, eps, out, xb, dgain, s), "rmsnorm_bwd_fused", 2);
      } else {
        L(cfk::rmsnorm_bwd(xin, gain, da, dres, T, d, eps, out, rstd, s), "rmsnorm_bwd");
        L(cfk::gain_grad(xin, da, rstd, T, d, dgain, s), "gain_grad", 2);
      }
    };
    if (m->has_head) {
      const float* xL = t.xin(m->L);
      const bf16* xnf = t.xnf;
      if (!xnf) {
        if (m->llama)
          L(cfk::rmsnorm_fwd(xL, m->gf, T, d, eps, A, s), "rmsnorm");
        else
          L(cfk::to_bf16(xL, A, T * d, s), "to_bf16");
        xnf = A;
      }
      const int32_t* tgt = meta<const int32_t>(cm.o_tgt);
      if (m->llama) {
        head_backward(xnf, T, tgt, t.lse_head, da);
        norm_bwd(xL, m->gf, nullptr, dx, m->d_gf);
      } else {
        head_backward(xnf, T, tgt, t.lse_head, dx);
      }
    }
    if (on_grads_final) on_grads_final(-1);

    for (int64_t l = m->L - 1; l >= 0; --l) {
      const Layer& ly = m->layers[static_cast<size_t>(l)];
      const float* x = t.xin(l);
      const float* xm = t.xmid(l);
      const bf16* act = t.actl(l);
      const bf16* O = t.ol(l);
      // FFN (toy_model.hpp:409-425)
      // bf16(dx) is left in xb by the previous norm_bwd, except when dx came
      // from the next pipeline stage
      if (!fused || (l == m->L - 1 && !m->has_head)) L(cfk::to_bf16(dx, xb, T * d, s), "to_bf16");
      if (m->llama) {
        gemm(xb, 1, d, ly.w2, 1, d, dh, m->ffn, T, m->ffn, d, cfk::EPI_BF16);
        const bf16* hl = t.h ? t.h + l * T * m->ffn : A;
        if (!t.h) L(cfk::swiglu_fwd(act, T, m->ffn, A, s), "swiglu");  // recompute h
        // down and gate|up weight gradients in one launch when h and xn2 are
        // tape-resident (xb, their shared dY operand, lives until norm_bwd)
        const cfk::GemmDesc dw2{hl, m->ffn, 0, xb, d, 0, ly.d_w2, d, nullptr, 0, m->ffn, d, T, cfk::EPI_F32_ACC};
        const bool group_ffn = t.h && t.xn2;
        if (!group_ffn) gemm_desc(dw2);
        L(cfk::swiglu_bwd(act, dh, T, m->ffn, dgu, s), "swiglu_bwd");
        const bf16* xn2 = t.xn2 ? t.xn2 + l * T * d : A;
        if (!t.xn2) L(cfk::rmsnorm_fwd(xm, ly.g2, T, d, eps, A, s), "rmsnorm");  // recompute xn2
        const cfk::GemmDesc dw1{xn2, d, 0, dgu, m->gu_w, 0, ly.d_w1, m->gu_w, nullptr, 0, d, m->gu_w, T,
                                cfk::EPI_F32_ACC};
        if (group_ffn)
          gemm_wgrad2(dw2, dw1);
        else
          gemm_desc(dw1);
        gemm(dgu, 1, m->gu_w, ly.w1, 1, m->gu_w, da, d, T, d, m->gu_w, cfk::EPI_F32);
        norm_bwd(xm, ly.g2, dx, dmid, ly.d_g2);
      } else {
        gemm(xb, 1, d, ly.w2, 1, d, dgu, m->ffn, T, m->ffn, d, cfk::EPI_BF16_TANHGRAD, act, m->ffn);
        gemm(act, 0, m->ffn, xb, 0, d, ly.d_w2, d, m->ffn, d, T, cfk::EPI_F32_ACC);
        gemm(dgu, 1, m->ffn, ly.w1, 1, m->ffn, dmid, d, T, d, m->ffn, cfk::EPI_F32_RES, dx, d);
        L(cfk::to_bf16(xm, A, T * d, s), "to_bf16");
        gemm(A, 0, d, dgu, 0, m->ffn, ly.d_w1, m->gu_w, d, m->ffn, T, cfk::EPI_F32_ACC);
      }
      // Attention output projection (toy_model.hpp:427-434)
      if (!fused) L(cfk::to_bf16(dmid, xb, T * d, s), "to_bf16");
      bf16* dO = A;  // reuse
      gemm(xb, 1, d, ly.wo, 1, d, dO, d, T, d, d, cfk::EPI_BF16);
      // the o weight gradient joins the q|k|v one below (same launch): O is
      // tape-resident and xb is not rewritten before norm_bwd
      const cfk::GemmDesc dwo{O, d, 0, xb, d, 0, ly.d_wo, d, nullptr, 0, d, d, T, cfk::EPI_F32_ACC};
      // Attention (toy_model.hpp:436-495)
      if (cm.dependent && gs->offload) kv_stage(cm, gs, l, true);
      AttnParams p = attn_params(cm, t, l, gs);
      p.dout = dO;
      p.dout_stride = d;
      p.dsum = dsum;
      p.dq = dqkv;
      p.dq_stride = qw;
      const float* own_dk = nullptr;
      const bool tc = cfk::attn_tc_supported(p);
      // tcgen05 path: RoPE backward of dQ in the dQ kernel; a standalone
      // chunk's dK (rotated back) / dV go straight to dqkv in bf16
      if (tc && m->llama) p.rope_tab = t.tab;
      const bool direct = tc && !cm.dependent;
      if (cm.dependent) {
        float* own = p.dk_acc + cm.start * 2 * kvw;
        if (corrupt) L(cfk::scale_rows_f32(own, T, 2 * kvw, 2 * kvw, 1.0000001f, s), "corrupt");
        own_dk = own;
      } else if (direct) {
        p.dkv_out = dqkv;
        p.dkv_out_ld = qw;
        p.col_k = d;
        p.col_v = d + kvw;
      } else {
        CK(cudaMemsetAsync(dkv_local, 0, static_cast<size_t>(T * 2 * kvw) * 4, s));
        p.dk_acc = dkv_local;
        p.dv_acc = dkv_local + kvw;
        own_dk = dkv_local;
      }
      cudaEvent_t t0 = mark();
      p.keys_per_query = T > 0 ? static_cast<double>(cm.pairs) / static_cast<double>(T) : 0.0;
      if (tc)
        L(cfk::attn_backward_tc(p, meta<const AttnTile>(cm.o_qt128), static_cast<int32_t>(cm.nqt128),
                                meta<const AttnTile>(cm.o_kt128), static_cast<int32_t>(cm.nkt128),
                                cm.dependent ? gs->S : T, s),
          "attn_bwd_tc", 3);
      else
        L(cfk::attn_backward(p, meta<const AttnTile>(cm.o_kt), static_cast<int32_t>(cm.nkt), s), "attn_bwd", 3);
      close(t0, 2, 8.0 * static_cast<double>(m->H * m->dh) * cm.pairs, 3, nullptr, cm.dependent);
      if (!direct)
        L(cfk::dkv_to_dqkv(own_dk, own_dk + kvw, 2 * kvw, T, static_cast<int>(m->KVH), static_cast<int>(m->dh),
                           m->llama ? t.tab : nullptr, dqkv, qw, d, d + kvw, s),
          "dkv_to_dqkv");
      if (cm.dependent && gs->offload) kv_release(cm, gs, l, true);
      if (m->llama && !p.rope_tab)
        L(cfk::rope_bwd_q(dqkv, qw, T, static_cast<int>(m->H), static_cast<int>(m->dh), t.tab, s), "rope_bwd");
      // Projections (toy_model.hpp:497-511)
      const bf16* xn1 = t.xn1 ? t.xn1 + l * T * d : A;
      if (!t.xn1) {
        if (m->llama)
          L(cfk::rmsnorm_fwd(x, ly.g1, T, d, eps, A, s), "rmsnorm");  // recompute xn
        else
          L(cfk::to_bf16(x, A, T * d, s), "to_bf16");
      }
      gemm_wgrad2(dwo, cfk::GemmDesc{xn1, d, 0, dqkv, qw, 0, ly.d_wqkv, qw, nullptr, 0, d, qw, T, cfk::EPI_F32_ACC});
      if (m->llama) {
        gemm(dqkv, 1, qw, ly.wqkv, 1, qw, da, d, T, d, qw, cfk::EPI_F32);
        norm_bwd(x, ly.g1, dmid, dx, ly.d_g1);
      } else {
        gemm(dqkv, 1, qw, ly.wqkv, 1, qw, dx, d, T, d, qw, cfk::EPI_F32_RES, dmid, d);
      }
      if (on_grads_final) on_grads_final(l);
    }
    // Embedding (toy_model.hpp:514-519), deterministic per-token sums.
    if (m->has_embed)
      L(cfk::embed_bwd(dx, d, meta<const int32_t>(cm.o_order), meta<const int32_t>(cm.o_uniq),
                       meta<const int32_t>(cm.o_uoff), cm.nuniq, m->d_emb, s),
        "embed_bwd");
    if (on_grads_final) on_grads_final(-2);
    pool_free(ctx, scratch);
  }
};

}  // namespace

namespace {

// Per-stage state of one training step (the B200 counterpart of run_plan's
// locals, plan_runner.hpp:84-110): retained tapes, per-group KV state, stage
// inputs kept for just-in-time recompute, loss slots and the run_plan
// instrumentation counters.  With one stage it runs plan.events directly;
// pipeline stages feed it their op streams (host/pp.hpp).
struct StageRunner {
  Exec ex;
  Ctx* ctx;
  Model* m;
  cf_step* st;
  double norm = 0;
  int64_t nslots = 0;
  std::map<int64_t, Tape> live;
  std::map<int64_t, GroupState> groups;
  std::map<int64_t, float*> kept_in;  // discarded chunk -> stage input, until its F'
  std::map<int64_t, int64_t> first_slot;
  std::vector<std::pair<int64_t, int64_t>> recompute_pairs;  // (slot, first slot)
  std::vector<int64_t> first_pass_slots;
  int64_t held = 0, peak = 0, violations = 0, recomputes = 0;
  // stage-input checkpointing (cf_run_opts.stage_tape_budget): a first-pass
  // retain-forward beyond `tape_budget` resident tapes keeps only its stage
  // input and is recomputed right before its backward
  int64_t tape_budget = 0, live_peak = 0, ckpt_recomputes = 0, next_extra_slot = 0;
  std::set<int64_t> ckpt;
  bool kv_offload = false;  // dependent groups keep their KV state in pinned host memory
  int64_t io_bytes = 0;  // stage-boundary buffers held (kept inputs)
  struct OpMark {
    int64_t kind, id;
    cudaEvent_t a, b;
  };
  std::vector<OpMark> marks;  // per-op device time when profiling
  cudaEvent_t op_begin() { return ctx->profile ? ex.mark() : nullptr; }
  void op_end(cudaEvent_t a, int64_t kind, int64_t id) {
    if (!ctx->profile) return;
    cudaEvent_t b = ex.ev();
    CK(cudaEventRecord(b, ex.s));
    marks.push_back({kind, id, a, b});
  }

  StageRunner(Ctx* c, Model* mm, cf_step* s, const cf_run_opts& opts, int64_t slots)
      : ctx(c), m(mm), st(s), nslots(slots + static_cast<int64_t>(s->chunks.size())) {
    // loss slots: one per op of the stream, then one per chunk for the
    // checkpoint recomputes the tape budget may add
    next_extra_slot = slots;
    tape_budget = opts.stage_tape_budget;
    if (tape_budget < 0) throw ValidationError("stage_tape_budget must be non-negative");
    const Plan& plan = *st->plan;
    if (!plan.violations.empty()) throw ValidationError("execution plan is invalid: " + plan.violations.front());
    ex.ctx = ctx;
    ex.m = m;
    ex.st = st;
    ex.s = ctx->stream;
    ex.corrupt = opts.corrupt_kv_grads != 0;
    kv_offload = opts.kv_offload != 0;
    if (!(opts.normalizer_override > 0) && !st->normalizer_error.empty())
      throw ValidationError(st->normalizer_error);
    norm = opts.normalizer_override > 0 ? opts.normalizer_override : st->normalizer;
    ex.inv_norm = static_cast<float>(1.0 / norm);
    ex.loss_slots = static_cast<double*>(pool_alloc(ctx, (nslots + 1) * 8));
    CK(cudaMemsetAsync(ex.loss_slots, 0, static_cast<size_t>(nslots + 1) * 8, ex.s));
    if (!opts.accumulate_grads) CK(cudaMemsetAsync(m->grads, 0, static_cast<size_t>(m->grad_numel) * 4, ex.s));
  }

  // A step that throws part-way (bad plan, CUDA error) still returns its
  // pool memory; finish() leaves nothing behind for this to release.
  ~StageRunner() {
    for (auto& kv : live) cudaFreeAsync(kv.second.mem, ex.s);
    for (auto& kv : groups) {
      if (kv.second.offload) {
        if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
        host_release(ctx, kv.second.hmem);
        for (int b = 0; b < 2; ++b) {
          cudaEventDestroy(kv.second.used[b]);
          cudaEventDestroy(kv.second.loaded[b]);
        }
      }
      if (kv.second.mem) cudaFreeAsync(kv.second.mem, ex.s);
    }
    for (auto& kv : kept_in) cudaFreeAsync(kv.second, ex.s);
    if (ex.loss_slots) cudaFreeAsync(ex.loss_slots, ex.s);
  }
  StageRunner(const StageRunner&) = delete;
  StageRunner& operator=(const StageRunner&) = delete;

  const ChunkMeta& chunk(int64_t id) const {
    auto it = st->pos_of.find(id);
    if (it == st->pos_of.end()) throw ValidationError("plan references unknown chunk " + std::to_string(id));
    return st->chunks[static_cast<size_t>(it->second)];
  }
  int64_t group_size(const ChunkMeta& cm) const {
    return static_cast<int64_t>(st->plan->groups.at(cm.group).size());
  }
  int64_t kv_state_bytes(int64_t S) const {
    return 3 * 256 + 2 * m->L * S * m->kvw * 2 + m->L * S * 2 * m->kvw * 4;
  }
  // offloaded group: two one-layer device staging buffers
  int64_t staging_bytes(int64_t S) const { return 6 * 256 + 2 * (2 * S * m->kvw * 2 + S * 2 * m->kvw * 4); }

  // KV offload: host state in pinned memory (from the context's cache of
  // pinned blocks), device staging for two layers, copy-stream events.
  void alloc_offloaded(GroupState& g) {
    const int64_t S = g.S, kvw = m->kvw, L_ = m->L;
    g.offload = true;
    const size_t hbytes = static_cast<size_t>(L_ * S * kvw) * (2 + 2 + 8) + 3 * 256;
    g.hmem = host_acquire(ctx, hbytes);
    Arena h{static_cast<char*>(g.hmem), 0};
    g.hk = h.take<bf16>(L_ * S * kvw);
    g.hv = h.take<bf16>(L_ * S * kvw);
    g.hdkv = h.take<float>(L_ * S * 2 * kvw);
    const int64_t bytes = staging_bytes(S);
    g.mem = pool_alloc(ctx, bytes);
    Arena a{static_cast<char*>(g.mem), 0};
    for (int b = 0; b < 2; ++b) {
      g.sk[b] = a.take<bf16>(S * kvw);
      g.sv[b] = a.take<bf16>(S * kvw);
      g.sdkv[b] = a.take<float>(S * 2 * kvw);
      g.used[b] = new_timing_free_event();
      g.loaded[b] = new_timing_free_event();
      CK(cudaEventRecord(g.used[b], ex.s));
    }
    // staged rows past the ones a layer loads are read (masked) by partial
    // 128-key tiles: they must be finite
    CK(cudaMemsetAsync(g.mem, 0, static_cast<size_t>(bytes), ex.s));
    CK(cudaEventRecord(g.used[0], ex.s));
    CK(cudaEventRecord(g.used[1], ex.s));
    if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    ex.kv_bytes += bytes;
    ex.kv_peak = std::max(ex.kv_peak, ex.kv_bytes);
  }
  void free_group(GroupState& g) {
    if (g.offload) {
      // the copy stream's last write-backs must finish before the buffers go
      CK(cudaEventRecord(g.used[0], ctx->copy_stream));
      CK(cudaStreamWaitEvent(ex.s, g.used[0], 0));
      CK(cudaStreamSynchronize(ctx->copy_stream));
      host_release(ctx, g.hmem);
      for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(g.used[b]);
        cudaEventDestroy(g.loaded[b]);
      }
      ex.kv_bytes -= staging_bytes(g.S);
    } else {
      ex.kv_bytes -= kv_state_bytes(g.S);
    }
    pool_free(ctx, g.mem);
    g.mem = nullptr;
  }

  GroupState* group_for(const ChunkMeta& cm) {
    if (!cm.dependent) return nullptr;
    auto git = groups.find(cm.group);
    if (git == groups.end()) {
      GroupState g;
      g.S = cm.seq_len;
      const int64_t n = group_size(cm);
      g.contributions.assign(static_cast<size_t>(n), 0);
      g.saved.assign(static_cast<size_t>(n), false);
      g.on_host.assign(static_cast<size_t>(n), false);
      if (kv_offload) {
        alloc_offloaded(g);
        git = groups.emplace(cm.group, std::move(g)).first;
        return &git->second;
      }
      const int64_t bytes = kv_state_bytes(g.S);
      g.mem = pool_alloc(ctx, bytes);
      Arena a{static_cast<char*>(g.mem), 0};
      g.kc = a.take<bf16>(m->L * g.S * m->kvw);
      g.vc = a.take<bf16>(m->L * g.S * m->kvw);
      g.dkv = a.take<float>(m->L * g.S * 2 * m->kvw);
      CK(cudaMemsetAsync(g.dkv, 0, static_cast<size_t>(m->L * g.S * 2 * m->kvw) * 4, ex.s));
      // K/V rows of later chunks are read (masked, P = 0) by the 128-key tiles
      // of earlier chunks whose length is not a multiple of 128: they must be
      // finite, since 0 * NaN garbage would poison O and dQ
      CK(cudaMemsetAsync(g.kc, 0, static_cast<size_t>(m->L * g.S * m->kvw) * 2, ex.s));
      CK(cudaMemsetAsync(g.vc, 0, static_cast<size_t>(m->L * g.S * m->kvw) * 2, ex.s));
      ex.kv_bytes += bytes;
      ex.kv_peak = std::max(ex.kv_peak, ex.kv_bytes);
      git = groups.emplace(cm.group, std::move(g)).first;
    }
    return &git->second;
  }

  // Forward of chunk `id` into loss slot `slot`.  `in` is the stage input
  // ([T, d] fp32, pool memory owned by the runner from here on) on stages
  // without the embedding; a recompute forward uses the input kept by the
  // chunk's first pass (keep_in).  Returns the stage output for the next
  // stage (caller-owned pool memory) or null on the last stage / for F'.
  float* forward(int64_t id, bool retain, bool recompute, bool save_kv, int64_t slot, float* in, bool keep_in,
                 bool ckpt_recompute = false) {
    cudaEvent_t t0 = op_begin();
    const ChunkMeta& cm = chunk(id);
    GroupState* gs = group_for(cm);
    const size_t act = static_cast<size_t>(cm.T * m->d) * 4;
    // over the tape budget: run this first-pass retain-forward as a discard
    // forward that keeps its stage input (plan semantics unchanged: the chunk
    // still counts as retained for the reference instrumentation).  One slot
    // of the budget stays free for the just-in-time tape of the backward in
    // progress (a checkpoint restore or a K-plan F'), so resident tapes never
    // exceed the budget.
    bool checkpoint = false;
    if (retain && !recompute && tape_budget > 0 && static_cast<int64_t>(live.size()) + 1 >= tape_budget) {
      checkpoint = true;
      retain = false;
      keep_in = true;
      ckpt.insert(id);
    }
    Tape t = ex.alloc_tape(cm.T, retain);
    if (!m->has_embed) {
      float* src = in;
      if (recompute) {
        auto k = kept_in.find(id);
        if (k == kept_in.end()) throw ValidationError("recompute of chunk " + std::to_string(id) + " without its stage input");
        src = k->second;
      }
      if (!src) throw ValidationError("stage input missing for chunk " + std::to_string(id));
      CK(cudaMemcpyAsync(t.xin(0), src, act, cudaMemcpyDeviceToDevice, ex.s));
    }
    ex.forward(cm, t, gs, slot, retain);
    if (gs && save_kv) gs->saved[static_cast<size_t>(cm.index)] = true;
    if (gs) gs->on_host[static_cast<size_t>(cm.index)] = true;
    if (!recompute) {
      first_slot[id] = slot;
      first_pass_slots.push_back(slot);
    } else {
      if (ckpt_recompute)
        ++ckpt_recomputes;
      else
        ++recomputes;
      auto f = first_slot.find(id);
      recompute_pairs.emplace_back(slot, f == first_slot.end() ? -1 : f->second);
    }
    float* out = nullptr;
    if (!m->has_head && !recompute) {
      out = static_cast<float*>(pool_alloc(ctx, static_cast<int64_t>(act)));
      CK(cudaMemcpyAsync(out, t.xin(m->L), act, cudaMemcpyDeviceToDevice, ex.s));
    }
    if (retain) {
      if (live.count(id)) ex.free_tape(live[id]);
      live[id] = t;
      live_peak = std::max(live_peak, static_cast<int64_t>(live.size()));
      if (!ckpt_recompute) {
        held += cm.T;
        peak = std::max(peak, held);
      }
    } else {
      ex.free_tape(t);
      if (checkpoint) {
        held += cm.T;
        peak = std::max(peak, held);
      }
    }
    if (recompute) {
      auto k = kept_in.find(id);
      if (k != kept_in.end()) {
        pool_free(ctx, k->second);
        io_bytes -= static_cast<int64_t>(act);
        kept_in.erase(k);
      }
    } else if (in) {
      if (keep_in) {
        kept_in[id] = in;
        io_bytes += static_cast<int64_t>(act);
      } else {
        pool_free(ctx, in);
      }
    }
    op_end(t0, recompute ? kPpRecompute : kPpForward, id);
    return out;
  }

  // A checkpointed chunk gets its tape back just before its backward: a
  // retain-forward from the kept stage input (stage 0: from its tokens).
  void restore_checkpoint(int64_t id) {
    auto c = ckpt.find(id);
    if (c == ckpt.end() || live.count(id)) return;
    ckpt.erase(c);
    forward(id, true, true, false, next_extra_slot++, nullptr, false, true);
  }

  // Backward of chunk `id`.  `dy` is the gradient of the stage output (pool
  // memory, owned by the runner from here on) on stages without the head.
  // Returns the gradient of the stage input for the previous stage (caller-
  // owned) or null on the first stage.
  float* backward(int64_t id, float* dy) {
    restore_checkpoint(id);
    cudaEvent_t t0 = op_begin();
    const ChunkMeta& cm = chunk(id);
    GroupState* gs = group_for(cm);
    auto lit = live.find(id);
    if (lit == live.end())
      throw ValidationError("backward of chunk " + std::to_string(id) + " without retained activations");
    if (gs) {  // KV-gradient completeness (plan_runner.hpp:266-275)
      const int64_t n = static_cast<int64_t>(gs->contributions.size());
      if (gs->saved[static_cast<size_t>(cm.index)] &&
          gs->contributions[static_cast<size_t>(cm.index)] != n - 1 - cm.index)
        ++violations;
    }
    float* dx = dy;
    if (!m->has_head && !dy) throw ValidationError("output gradient missing for chunk " + std::to_string(id));
    if (!dx && !m->has_embed) dx = static_cast<float*>(pool_alloc(ctx, cm.T * m->d * 4));
    // this stage's last backward: each gradient range is final as soon as
    // the backward has enqueued it, so its DP all-reduce starts then, on
    // the DP stream, under the rest of the backward
    if (id == final_bwd && dp_overlap_on()) ex.on_grads_final = [this](int64_t which) { dp_allreduce(which); };
    ex.backward(cm, lit->second, gs, dx);
    if (ex.on_grads_final) {
      ex.on_grads_final = nullptr;
      dp_overlapped = true;
    }
    if (gs) {
      for (int64_t i = 0; i < cm.index; ++i) ++gs->contributions[static_cast<size_t>(i)];
      if (gs->offload) gs->dkv_valid = std::max(gs->dkv_valid, cm.start);
      if (cm.index == 0) {  // group complete: release its KV state
        free_group(*gs);
        groups.erase(cm.group);
      }
    }
    ex.free_tape(lit->second);
    live.erase(lit);
    held -= cm.T;
    op_end(t0, kPpBackward, id);
    if (m->has_embed) {
      if (dx) pool_free(ctx, dx);
      return nullptr;
    }
    return dx;
  }

  // ---- data-parallel gradient all-reduce
  int64_t final_bwd = -1;  // chunk id of this stage's last backward (set by the driver)
  bool dp_overlapped = false;
  std::vector<cudaEvent_t> dp_events;
  bool dp_overlap_on() const {
    static const bool on = [] {
      const char* e = std::getenv("CF_DP_OVERLAP");
      return !(e && std::atoi(e) == 0);
    }();
    return ctx->nccl_comm && on;
  }
  // Sum one gradient range over the DP group on the DP stream, after
  // everything enqueued so far on the step stream: -1 final norm + head,
  // l layer l, -2 the embedding.  Every replica issues the same ranges in
  // the same order (-1, L-1 .. 0, -2), which NCCL requires.
  void dp_allreduce(int64_t which) {
    const std::vector<int64_t>& go = m->layer_goff;
    int64_t lo = 0, hi = 0;
    if (which == -1) {
      lo = go.back();
      hi = m->grad_numel;
    } else if (which == -2) {
      hi = go.front();
    } else {
      lo = go[static_cast<size_t>(which)];
      hi = go[static_cast<size_t>(which) + 1];
    }
    if (hi <= lo) return;
    if (!ctx->dp_stream) CK(cudaStreamCreateWithFlags(&ctx->dp_stream, cudaStreamNonBlocking));
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    dp_events.push_back(e);
    CK(cudaEventRecord(e, ex.s));
    CK(cudaStreamWaitEvent(ctx->dp_stream, e, 0));
    nccl_check(nccl().all_reduce(m->grads + lo, m->grads + lo, static_cast<size_t>(hi - lo), kNcclFloat32, kNcclSum,
                                 ctx->nccl_comm, ctx->dp_stream),
               "ncclAllReduce(grads range)");
  }

  // Loss read-back, recompute-loss check, DP all-reduce, result fields.
  void finish(cf_run_result* res, bool dp_reduce) {
    for (auto& kv : live) ex.free_tape(kv.second);
    live.clear();
    for (auto& kv : groups) free_group(kv.second);
    groups.clear();
    for (auto& kv : kept_in) pool_free(ctx, kv.second);
    kept_in.clear();
    std::vector<double> slots(static_cast<size_t>(nslots + 1));
    CK(cudaMemcpyAsync(slots.data(), ex.loss_slots, static_cast<size_t>(nslots + 1) * 8, cudaMemcpyDeviceToHost,
                       ex.s));
    CK(cudaStreamSynchronize(ex.s));
    // per-class device time = union of the class's launch intervals (the
    // time during which at least one launch of the class was in flight);
    // equals the plain sum for launches serialised on one stream
    double cls_ms[3] = {0, 0, 0}, cls_flops[3] = {0, 0, 0};
    int64_t cls_n[3] = {0, 0, 0};
    std::vector<std::pair<double, double>> iv[3];
    for (const auto& r : ex.recs) {
      float t0 = 0, t1 = 0;
      CK(cudaEventElapsedTime(&t0, ex.recs.front().a, r.a));
      CK(cudaEventElapsedTime(&t1, ex.recs.front().a, r.b));
      iv[r.cls].emplace_back(t0, t1);
      cls_flops[r.cls] += r.flops;
      cls_n[r.cls] += r.n;
    }
    for (int c = 0; c < 3; ++c) {
      std::sort(iv[c].begin(), iv[c].end());
      double end = -1e300;
      for (const auto& [a0, a1] : iv[c]) {
        if (a0 >= end) {
          cls_ms[c] += a1 - a0;
          end = a1;
        } else if (a1 > end) {
          cls_ms[c] += a1 - end;
          end = a1;
        }
      }
    }
    // attention launches of dependent chunks (the split long sequence), the
    // same union rule restricted to them: [0] forward, [1] backward
    double dep_ms[2] = {0, 0}, dep_flops[2] = {0, 0};
    for (int c = 1; c <= 2; ++c) {
      std::vector<std::pair<double, double>> dv;
      for (const auto& r : ex.recs) {
        if (r.cls != c || !r.dep) continue;
        float t0 = 0, t1 = 0;
        CK(cudaEventElapsedTime(&t0, ex.recs.front().a, r.a));
        CK(cudaEventElapsedTime(&t1, ex.recs.front().a, r.b));
        dv.emplace_back(t0, t1);
        dep_flops[c - 1] += r.flops;
      }
      std::sort(dv.begin(), dv.end());
      double end = -1e300;
      for (const auto& [a0, a1] : dv) {
        if (a0 >= end) {
          dep_ms[c - 1] += a1 - a0;
          end = a1;
        } else if (a1 > end) {
          dep_ms[c - 1] += a1 - end;
          end = a1;
        }
      }
    }
    for (const OpMark& mk : marks) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, mk.a, mk.b));
      st->op_times.push_back({static_cast<double>(mk.kind), static_cast<double>(mk.id), static_cast<double>(ms)});
    }
    double total = 0;
    for (int64_t sl : first_pass_slots) total += slots[static_cast<size_t>(sl)];
    int64_t mism = 0;
    if (m->has_head)
      for (const auto& [sl, f] : recompute_pairs)
        if (f < 0 || slots[static_cast<size_t>(sl)] != slots[static_cast<size_t>(f)]) ++mism;
    double loss = total / norm;
    if (dp_reduce && ctx->nccl_comm) {
      // DP: gradients and loss are sums of per-rank partials (global normalizer)
      double* dl = ex.loss_slots + nslots;
      CK(cudaMemcpyAsync(dl, &loss, 8, cudaMemcpyHostToDevice, ex.s));
      if (dp_overlap_on()) {
        if (!dp_overlapped) {  // no backward on this rank: the same ranges, now
          dp_allreduce(-1);
          for (int64_t l = m->L - 1; l >= 0; --l) dp_allreduce(l);
          dp_allreduce(-2);
        }
        if (ctx->dp_stream) {
          cudaEvent_t e;
          CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          dp_events.push_back(e);
          CK(cudaEventRecord(e, ctx->dp_stream));
          CK(cudaStreamWaitEvent(ex.s, e, 0));
        }
      } else {
        nccl_check(nccl().all_reduce(m->grads, m->grads, static_cast<size_t>(m->grad_numel), kNcclFloat32,
                                     kNcclSum, ctx->nccl_comm, ex.s),
                   "ncclAllReduce(grads)");
      }
      nccl_check(nccl().all_reduce(dl, dl, 1, kNcclFloat64, kNcclSum, ctx->nccl_comm, ex.s), "ncclAllReduce(loss)");
      CK(cudaMemcpyAsync(&loss, dl, 8, cudaMemcpyDeviceToHost, ex.s));
      CK(cudaStreamSynchronize(ex.s));
      for (cudaEvent_t e : dp_events) cudaEventDestroy(e);
      dp_events.clear();
    }
    pool_free(ctx, ex.loss_slots);
    ex.loss_slots = nullptr;
    ctx->launches += ex.launches;
    if (!res) return;
    res->loss = loss;
    res->peak_retained_tokens = peak;
    res->recompute_forward_count = recomputes;
    res->recompute_loss_mismatches = mism;
    res->kv_completeness_violations = violations;
    res->tokens = st->tokens;
    res->gpu_launches = ex.launches;
    res->static_hbm_bytes = m->wbytes + m->grad_numel * 4;
    res->act_hbm_bytes = ex.act_peak;
    res->kv_hbm_bytes = ex.kv_peak;
    uint64_t high = 0;
    if (ctx->pool) cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemHigh, &high);
    res->peak_hbm_bytes = res->static_hbm_bytes + static_cast<int64_t>(high);
    const double L_ = static_cast<double>(m->L);
    res->model_flops = st->mf_layer * L_ + (m->has_head ? st->mf_head : 0.0);
    res->hw_flops = st->hw_layer * L_ + (m->has_head ? st->hw_head : 0.0);
    res->gemm_ms = cls_ms[0];
    res->gemm_flops = cls_flops[0];
    res->gemm_launches = cls_n[0];
    res->attn_ms = cls_ms[1];
    res->attn_flops = cls_flops[1];
    res->attn_launches = cls_n[1];
    res->attn_bwd_ms = cls_ms[2];
    res->attn_bwd_flops = cls_flops[2];
    res->attn_bwd_launches = cls_n[2];
    res->other_launches = ex.launches - cls_n[0] - cls_n[1] - cls_n[2];
    res->attn_dep_ms = dep_ms[0];
    res->attn_dep_flops = dep_flops[0];
    res->attn_bwd_dep_ms = dep_ms[1];
    res->attn_bwd_dep_flops = dep_flops[1];
    res->peak_live_tapes = live_peak;
    res->checkpoint_recomputes = ckpt_recomputes;
  }
};

void reset_pool_high(Ctx* ctx) {
  if (ctx->pool) {
    uint64_t zero = 0;
    cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrUsedMemHigh, &zero);
  }
}

// The stage's view of the plan: chunk-aware 1F1B op stream + per-position
// flags (pipeline.hpp:250-304 with scheduler.hpp:87-100 KV actions).
struct StagePlan {
  PpChunks info;
  std::vector<std::vector<PpOp>> orders;
};
StagePlan stage_plan(const cf_step* st, int64_t k, int64_t stages) {
  StagePlan sp;
  sp.info = pp_chunks(*st->plan, k, PpCost{});
  for (int64_t s = 0; s < stages; ++s) sp.orders.push_back(pp_stage_order(sp.info, s, stages, true));
  return sp;
}
bool first_pass_saves_kv(const cf_step* st, const ChunkMeta& cm) {
  return cm.dependent && cm.index + 1 < static_cast<int64_t>(st->plan->groups.at(cm.group).size());
}

}  // namespace

void step_run(Ctx* ctx, Model* m, cf_step* st, const cf_run_opts& opts, cf_run_result* res) {
  if (!m->has_embed || !m->has_head) throw ValidationError("a pipeline-stage model needs cf_pp_step_run");
  const Plan& plan = *st->plan;
  st->op_times.clear();
  reset_pool_high(ctx);
  StageRunner r(ctx, m, st, opts, static_cast<int64_t>(plan.events.size()));
  for (const Event& e : plan.events)
    if (e.kind == kBackward) r.final_bwd = e.chunk;
  for (size_t ei = 0; ei < plan.events.size(); ++ei) {
    const Event& e = plan.events[ei];
    if (e.kind == kBackward)
      r.backward(e.chunk, nullptr);
    else
      r.forward(e.chunk, e.kind == kFwdRetain, e.recompute, e.save_kv, static_cast<int64_t>(ei), nullptr, false);
  }
  r.finish(res, true);
}

void pp_step_run_local(Ctx* ctx, Model* const* models, int64_t P, cf_step* st, int64_t k, const cf_run_opts& opts,
                       cf_run_result* res) {
  if (P < 1) throw ValidationError("num_stages must be at least 1");
  for (int64_t s = 0; s < P; ++s) {
    int64_t b = 0, e = 0;
    pp_stage_layers(models[0]->cfg.num_layers, s, P, &b, &e);
    const Model* ms = models[s];
    if (!ms || ms->l_begin != b || ms->l_end != e || ms->has_embed != (s == 0) || ms->has_head != (s == P - 1) ||
        std::memcmp(&ms->cfg, &models[0]->cfg, sizeof(cf_model_cfg)) != 0)
      throw ValidationError("models[" + std::to_string(s) + "] is not stage " + std::to_string(s) + " of " +
                            std::to_string(P) + " of the same model");
  }
  const StagePlan sp = stage_plan(st, k, P);
  // one global order consistent with every cross-stage dependency: the
  // simulated dispatch order (start time, then stage)
  const PpTrace tr = pp_dispatch(sp.orders, sp.info.fwd, sp.info.bwd, 0.0);
  std::vector<std::tuple<double, int64_t, size_t>> seq;
  for (int64_t s = 0; s < P; ++s)
    for (size_t i = 0; i < tr.stages[static_cast<size_t>(s)].size(); ++i)
      seq.emplace_back(tr.stages[static_cast<size_t>(s)][i].start, s, i);
  std::sort(seq.begin(), seq.end());
  st->op_times.clear();
  reset_pool_high(ctx);
  std::vector<std::unique_ptr<StageRunner>> run;
  for (int64_t s = 0; s < P; ++s)
    run.emplace_back(new StageRunner(ctx, models[s], st, opts,
                                     static_cast<int64_t>(tr.stages[static_cast<size_t>(s)].size())));
  std::map<std::pair<int64_t, int64_t>, float*> act, grad;  // (stage, position) -> hand-over buffer
  auto take = [](std::map<std::pair<int64_t, int64_t>, float*>& box, int64_t s, int64_t p) {
    auto it = box.find({s, p});
    if (it == box.end()) throw std::logic_error("pipeline hand-over buffer missing");
    float* b = it->second;
    box.erase(it);
    return b;
  };
  for (const auto& [start, s, i] : seq) {
    const PpTimedOp& op = tr.stages[static_cast<size_t>(s)][i];
    const int64_t id = sp.info.ids[static_cast<size_t>(op.pos)];
    StageRunner& r = *run[static_cast<size_t>(s)];
    const ChunkMeta& cm = r.chunk(id);
    const int64_t slot = static_cast<int64_t>(i);
    if (op.kind == kPpForward) {
      const bool disc = sp.info.discarded[static_cast<size_t>(op.pos)] != 0;
      float* in = s > 0 ? take(act, s, op.pos) : nullptr;
      float* out = r.forward(id, !disc, false, first_pass_saves_kv(st, cm), slot, in, disc);
      if (out) act[{s + 1, op.pos}] = out;
    } else if (op.kind == kPpRecompute) {
      r.forward(id, true, true, false, slot, nullptr, false);
    } else {
      float* dy = s + 1 < P ? take(grad, s, op.pos) : nullptr;
      float* dx = r.backward(id, dy);
      if (dx) grad[{s - 1, op.pos}] = dx;
    }
  }
  if (!act.empty() || !grad.empty()) throw std::logic_error("unconsumed pipeline hand-over buffers");
  cf_run_result total{};
  for (int64_t s = 0; s < P; ++s) {
    cf_run_result rs{};
    run[static_cast<size_t>(s)]->finish(&rs, true);
    if (s == P - 1) {
      total.loss = rs.loss;
      total.recompute_loss_mismatches = rs.recompute_loss_mismatches;
      total.peak_retained_tokens = rs.peak_retained_tokens;
      total.recompute_forward_count = rs.recompute_forward_count;
      total.tokens = rs.tokens;
    }
    total.kv_completeness_violations += rs.kv_completeness_violations;
    total.gpu_launches += rs.gpu_launches;
    total.static_hbm_bytes += rs.static_hbm_bytes;
    total.act_hbm_bytes += rs.act_hbm_bytes;
    total.kv_hbm_bytes += rs.kv_hbm_bytes;
    total.model_flops += rs.model_flops;
    total.hw_flops += rs.hw_flops;
    total.gemm_ms += rs.gemm_ms;
    total.gemm_flops += rs.gemm_flops;
    total.gemm_launches += rs.gemm_launches;
    total.attn_ms += rs.attn_ms;
    total.attn_flops += rs.attn_flops;
    total.attn_launches += rs.attn_launches;
    total.attn_bwd_ms += rs.attn_bwd_ms;
    total.attn_bwd_flops += rs.attn_bwd_flops;
    total.attn_bwd_launches += rs.attn_bwd_launches;
    total.other_launches += rs.other_launches;
    total.attn_dep_ms += rs.attn_dep_ms;
    total.attn_dep_flops += rs.attn_dep_flops;
    total.attn_bwd_dep_ms += rs.attn_bwd_dep_ms;
    total.attn_bwd_dep_flops += rs.attn_bwd_dep_flops;
    total.peak_live_tapes = std::max(total.peak_live_tapes, rs.peak_live_tapes);
    total.checkpoint_recomputes += rs.checkpoint_recomputes;
  }
  uint64_t high = 0;
  if (ctx->pool) cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemHigh, &high);
  total.peak_hbm_bytes = total.static_hbm_bytes + static_cast<int64_t>(high);
  if (res) *res = total;
}

// ------------------------------------------------- in-process stage links
struct LocalMsg {
  float* buf = nullptr;
  size_t n = 0;
  cudaEvent_t ready = nullptr;     // sender: buffer produced
  cudaEvent_t consumed = nullptr;  // receiver: buffer copied out
  std::atomic<bool> taken{false};  // `consumed` has been recorded
};
struct LocalLink {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<std::shared_ptr<LocalMsg>> q;
};
struct LocalPipe {
  int stages = 0;
  std::vector<std::unique_ptr<LocalLink>> act, grad;  // act[s]: s -> s+1, grad[s]: s+1 -> s
};

LocalPipe* local_pipe_create(int stages) {
  if (stages < 1) throw ValidationError("num_stages must be at least 1");
  auto p = std::make_unique<LocalPipe>();
  p->stages = stages;
  for (int s = 0; s + 1 < stages; ++s) {
    p->act.emplace_back(new LocalLink);
    p->grad.emplace_back(new LocalLink);
  }
  return p.release();
}
void local_pipe_destroy(LocalPipe* p) { delete p; }
void pp_init_local(Ctx* ctx, LocalPipe* p, int stage) {
  if (!p || stage < 0 || stage >= p->stages) throw ValidationError("bad local pipeline stage");
  ctx->local = p;
  ctx->stage = stage;
  ctx->stages = p->stages;
}

namespace {

// One stage-boundary transfer, ordered against the compute stream with
// events in both directions: NCCL p2p on a link stream, or (in-process
// pipeline) a device copy on the receiver's compute stream.
struct LinkOp {
  float* buf;
  cudaEvent_t done;                // NCCL: transfer complete
  std::shared_ptr<LocalMsg> msg;   // local send: receiver's copy-out
};

cudaEvent_t new_event() {
  cudaEvent_t e;
  CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

LocalLink* local_link(Ctx* ctx, int li) {
  LocalPipe* p = ctx->local;
  const int s = ctx->stage;
  switch (li) {
    case 0: return p->act[static_cast<size_t>(s)].get();       // act up
    case 1: return p->act[static_cast<size_t>(s - 1)].get();   // act down
    case 2: return p->grad[static_cast<size_t>(s)].get();      // grad from above
    default: return p->grad[static_cast<size_t>(s - 1)].get(); // grad down
  }
}

LinkOp local_xfer(Ctx* ctx, int li, float* buf, size_t n, bool send) {
  LocalLink* L = local_link(ctx, li);
  if (send) {
    auto msg = std::make_shared<LocalMsg>();
    msg->buf = buf;
    msg->n = n;
    msg->ready = new_event();
    msg->consumed = new_event();
    CK(cudaEventRecord(msg->ready, ctx->stream));
    {
      std::lock_guard<std::mutex> lk(L->mu);
      L->q.push_back(msg);
    }
    L->cv.notify_all();
    return {buf, nullptr, msg};
  }
  std::shared_ptr<LocalMsg> msg;
  {
    std::unique_lock<std::mutex> lk(L->mu);
    if (!L->cv.wait_for(lk, std::chrono::seconds(120), [&] { return !L->q.empty(); }))
      throw std::logic_error("in-process pipeline: receive timed out (stage op streams disagree)");
    msg = L->q.front();
    L->q.pop_front();
  }
  if (msg->n != n) throw std::logic_error("in-process pipeline: transfer size mismatch");
  CK(cudaStreamWaitEvent(ctx->stream, msg->ready, 0));
  CK(cudaMemcpyAsync(buf, msg->buf, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaEventRecord(msg->consumed, ctx->stream));
  msg->taken.store(true, std::memory_order_release);
  return {buf, nullptr, nullptr};
}

LinkOp link_xfer(Ctx* ctx, int li, void* comm, int peer, float* buf, size_t n, bool send) {
  if (ctx->local) return local_xfer(ctx, li, buf, n, send);
  cudaStream_t ls = ctx->link_stream[li];
  cudaEvent_t ready = new_event(), done = new_event();
  CK(cudaEventRecord(ready, ctx->stream));  // buffer allocated / produced on the compute stream
  CK(cudaStreamWaitEvent(ls, ready, 0));
  if (send)
    nccl_check(nccl().send(buf, n, kNcclFloat32, peer, comm, ls), "ncclSend");
  else
    nccl_check(nccl().recv(buf, n, kNcclFloat32, peer, comm, ls), "ncclRecv");
  CK(cudaEventRecord(done, ls));
  if (!send) CK(cudaStreamWaitEvent(ctx->stream, done, 0));  // consumer waits for the data
  CK(cudaEventDestroy(ready));
  return {buf, done, nullptr};
}

// A send buffer may be released once the transfer (NCCL) or the receiver's
// copy (in-process) has completed; `wait` blocks until then.
bool send_complete(LinkOp& op, bool wait) {
  if (op.msg) {
    while (!op.msg->taken.load(std::memory_order_acquire)) {
      if (!wait) return false;
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    if (wait) CK(cudaEventSynchronize(op.msg->consumed));
    return cudaEventQuery(op.msg->consumed) == cudaSuccess;
  }
  if (wait) CK(cudaEventSynchronize(op.done));
  return cudaEventQuery(op.done) == cudaSuccess;
}
cudaEvent_t send_event(const LinkOp& op) { return op.msg ? op.msg->consumed : op.done; }
void release_send(LinkOp& op) {
  if (op.msg) {
    CK(cudaEventDestroy(op.msg->ready));
    CK(cudaEventDestroy(op.msg->consumed));
    op.msg.reset();
  } else {
    CK(cudaEventDestroy(op.done));
  }
}

}  // namespace

void pp_step_run(Ctx* ctx, Model* m, cf_step* st, int64_t k, const cf_run_opts& opts, cf_run_result* res) {
  const int64_t P = ctx->stages, s = ctx->stage;
  {
    int64_t b = 0, e = 0;
    pp_stage_layers(m->cfg.num_layers, s, P, &b, &e);
    if (m->l_begin != b || m->l_end != e || m->has_embed != (s == 0) || m->has_head != (s == P - 1))
      throw ValidationError("model is not stage " + std::to_string(s) + " of " + std::to_string(P));
  }
  if (P > 1 && !ctx->local &&
      ((s + 1 < P && (!ctx->act_up || !ctx->grad_up)) || (s > 0 && (!ctx->act_down || !ctx->grad_down))))
    throw ValidationError("pipeline links not initialised (cf_ctx_init_pp)");
  const StagePlan sp = stage_plan(st, k, P);
  const std::vector<PpOp>& order = sp.orders[static_cast<size_t>(s)];
  st->op_times.clear();
  reset_pool_high(ctx);
  StageRunner r(ctx, m, st, opts, static_cast<int64_t>(order.size()));
  for (const PpOp& op : order)
    if (op.kind != kPpForward && op.kind != kPpRecompute) r.final_bwd = sp.info.ids[static_cast<size_t>(op.pos)];
  std::vector<LinkOp> sends;  // output buffers in flight to a neighbour
  auto reap = [&](bool all) {
    for (size_t i = 0; i < sends.size();) {
      if (send_complete(sends[i], all)) {
        CK(cudaStreamWaitEvent(ctx->stream, send_event(sends[i]), 0));
        pool_free(ctx, sends[i].buf);
        release_send(sends[i]);
        sends[i] = sends.back();
        sends.pop_back();
      } else {
        ++i;
      }
    }
  };
  std::vector<cudaEvent_t> recv_done;
  for (size_t i = 0; i < order.size(); ++i) {
    reap(false);
    const PpOp& op = order[i];
    const int64_t id = sp.info.ids[static_cast<size_t>(op.pos)];
    const ChunkMeta& cm = r.chunk(id);
    const size_t n = static_cast<size_t>(cm.T * m->d);
    if (op.kind == kPpForward) {
      float* in = nullptr;
      if (s > 0) {
        in = static_cast<float*>(pool_alloc(ctx, static_cast<int64_t>(n) * 4));
        recv_done.push_back(link_xfer(ctx, 1, ctx->act_down, 0, in, n, false).done);
      }
      const bool disc = sp.info.discarded[static_cast<size_t>(op.pos)] != 0;
      float* out = r.forward(id, !disc, false, first_pass_saves_kv(st, cm), static_cast<int64_t>(i), in, disc);
      if (out) sends.push_back(link_xfer(ctx, 0, ctx->act_up, 1, out, n, true));
    } else if (op.kind == kPpRecompute) {
      r.forward(id, true, true, false, static_cast<int64_t>(i), nullptr, false);
    } else {
      float* dy = nullptr;
      if (s + 1 < P) {
        dy = static_cast<float*>(pool_alloc(ctx, static_cast<int64_t>(n) * 4));
        recv_done.push_back(link_xfer(ctx, 2, ctx->grad_up, 1, dy, n, false).done);
      }
      float* dx = r.backward(id, dy);
      if (dx) sends.push_back(link_xfer(ctx, 3, ctx->grad_down, 0, dx, n, true));
    }
  }
  reap(true);
  for (cudaEvent_t e : recv_done)
    if (e) CK(cudaEventDestroy(e));
  r.finish(res, true);
}

// ------------------------------------------------------ segment operators
// detail::segment_forward / segment_backward (toy_model.hpp:206, :341) on
// the GPU: one contiguous segment of one sequence with its prefix K/V passed
// in by the caller.  It runs as a one-chunk dependent step whose KV state
// spans positions [0, prefix_len + len): the caller's prefix rows are
// uploaded, the segment's own rows are written by the forward, and the same
// Exec forward / backward as run_plan does the math.
struct SegmentState {
  Ctx* ctx = nullptr;
  Model* m = nullptr;
  cf_step* st = nullptr;
  GroupState gs;
  Tape tape;
  bool kept = false;
  int64_t len = 0, prefix = 0;
  ~SegmentState() {  // no throwing frees in a destructor
    if (tape.mem) cudaFreeAsync(tape.mem, ctx->stream);
    if (gs.mem) cudaFreeAsync(gs.mem, ctx->stream);
    step_destroy(st);
  }
};

namespace {

// host fp64 [L][rows][kvw] -> bf16 rows [row0, row0 + rows) of a [L][S][kvw] cache
void upload_kv_rows(Ctx* ctx, Model* m, const double* host, int64_t rows, bf16* cache, int64_t S, int64_t row0) {
  if (rows <= 0) return;
  const int64_t n = m->L * rows * m->kvw;
  double* tmp = static_cast<double*>(pool_alloc(ctx, n * 8));
  CK(cudaMemcpyAsync(tmp, host, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, ctx->stream));
  for (int64_t l = 0; l < m->L; ++l)
    CK(cfk::f64_to_bf16(tmp + l * rows * m->kvw, rows, m->kvw, cache + (l * S + row0) * m->kvw, m->kvw, ctx->stream));
  pool_free(ctx, tmp);
  CK(cudaStreamSynchronize(ctx->stream));  // the host buffer may be reused on return
}

void upload_segment_prefix(Ctx* ctx, Model* m, SegmentState& sg, const double* pk, const double* pv) {
  if (sg.prefix == 0) return;
  if (!pk || !pv) throw ValidationError("prefix keys/values required when prefix_len > 0");
  upload_kv_rows(ctx, m, pk, sg.prefix, sg.gs.kc, sg.gs.S, 0);
  upload_kv_rows(ctx, m, pv, sg.prefix, sg.gs.vc, sg.gs.S, 0);
}

}  // namespace

SegmentState* segment_forward(Ctx* ctx, Model* m, const int32_t* tokens, int64_t len, const int64_t* targets,
                              const double* prefix_k, const double* prefix_v, int64_t prefix_len, bool keep_tape,
                              double* loss_sum, double* saved_k, double* saved_v) {
  if (!m->has_embed || !m->has_head) throw ValidationError("segment operators need an unstaged model");
  if (len < 1) throw ValidationError("segment length must be positive");
  if (prefix_len < 0) throw ValidationError("prefix_len must be non-negative");
  if (!tokens || !targets) throw ValidationError("tokens and targets are required");
  std::vector<int32_t> tk(tokens, tokens + len), tg(static_cast<size_t>(len)), ps(static_cast<size_t>(len));
  for (int64_t t = 0; t < len; ++t) {
    if (tokens[t] < 0 || tokens[t] >= m->V)
      throw ValidationError("token id " + std::to_string(tokens[t]) + " out of vocabulary range");
    if (targets[t] < -1 || targets[t] >= m->V)
      throw ValidationError("target id " + std::to_string(targets[t]) + " out of vocabulary range");
    tg[static_cast<size_t>(t)] = static_cast<int32_t>(targets[t]);
    ps[static_cast<size_t>(t)] = static_cast<int32_t>(prefix_len + t);
  }
  auto sg = std::make_unique<SegmentState>();
  sg->ctx = ctx;
  sg->m = m;
  sg->len = len;
  sg->prefix = prefix_len;
  sg->st = new cf_step();
  cf_step* st = sg->st;
  ChunkMeta cm;
  cm.dependent = true;
  cm.group = 0;
  cm.index = 0;
  cm.seq = 0;
  cm.start = prefix_len;
  cm.seq_len = prefix_len + len;
  std::vector<int32_t> meta;
  append_chunk_meta(cm, meta, tk, tg, ps, {{len, prefix_len}});
  st->chunks.push_back(cm);
  st->pos_of[0] = 0;
  st->tokens = len;
  st->meta_len = static_cast<int64_t>(meta.size());
  CK(cudaMalloc(&st->meta_dev, static_cast<size_t>(st->meta_len + 4) * 4));
  CK(cudaMemcpyAsync(st->meta_dev, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice, ctx->stream));

  GroupState& g = sg->gs;
  g.S = prefix_len + len;
  const int64_t cache = m->L * g.S * m->kvw;
  g.mem = pool_alloc(ctx, 3 * 256 + cache * 2 * 2 + cache * 2 * 4);
  Arena a{static_cast<char*>(g.mem), 0};
  g.kc = a.take<bf16>(cache);
  g.vc = a.take<bf16>(cache);
  g.dkv = a.take<float>(cache * 2);
  CK(cudaMemsetAsync(g.kc, 0, static_cast<size_t>(cache) * 2, ctx->stream));
  CK(cudaMemsetAsync(g.vc, 0, static_cast<size_t>(cache) * 2, ctx->stream));
  upload_segment_prefix(ctx, m, *sg, prefix_k, prefix_v);

  Exec ex;
  ex.ctx = ctx;
  ex.m = m;
  ex.st = st;
  ex.s = ctx->stream;
  ex.inv_norm = 1.0f;  // dlogits are rebuilt with the normalizer by segment_backward
  // everything allocated here is owned by sg (or the guard) from the moment
  // it exists, so a throwing launch leaks nothing
  struct SlotGuard {
    Ctx* c;
    double* p;
    ~SlotGuard() {
      if (p) cudaFreeAsync(p, c->stream);
    }
  } slot_guard{ctx, static_cast<double*>(pool_alloc(ctx, 8))};
  ex.loss_slots = slot_guard.p;
  CK(cudaMemsetAsync(ex.loss_slots, 0, 8, ex.s));
  sg->tape = ex.alloc_tape(len, keep_tape);
  Tape& t = sg->tape;
  ex.forward(cm, t, &g, 0, keep_tape);
  double ls = 0;
  CK(cudaMemcpyAsync(&ls, ex.loss_slots, 8, cudaMemcpyDeviceToHost, ex.s));
  // the segment's own key/value rows (what a later segment's prefix is built from)
  const int64_t n = m->L * len * m->kvw;
  double* tmp = (saved_k || saved_v) ? static_cast<double*>(pool_alloc(ctx, n * 8)) : nullptr;
  for (int kv = 0; kv < 2; ++kv) {
    double* host = kv ? saved_v : saved_k;
    if (!host) continue;
    const bf16* src = kv ? g.vc : g.kc;
    for (int64_t l = 0; l < m->L; ++l)
      CK(cfk::bf16_to_f64(src + (l * g.S + prefix_len) * m->kvw, m->kvw, len, m->kvw, tmp + l * len * m->kvw, ex.s));
    CK(cudaMemcpyAsync(host, tmp, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ex.s));
  }
  if (tmp) pool_free(ctx, tmp);
  CK(cudaStreamSynchronize(ex.s));
  ctx->launches += ex.launches;
  if (loss_sum) *loss_sum = ls;
  if (!keep_tape) return nullptr;  // ~SegmentState releases the tape and KV state
  sg->kept = true;
  return sg.release();
}

void segment_backward(Ctx* ctx, Model* m, SegmentState* sg, const double* prefix_k, const double* prefix_v,
                      double* d_prefix_k, double* d_prefix_v, const double* incoming_dk, const double* incoming_dv,
                      double normalizer) {
  if (!sg || !sg->kept) throw ValidationError("segment backward requires a retained tape");
  if (sg->m != m) throw ValidationError("segment tape belongs to another model");
  if (!(normalizer > 0)) throw ValidationError("normalizer must be positive");
  const ChunkMeta& cm = sg->st->chunks[0];
  GroupState& g = sg->gs;
  Tape& t = sg->tape;
  const int64_t T = sg->len, kvw = m->kvw;
  cudaStream_t s = ctx->stream;
  upload_segment_prefix(ctx, m, *sg, prefix_k, prefix_v);
  // dK/dV store: gradients of the segment's own rows from later chunks
  CK(cudaMemsetAsync(g.dkv, 0, static_cast<size_t>(m->L * g.S * 2 * kvw) * 4, s));
  for (int kv = 0; kv < 2; ++kv) {
    const double* host = kv ? incoming_dv : incoming_dk;
    if (!host) continue;
    const int64_t n = m->L * T * kvw;
    double* tmp = static_cast<double*>(pool_alloc(ctx, n * 8));
    CK(cudaMemcpyAsync(tmp, host, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, s));
    for (int64_t l = 0; l < m->L; ++l)
      CK(cfk::f64_to_f32(tmp + l * T * kvw, T, kvw, g.dkv + (l * g.S + sg->prefix) * 2 * kvw + kv * kvw, 2 * kvw, s));
    pool_free(ctx, tmp);
    CK(cudaStreamSynchronize(s));
  }
  Exec ex;
  ex.ctx = ctx;
  ex.m = m;
  ex.st = sg->st;
  ex.s = s;
  ex.inv_norm = static_cast<float>(1.0 / normalizer);
  // the head's dlogits are rebuilt from the forward's LSE with the caller's
  // normalizer inside ex.backward (head_backward)
  ex.backward(cm, t, &g, nullptr);
  // gradients for the prefix rows
  if (sg->prefix > 0 && (d_prefix_k || d_prefix_v)) {
    const int64_t n = m->L * sg->prefix * kvw;
    double* tmp = static_cast<double*>(pool_alloc(ctx, n * 8));
    std::vector<double> host(static_cast<size_t>(n));
    for (int kv = 0; kv < 2; ++kv) {
      double* out = kv ? d_prefix_v : d_prefix_k;
      if (!out) continue;
      for (int64_t l = 0; l < m->L; ++l)
        CK(cfk::f32_to_f64(g.dkv + l * g.S * 2 * kvw + kv * kvw, 2 * kvw, sg->prefix, kvw, tmp + l * sg->prefix * kvw,
                           s));
      CK(cudaMemcpyAsync(host.data(), tmp, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int64_t i = 0; i < n; ++i) out[i] += host[static_cast<size_t>(i)];  // accumulated, as the reference does
    }
    pool_free(ctx, tmp);
  }
  CK(cudaStreamSynchronize(s));
  ctx->launches += ex.launches;
}

void segment_destroy(SegmentState* sg) { delete sg; }

void run_plan(Ctx* ctx, Model* m, const Plan& plan, const Batch& b, const cf_run_opts& opts, cf_run_result* res) {
  cf_step* st = step_prepare(ctx, m, plan, b);
  try {
    step_run(ctx, m, st, opts, res);
  } catch (...) {
    step_destroy(st);
    throw;
  }
  step_destroy(st);
}

}  // namespace cfb
