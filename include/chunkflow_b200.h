/* chunkflow_b200.h — C-ABI of the B200-native ChunkFlow training path.
 *
 * This is the drop-in boundary for the reference's header-only C++ API
 * (namespace chunkflow, /root/reference/proj/include/chunkflow/).  Every
 * entry point below names the reference interface it replaces.  No torch or
 * C++ types cross this boundary: plain pointers, sizes and POD records only.
 * Errors are status codes (never exceptions); cf_last_error() returns the
 * thread-local message of the last failing call.
 *
 * Ownership: opaque handles own all device memory; host buffers are
 * caller-owned.  Threading: one host thread per cf_ctx (per GPU); a context is
 * not re-entrant.  Each call runs on the context's stream.
 */
#ifndef CHUNKFLOW_B200_H_
#define CHUNKFLOW_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Exported even when the library is built with -fvisibility=hidden. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ---- status codes: mirror the reference exception taxonomy
 *      (common.hpp:15-30) and the CLI exit codes (chunkflow_main.cpp:29-32) */
#define CF_OK 0
#define CF_EVALIDATION 1 /* chunkflow::ValidationError */
#define CF_EVERIFY 2     /* verification failure (kExitVerification) */
#define CF_EIO 3         /* chunkflow::IoError */
#define CF_ECUDA 4       /* CUDA runtime / driver error */
#define CF_ENCCL 5       /* NCCL error */
#define CF_EPARSE 6      /* chunkflow::ParseError */
#define CF_EINTERNAL 7   /* std::logic_error and anything else */

/* ---- flat plan records (exact field-for-field images of the reference
 *      structs, so layouts can be diffed bit-exactly) */

/* ChunkKind (chunker.hpp:16) */
#define CF_CHUNK_STANDALONE 0
#define CF_CHUNK_DEPENDENT 1
/* ExecKind (scheduler.hpp:17) */
#define CF_EXEC_FORWARD_DISCARD 0
#define CF_EXEC_FORWARD_RETAIN 1
#define CF_EXEC_BACKWARD 2

/* Chunk (chunker.hpp:25-32); segments live in a separate array at
 * [seg_offset, seg_offset + seg_count). */
typedef struct cf_chunk_rec {
  int64_t chunk_id;
  int64_t kind;
  int64_t group_id;       /* -1 for standalone */
  int64_t index_in_group; /* -1 for standalone */
  int64_t total_tokens;
  int64_t seg_offset;
  int64_t seg_count;
} cf_chunk_rec;

/* ChunkSegment (chunker.hpp:19-23) */
typedef struct cf_segment_rec {
  int64_t sequence_id;
  int64_t start_token;
  int64_t length;
} cf_segment_rec;

/* ExecEvent + KvActions (scheduler.hpp:20-34) */
typedef struct cf_event_rec {
  int64_t kind;
  int64_t chunk_id;
  int64_t group_id;
  int64_t index_in_group;
  int64_t is_recompute;
  int64_t save_kv;
  int64_t read_kv_prefix;
  int64_t accumulate_kv_grad;
} cf_event_rec;

/* PlanDiagnostics (scheduler.hpp:173-177); violations are counted here and
 * their text is available through cf_plan_violation(). */
typedef struct cf_plan_diag {
  int64_t peak_retained_tokens;
  int64_t recompute_token_count;
  int64_t num_violations;
} cf_plan_diag;

/* ---- model configuration (ToyModelConfig, toy_model.hpp:20-46, extended
 *      with the Llama/Qwen layer shape the north star asks for) */
#define CF_ARCH_TOY 0   /* reference toy: norm-free, no RoPE, tanh FFN (2d) */
#define CF_ARCH_LLAMA 1 /* RMSNorm + RoPE + SwiGLU, GQA, untied head */

typedef struct cf_model_cfg {
  int32_t arch;
  int32_t reserved;
  int64_t vocab_size;
  int64_t d_model;
  int64_t num_heads;
  int64_t num_kv_heads;
  int64_t num_layers;
  int64_t ffn_width; /* 0 => 2*d_model (toy); required for llama */
  uint64_t seed;
  double rope_theta; /* llama only */
  double rms_eps;    /* llama only */
} cf_model_cfg;

/* RunPlanOptions (plan_runner.hpp:49-54) */
typedef struct cf_run_opts {
  int32_t corrupt_kv_grads;   /* fault-injection hook: scale incoming dK/dV */
  int32_t accumulate_grads;   /* 0: zero grads first (reference semantics) */
  double normalizer_override; /* > 0 replaces the global target count */
  /* at most this many full activation tapes resident per stage / runner
   * (0 = no limit; meant for pipeline stages, cf_pp_step_run /
   * cf_pp_run_local, whose 1F1B warm-up keeps min(P - s, M) chunks in
   * flight).  A first-pass retain-forward that would leave no free slot keeps
   * only its stage input ([T, d] fp32; nothing on stage 0, which re-embeds its
   * tokens) and is recomputed just before its backward (stage-input
   * checkpointing); the free slot holds that just-in-time tape.  Results are
   * bitwise those without a budget. */
  int64_t stage_tape_budget;
  /* 1: dependent groups keep their KV state (K, V bf16 and the fp32 dK/dV
   * accumulators, [L][S] each) in pinned host memory; the device holds two
   * one-layer staging buffers and the rows a layer needs move on a copy
   * stream while the neighbouring layer computes (the KV offloading the
   * paper leaves for future work).  Device KV memory becomes
   * 2/L of the state; results are bitwise those without offload. */
  int32_t kv_offload;
  int32_t reserved2;
} cf_run_opts;

/* RunPlanResult + RunInstrumentation (plan_runner.hpp:36-60), plus the
 * device-side numbers the B200 runtime adds. */
typedef struct cf_run_result {
  double loss;
  int64_t peak_retained_tokens;
  int64_t recompute_forward_count;
  int64_t recompute_loss_mismatches;
  int64_t kv_completeness_violations;
  int64_t tokens;            /* real tokens processed */
  int64_t gpu_launches;      /* kernels this call launched */
  int64_t peak_hbm_bytes;    /* arena high-water mark incl. static */
  int64_t static_hbm_bytes;  /* params + grads */
  int64_t act_hbm_bytes;     /* retained-activation arena high-water */
  int64_t kv_hbm_bytes;      /* per-sequence KV-state high-water */
  double model_flops;        /* algorithmic FLOPs (no recompute) */
  double hw_flops;           /* incl. recompute */
  /* per-kernel-class device time, filled when cf_ctx_set_profiling(ctx,1):
   * CUDA events around every launch of the class on the stream it runs on;
   * *_ms is the union of those intervals (time with >= 1 launch of the
   * class in flight), so overlapping side-stream launches are not counted
   * twice */
  double gemm_ms, gemm_flops;
  int64_t gemm_launches;
  double attn_ms, attn_flops; /* attention forward */
  int64_t attn_launches;
  double attn_bwd_ms, attn_bwd_flops; /* attention backward (algorithmic FLOPs) */
  int64_t attn_bwd_launches;
  int64_t other_launches;
  /* stage-input checkpointing (cf_run_opts.stage_tape_budget): high-water of
   * full tapes resident on one stage, and the extra forwards it cost */
  int64_t peak_live_tapes;
  int64_t checkpoint_recomputes;
  /* the attention classes restricted to dependent chunks (the pieces of
   * split long sequences, which carry a KV prefix): forward / backward */
  double attn_dep_ms, attn_dep_flops;
  double attn_bwd_dep_ms, attn_bwd_dep_flops;
} cf_run_result;

typedef struct cf_ctx cf_ctx;
typedef struct cf_model cf_model;
typedef struct cf_plan cf_plan;

/* ---- errors ---- */
const char* cf_last_error(void);
const char* cf_version(void);

/* ---- planning (host, integer; bit-exact with the reference) ---- */

/* construct_chunks (chunker.hpp:177) + schedule_step (scheduler.hpp:132) +
 * validate_plan (scheduler.hpp:182).  seq_ids/lengths describe the batch
 * (Batch::sequences, dataset.hpp:75-82) in batch order. */
int cf_plan_build(const int64_t* seq_ids, const int64_t* lengths, int64_t n,
                  int64_t chunk_size, int64_t k, cf_plan** out);
/* schedule_group (scheduler.hpp:106): one abstract dependent group. */
int cf_plan_build_group(int64_t n, int64_t k, int64_t chunk_size, cf_plan** out);
/* validate_plan (scheduler.hpp:182-271) over a caller-built ExecutionPlan
 * (scheduler.hpp:36-43): `events` in execution order; ExecutionPlan.groups as
 * CSR (group_ids[g], members[group_offsets[g] .. group_offsets[g+1]), index
 * order; n_groups may be 0); ExecutionPlan.chunk_tokens as parallel arrays (a
 * chunk without an entry counts chunk_size tokens).  The result's
 * diagnostics and violation texts (the reference's, verbatim) are read with
 * cf_plan_export / cf_plan_violation, its listing with cf_plan_listing.
 * chunk_plan (may be NULL) supplies the chunks the events refer to (e.g. the
 * plan of cf_plan_build): the result then carries them and can be executed by
 * cf_run_plan / cf_step_prepare — a caller-reordered schedule.  Violations are
 * data, not an error status (as in the reference); cf_run_plan refuses a plan
 * that has any ("execution plan is invalid: ...", plan_runner.hpp:80). */
int cf_plan_validate_events(int64_t chunk_size, int64_t k, const cf_event_rec* events, int64_t n_events,
                            const int64_t* group_ids, const int64_t* group_offsets, const int64_t* members,
                            int64_t n_groups, const int64_t* token_chunk_ids, const int64_t* token_counts,
                            int64_t n_token_entries, const cf_plan* chunk_plan, cf_plan** out);
int cf_plan_counts(const cf_plan* plan, int64_t* n_chunks, int64_t* n_segments,
                   int64_t* n_events, int64_t* n_groups);
int cf_plan_export(const cf_plan* plan, cf_chunk_rec* chunks,
                   cf_segment_rec* segments, cf_event_rec* events,
                   cf_plan_diag* diag);
/* ExecutionPlan.groups (scheduler.hpp:41): group ids ascending, members in
 * index order; offsets has n_groups+1 entries.  group_ids / members may be
 * NULL to size the members array (offsets[n_groups]). */
int cf_plan_export_groups(const cf_plan* plan, int64_t* group_ids,
                          int64_t* offsets, int64_t* members);
/* text of violation i (validate_plan messages). */
int cf_plan_violation(const cf_plan* plan, int64_t i, char* buf, size_t cap);
/* execution_plan_listing (scheduler.hpp:284): writes up to cap bytes,
 * returns the full length via *len. */
int cf_plan_listing(const cf_plan* plan, char* buf, size_t cap, size_t* len);
/* Data-parallel partition (new): split the global plan's units
 * (standalone chunks and whole dependent groups) across world ranks by
 * deterministic LPT on attention+GEMM cost, then re-schedule rank's units
 * with schedule_step semantics (global chunk ids preserved). */
int cf_plan_partition(const cf_plan* global, int64_t world, int64_t rank,
                      cf_plan** out);
/* Per-unit costs used by the partitioner (for tests / reporting). */
int cf_plan_rank_tokens(const cf_plan* global, int64_t world, int64_t* tokens);
void cf_plan_destroy(cf_plan* plan);

/* ---- wire formats of the reference's planning tools ----
 * Text outputs: the full length is returned in *len; up to cap-1 bytes plus
 * a terminating NUL are written to buf (buf may be NULL to size). */

/* chunk_plan_to_json(plan).dump(2) + "\n" (chunker.hpp:233): byte-identical
 * to chunk_plan.json written by `chunkflow pack`. */
int cf_plan_chunk_json(const cf_plan* plan, char* buf, size_t cap, size_t* len);
/* execution_plan_to_json(plan).dump(2) + "\n" (scheduler.hpp:300):
 * execution_plan.json of `chunkflow schedule`. */
int cf_plan_exec_json(const cf_plan* plan, char* buf, size_t cap, size_t* len);
/* chunk_plan_from_json (chunker.hpp:261) + schedule_step(k) + validate_plan:
 * runs a chunk_plan.json produced by the reference.  CF_EPARSE on a
 * malformed document. */
int cf_plan_from_chunk_json(const char* json, int64_t k, cf_plan** out);
/* load_lengths (dataset.hpp:112): line-delimited records {id?, length,
 * tokens?}.  Call with NULL arrays to get *n and *n_tokens; has_tokens[i] is
 * 1 when record i carries its token list (concatenated into tokens). */
int cf_dataset_load_jsonl(const char* text, int64_t* n, int64_t* ids, int64_t* lengths,
                          int64_t* has_tokens, int64_t* n_tokens, int32_t* tokens);
/* write_records (dataset.hpp:169); tokens may be NULL (lengths only). */
int cf_dataset_write_jsonl(const int64_t* ids, const int64_t* lengths, const int32_t* tokens,
                           int64_t n, char* buf, size_t cap, size_t* len);

/* ---- memory model (memory_model.hpp) ---- */
typedef struct cf_mem_coeffs { /* MemoryModelCoefficients (:20-33) */
  double base_gib;
  double per_chunk_token_gib;
  double per_context_token_gib;
  double gqa_ratio;
} cf_mem_coeffs;
/* calibrate (memory_model.hpp:59): least squares of peak_gib on
 * [1, k*chunk_size, gqa_ratio*context_len]. */
int cf_mem_calibrate(const int64_t* chunk_size, const int64_t* k, const int64_t* context_len,
                     const double* peak_gib, int64_t n, double gqa_ratio, cf_mem_coeffs* out,
                     double* max_residual_gib);
/* predict_peak (memory_model.hpp:47) */
int cf_mem_predict(const cf_mem_coeffs* c, int64_t chunk_size, int64_t k, int64_t context_len,
                   double* peak_gib);
/* parse_measurements (memory_model.hpp:142): CSV rows chunk_size,k,
 * context_len,peak_gib (optional header).  NULL arrays to size *n. */
int cf_mem_parse_csv(const char* csv, int64_t* n, int64_t* chunk_size, int64_t* k,
                     int64_t* context_len, double* peak_gib);
/* coefficients_to_json(c).dump(2) + "\n" (memory_model.hpp:133) */
int cf_mem_coeffs_json(const cf_mem_coeffs* c, char* buf, size_t cap, size_t* len);

/* ---- pipeline-parallel planning (pipeline.hpp; config C5) ---- */

/* TraceEventKind (pipeline.hpp:51) */
#define CF_PP_FORWARD 0   /* first-pass forward */
#define CF_PP_RECOMPUTE 1 /* just-in-time recompute forward (F') */
#define CF_PP_BACKWARD 2

/* CostModel (pipeline.hpp:24-47) */
typedef struct cf_pp_cost {
  double gamma;
  double alpha;
  double beta;
  double backward_multiplier;
  double hop_latency;
} cf_pp_cost;

/* TraceEvent (pipeline.hpp:53-58); chunk_id is the plan's chunk id. */
typedef struct cf_pp_op {
  int64_t kind;
  int64_t chunk_id;
  double start;
  double end;
} cf_pp_op;

/* PipelineTrace summary + bubble_ratio (pipeline.hpp:64-72, 325-331). */
typedef struct cf_pp_result {
  double makespan;
  double bubble_ratio;          /* reference convention: recompute = bubble */
  double occupancy_bubble;      /* SPEC.md:344-345 convention: recompute = busy */
  int64_t ops_per_stage;        /* every stage runs the same number of ops */
} cf_pp_result;

/* simulate_state_aware_1f1b (pipeline.hpp:250-319): stage s's op stream is
 * build_stage_order (:178-210) under retention budget k; backward_first = 1
 * is DispatchPolicy::kBackwardFirst.  fwd_cost / bwd_cost (optional, one per
 * plan chunk in plan order) replace the cost model with measured per-chunk
 * times (simulator-in-the-loop).  ops (optional) receives num_stages x
 * ops_per_stage records, stage-major, in dispatch order; busy/busy_total
 * (optional) num_stages entries each. */
int cf_pp_simulate(const cf_plan* plan, int64_t num_stages, int64_t k,
                   const cf_pp_cost* cost, int backward_first,
                   const double* fwd_cost, const double* bwd_cost,
                   cf_pp_op* ops, double* busy, double* busy_total,
                   cf_pp_result* result);
/* cf_pp_simulate for the executor under a per-stage tape budget
 * (cf_run_opts.stage_tape_budget): each stage's checkpointed chunks (its op
 * stream replayed as cf_pp_stage_memory does) pay their forward again inside
 * their backward.  tape_budget = 0 is exactly cf_pp_simulate. */
int cf_pp_simulate_budget(const cf_plan* plan, int64_t num_stages, int64_t k, const cf_pp_cost* cost,
                          int backward_first, const double* fwd_cost, const double* bwd_cost, int64_t tape_budget,
                          cf_pp_op* ops, double* busy, double* busy_total, cf_pp_result* result);
/* simulate_1f1b (pipeline.hpp:218-242): whole sequences as microbatches. */
int cf_pp_simulate_1f1b(const int64_t* lengths, int64_t n, int64_t num_stages,
                        const cf_pp_cost* cost, cf_pp_op* ops, double* busy,
                        double* busy_total, cf_pp_result* result);
/* export_trace (pipeline.hpp:353-396) of num_stages x ops_per_stage records
 * (stage-major, e.g. cf_pp_simulate's output, or a measured timeline built
 * from cf_step_op_times): format 0 = chrome-trace JSON, 1 = table Gantt. */
int cf_pp_export_trace(const cf_pp_op* ops, int64_t num_stages, int64_t ops_per_stage,
                       int format, char* buf, size_t cap, size_t* len);
/* grid_search (tuner.hpp:39-112) over chunk_sizes x ks on batches sampled
 * from the sequence set (ids/lengths): state-aware 1F1B makespan (cost
 * model) averaged over batches_to_sample batches, feasibility from the memory
 * model at the longest sampled sequence vs budget_gib.  Writes ncs x nk rows
 * (chunk-size-major), the best (chunk_size, k) (-1 when none is feasible),
 * the number of simulations, and optionally the reference's CSV table
 * (csv = 1, tuner_table_csv) or ranked report (csv = 0, tuner_report) text. */
typedef struct cf_tune_row {
  int64_t chunk_size;
  int64_t k;
  double mean_time;
  double predicted_peak_gib;
  int64_t feasible;
} cf_tune_row;
int cf_tune_grid_search(const int64_t* ids, const int64_t* lengths, int64_t n,
                        const int64_t* chunk_sizes, int64_t ncs, const int64_t* ks,
                        int64_t nk, int64_t num_stages, const cf_pp_cost* cost,
                        const cf_mem_coeffs* mem, double budget_gib,
                        int64_t global_batch_size, int64_t batches_to_sample,
                        uint64_t seed, cf_tune_row* table, int64_t* best_chunk_size,
                        int64_t* best_k, int64_t* evaluations, int csv, char* buf,
                        size_t cap, size_t* len);
/* Pipeline-aware grid_search (new; the reference's tuner.hpp:39-112 sizes
 * memory as k * chunk_size retained tokens, but a 1F1B stage holds min(P - s,
 * M) chunks in flight): every sampled batch's stage op streams are replayed
 * under the executor's rules with `tape_budget` (cf_run_opts.
 * stage_tape_budget; 0 = none); a candidate is feasible when every stage's
 * base + per_chunk_token_gib * peak tape tokens + kept_token_gib * peak
 * kept-input tokens + per_context_token_gib * gqa * longest sequence fits
 * budget_gib (table rows report the worst stage).  Timing adds each stage's
 * checkpoint recomputes to its backwards.  Other arguments and outputs as
 * cf_tune_grid_search. */
int cf_tune_grid_search_pp(const int64_t* ids, const int64_t* lengths, int64_t n, const int64_t* chunk_sizes,
                           int64_t ncs, const int64_t* ks, int64_t nk, int64_t num_stages, const cf_pp_cost* cost,
                           const cf_mem_coeffs* mem, double kept_token_gib, int64_t tape_budget, double budget_gib,
                           int64_t global_batch_size, int64_t batches_to_sample, uint64_t seed,
                           cf_tune_row* table, int64_t* best_chunk_size, int64_t* best_k, int64_t* evaluations,
                           int csv, char* buf, size_t cap, size_t* len);
/* Activation memory of each stage of the chunk-aware 1F1B (retention budget
 * k) under a per-stage tape budget, replayed with the executor's rules:
 * peak resident tapes and their tokens, peak tokens of kept stage inputs
 * ([T, d] fp32 each), and how many first-pass forwards were checkpointed.
 * Arrays (may be NULL) have num_stages entries. */
int cf_pp_stage_memory(const cf_plan* plan, int64_t num_stages, int64_t k, int64_t tape_budget,
                       int64_t* peak_tapes, int64_t* peak_tape_tokens, int64_t* peak_kept_tokens,
                       int64_t* checkpointed);
/* Layer range [begin, end) that stage `stage` of `num_stages` executes. */
int cf_pp_stage_layers(int64_t num_layers, int64_t stage, int64_t num_stages,
                       int64_t* begin, int64_t* end);

/* SplitMix64 token payload exactly as chunkflow_main.cpp:427-443: one
 * stream over all sequences in order, next_below(vocab) per token. */
int cf_gen_tokens(const int64_t* lengths, int64_t n, int64_t vocab,
                  uint64_t seed, int32_t* tokens_out);
/* synthesize (dataset.hpp:207): `count` lengths from a long-tail CDF spec
 * (bounds strictly increasing, cumulative fractions in (0,1]); preset 1 =
 * eval_table5_spec (dataset.hpp:88-97), preset 2 = lmsys_table2_spec. */
int cf_synthesize(const int64_t* bounds, const double* fracs, int64_t nb,
                  int64_t max_length, int64_t preset, int64_t count,
                  uint64_t seed, int64_t* lengths_out);
/* sample_batch (dataset.hpp:242): indices of step's global batch under a
 * seed-keyed epoch shuffle of n records; *count_out = 0 past the epoch. */
int cf_sample_batch(int64_t n, int64_t global_batch, int64_t step,
                    uint64_t seed, int64_t* idx_out, int64_t* count_out);

/* ---- device context / model ---- */
int cf_ctx_create(int device, cf_ctx** out);
void cf_ctx_destroy(cf_ctx* ctx);
/* Stream the context runs on (cudaStream_t as an opaque pointer). */
void* cf_ctx_stream(cf_ctx* ctx);
/* 1: bracket every kernel launch with CUDA events and report per-class
 * device time in cf_run_result (roofline evidence); 0: off (default). */
int cf_ctx_set_profiling(cf_ctx* ctx, int on);
/* NCCL data-parallel group: nccl_unique_id is the 128-byte ncclUniqueId
 * produced by cf_nccl_unique_id on rank 0 and broadcast by the launcher. */
int cf_nccl_unique_id(uint8_t* out128);
int cf_ctx_init_dp(cf_ctx* ctx, int rank, int world, const uint8_t* id128);

/* init_model (toy_model.hpp:110): parameters drawn on the device by a
 * counter-based SplitMix64 identical to the reference's sequential stream. */
int cf_model_create(cf_ctx* ctx, const cf_model_cfg* cfg, cf_model** out);
void cf_model_destroy(cf_model* model);
int64_t cf_model_num_tensors(const cf_model* model);
/* ToyModelParams::tensors order and [rows, cols] row-major shapes. */
int cf_model_tensor_info(const cf_model* model, int64_t idx, char* name,
                         size_t cap, int64_t* rows, int64_t* cols);
int cf_model_get_param(cf_model* model, int64_t idx, double* host);
int cf_model_set_param(cf_model* model, int64_t idx, const double* host);
int cf_model_get_grad(cf_model* model, int64_t idx, double* host);
int cf_model_zero_grads(cf_model* model);
/* Flat fp32 gradient buffer (device pointer + element count), for callers
 * that reduce gradients themselves. */
int cf_model_grad_buffer(cf_model* model, void** dev_ptr, int64_t* numel);
int64_t cf_model_num_params(const cf_model* model);

/* ---- optimizer (the reference's step ends at the
 *      gradients, so this is new): fused AdamW over the flat fp32 gradient
 *      buffer with fp32 master weights, torch.optim.AdamW semantics
 *      (decoupled weight decay, bias-corrected moments) ---- */
typedef struct cf_adamw_cfg {
  double lr;
  double beta1, beta2, eps;
  double weight_decay;   /* decoupled; RMSNorm gains only with decay_gains */
  double max_grad_norm;  /* > 0: clip the global L2 norm first (clip_grad_norm_) */
  int32_t decay_gains;
  int32_t reserved;
} cf_adamw_cfg;
/* Allocates master weights (= the current weights, fp32) and zeroed moments
 * (3 x 4 bytes per parameter); resets the step counter.  Re-initialises when
 * called again.  cf_model_set_param keeps the master copy in step. */
int cf_model_adamw_init(cf_model* model);
/* One step on the gradients currently in the model (after cf_run_plan /
 * cf_step_run, all-reduced under DP): one fused HBM pass updates master,
 * moments and the bf16 working weights.  grad_norm (may be NULL) receives
 * the pre-clip global gradient norm (fp64, deterministic reduction). */
int cf_model_adamw_step(cf_model* model, const cf_adamw_cfg* cfg, double* grad_norm);
/* fp32 master copy of tensor idx (reference order / shape), as fp64. */
int cf_model_get_master(cf_model* model, int64_t idx, double* host);

/* ---- execution ---- */

/* run_plan (plan_runner.hpp:67): executes the plan's events on the GPU.
 * seq_ids/lengths/tokens: the batch, tokens concatenated in batch order
 * (host pointer).  If ctx has a DP group the gradients (and loss) are
 * all-reduced after the last event. */
int cf_run_plan(cf_ctx* ctx, cf_model* model, const cf_plan* plan,
                const int64_t* seq_ids, const int64_t* lengths,
                const int32_t* tokens, int64_t n, const cf_run_opts* opts,
                cf_run_result* result);
/* Split form of cf_run_plan for callers that keep a step's inputs resident:
 * cf_step_prepare uploads the batch (tokens + per-chunk index metadata:
 * targets, positions, cu_seqlens-style segment tables, attention tiles) once;
 * cf_step_run executes the plan's events from HBM-resident inputs. */
typedef struct cf_step cf_step;
int cf_step_prepare(cf_ctx* ctx, cf_model* model, const cf_plan* plan,
                    const int64_t* seq_ids, const int64_t* lengths,
                    const int32_t* tokens, int64_t n, cf_step** out);
int cf_step_run(cf_ctx* ctx, cf_model* model, cf_step* step,
                const cf_run_opts* opts, cf_run_result* result);
void cf_step_destroy(cf_step* step);
/* Bytes copied host -> device for the step's inputs (token ids, targets,
 * positions, segment tables, attention tiles, embedding-backward CSR): what
 * cf_step_prepare / cf_run_plan upload per step. */
int cf_step_input_bytes(const cf_step* step, int64_t* bytes);
/* Device time of every executed op (forward / recompute / backward, the
 * CF_PP_* kinds) of the step's last run when the context profiles
 * (cf_ctx_set_profiling): measured per-chunk costs for cf_pp_simulate.
 * Arrays may be NULL to query *n. */
int cf_step_op_times(const cf_step* step, int64_t* n, int64_t* kinds,
                     int64_t* chunk_ids, double* ms);
/* backward_full (toy_model.hpp:575): every sequence alone, unchunked. */
int cf_backward_full(cf_ctx* ctx, cf_model* model, const int64_t* seq_ids,
                     const int64_t* lengths, const int32_t* tokens, int64_t n,
                     double normalizer_override, cf_run_result* result);

/* Operator level: detail::segment_forward (toy_model.hpp:206-334) and
 * detail::segment_backward (toy_model.hpp:341-520) on the GPU.  One
 * contiguous segment of one sequence at positions [prefix_len,
 * prefix_len + len).  Host buffers, fp64, per layer in layer order:
 *   prefix_k / prefix_v   [L][prefix_len][kv_width] (NULL when prefix_len = 0)
 *   saved_k / saved_v     [L][len][kv_width], the segment's own key/value rows
 *                         (SegmentTape::saved_k/v; may be NULL)
 *   incoming_dk / _dv     [L][len][kv_width], gradients of those rows from
 *                         later chunks (NULL = absent)
 *   d_prefix_k / _v       [L][prefix_len][kv_width], accumulated (+=)
 * targets[t] = -1 marks a position without a prediction target.  loss_sum
 * is the unnormalized cross-entropy over target positions
 * (SegmentTape::loss_sum).  keep_tape = 0 returns *tape = NULL (a
 * discarded forward); otherwise the retained activations stay on the device
 * until cf_segment_destroy.  cf_segment_backward accumulates the parameter
 * gradients into the model's gradient buffer (the reference's GradientSet&;
 * cf_model_zero_grads clears it) with the normalizer given here.  Keys are
 * post-RoPE for the Llama arch (what the executor caches).  A tape without
 * retained activations is CF_EVALIDATION, like the reference's
 * "segment backward requires a retained tape". */
typedef struct cf_segment cf_segment;
int cf_segment_forward(cf_ctx* ctx, cf_model* model, const int32_t* tokens, int64_t len,
                       const int64_t* targets, const double* prefix_k, const double* prefix_v,
                       int64_t prefix_len, int keep_tape, double* loss_sum, double* saved_k,
                       double* saved_v, cf_segment** tape);
int cf_segment_backward(cf_ctx* ctx, cf_model* model, const cf_segment* tape,
                        const double* prefix_k, const double* prefix_v, double* d_prefix_k,
                        double* d_prefix_v, const double* incoming_dk, const double* incoming_dv,
                        double normalizer);
void cf_segment_destroy(cf_segment* tape);
int cf_ctx_synchronize(cf_ctx* ctx);

/* ---- pipeline-parallel execution (config C5; the reference only simulates
 *      this, pipeline.hpp:214-319) ---- */

/* Stage `stage` of `num_stages` of the model cfg describes: global layers
 * cf_pp_stage_layers(...), the embedding on stage 0, final norm + head + loss
 * on the last stage.  Weights equal the full model's (same SplitMix64 draws);
 * tensor names keep global layer numbers. */
int cf_model_create_stage(cf_ctx* ctx, const cf_model_cfg* cfg, int64_t stage,
                          int64_t num_stages, cf_model** out);
/* PP x DP communicators: rank = replica * num_stages + stage; id128 from
 * cf_nccl_unique_id on rank 0.  Gradients are all-reduced over the ranks of
 * the same stage; activations/gradients cross stage links with NCCL p2p. */
int cf_ctx_init_pp(cf_ctx* ctx, int rank, int world, int num_stages,
                   const uint8_t* id128);
/* This rank's stage of the chunk-aware 1F1B step: runs the stage's op stream
 * (build_stage_order semantics, retention budget k) with fp32 [T, d]
 * activations sent up and gradients sent down.  result->loss is the loss on
 * the last stage (0 elsewhere). */
int cf_pp_step_run(cf_ctx* ctx, cf_model* model, cf_step* step, int64_t k,
                   const cf_run_opts* opts, cf_run_result* result);
/* In-process pipeline links (testing the per-rank path on one device): each
 * stage's context — driven by its own host thread — attaches to one shared
 * cf_pp_local; cf_pp_step_run then exchanges stage-boundary buffers through
 * host mailboxes, CUDA events and device copies instead of NCCL. */
typedef struct cf_pp_local cf_pp_local;
int cf_pp_local_create(int num_stages, cf_pp_local** out);
void cf_pp_local_destroy(cf_pp_local* pipe);
int cf_ctx_init_pp_local(cf_ctx* ctx, cf_pp_local* pipe, int stage);
/* Every stage of one pipeline on this context's device (models[i] = stage
 * i): the same op streams in dispatch order with in-memory hand-over.
 * Gradients are bitwise those of cf_step_run on the unsplit model. */
int cf_pp_run_local(cf_ctx* ctx, cf_model* const* models, int64_t num_stages,
                    cf_step* step, int64_t k, const cf_run_opts* opts,
                    cf_run_result* result);

/* ---- operator level (kernel unit tests); all pointers are device ---- */

/* C[M,N] (+)= sum_k A(m,k) B(n,k).  a_kmajor: A stored [M,K] (else [K,M]);
 * b_kmajor: B stored [N,K] (else [K,N]).  epi: 0 store bf16, 1 store fp32,
 * 2 accumulate into fp32, 3 fp32 store of acc + residual(fp32), 4 bf16 tanh,
 * 5 bf16 acc*(1-R^2) (toy FFN backward). */
/* Chunked causal attention over packed segments (toy_model.hpp:263-302
 * forward, :436-486 backward).  segs: host int32 [nseg][4] = {q_start, len,
 * kv_row0, prefix}.  impl 0 = warp-MMA kernels, 1 = tcgen05 (head_dim 128),
 * 2 = first tcgen05 backward, 3 = ping-pong tcgen05 forward (two q heads of a
 * GQA group per CTA; H/KVH even).
 * Backward writes dq and ADDS dK/dV into the fp32 accumulators. */
int cf_op_attention(cf_ctx* ctx, int impl, int backward, const void* q,
                    int64_t q_stride, const void* k, const void* v,
                    int64_t kv_stride, int64_t kv_rows, void* o, float* lse,
                    const void* dout, void* dq, float* dk_acc, float* dv_acc,
                    int64_t acc_stride, const int32_t* segs, int64_t nseg,
                    int64_t T, int64_t H, int64_t KVH, int64_t dh);
/* GEMM kernel selection (testing / A-B measurement): 0 = auto (CTA-pair
 * tcgen05.mma.cta_group::2 kernel for large GEMMs), 1 = single-CTA kernel
 * only, 2 = CTA pairs whenever M, N > 128. */
int cf_debug_set_gemm_mode(int mode);
/* Attention-backward synchronisation stress (testing): nonzero inserts
 * pseudo-random 0-2 us delays at every mbarrier hand-off of the tcgen05
 * dQ and dK/dV kernels (producer, MMA issuer, softmax warps); the results
 * must not change. */
int cf_debug_set_attn_stress(int on);
int cf_op_gemm(cf_ctx* ctx, const void* a, int a_kmajor, int64_t lda,
               const void* b, int b_kmajor, int64_t ldb, void* c, int64_t ldc,
               int64_t m, int64_t n, int64_t k, int epi, const void* residual,
               int64_t ld_res);
/* The q|k|v projection with RoPE (and the KV-cache copy) in its epilogue:
 * C[m, n] = bf16(A[m, k] W[k, n]) then rotate-half RoPE on the q and k heads
 * (head_dim 128; columns [0, col_v)) with tab = float2 (cos, sin) [m][64];
 * kc / vc (may be NULL) receive the k columns [col_k, col_v) and the v
 * columns [col_v, n) with row pitch cache_ld.  CF_EVALIDATION-class error
 * (cudaErrorInvalidValue) when the shape is not eligible (tile alignment). */
/* Fused LM head + cross-entropy (the path run_plan uses): x bf16 [T, d]
 * (row pitch d), head bf16 [d, ldh] ([in, out], columns >= V ignored),
 * targets int32 [T] (-1 = no target).  Writes lse [T] and row_loss [T]
 * (lse - logit[target], 0 without a target) from the head GEMM's epilogue
 * partials; when dlogits != NULL also the bf16 [T, ldh] gradient
 * (softmax - onehot) * inv_norm recomputed by a second head GEMM.  All
 * pointers are device pointers. */
int cf_op_lm_head_ce(cf_ctx* ctx, const void* x, const void* head, int64_t ldh, int64_t T, int64_t V, int64_t d,
                     const int32_t* targets, float inv_norm, float* lse, float* row_loss, void* dlogits);
int cf_op_gemm_rope(cf_ctx* ctx, const void* a, int64_t lda, const void* w, int64_t ldw,
                    void* c, int64_t m, int64_t n, int64_t k, const void* tab,
                    int64_t col_k, int64_t col_v, void* kc, void* vc, int64_t cache_ld);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* CHUNKFLOW_B200_H_ */
