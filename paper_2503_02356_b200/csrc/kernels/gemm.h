// tcgen05 GEMM launcher (see gemm.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cfk {

enum GemmEpi : int {
  EPI_BF16 = 0,          // C(bf16)  = acc
  EPI_F32 = 1,           // C(fp32)  = acc
  EPI_F32_ACC = 2,       // C(fp32) += acc              (weight-gradient accumulation)
  EPI_F32_RES = 3,       // C(fp32)  = acc + R(fp32)    (residual; R may alias C)
  EPI_BF16_TANH = 4,     // C(bf16)  = tanh(acc)        (toy FFN)
  EPI_BF16_TANHGRAD = 5, // C(bf16)  = acc * (1 - R^2)  (toy FFN backward, R = h bf16)
  // C(bf16) = acc over [gate | up] (N = 2F columns) and, in the same
  // epilogue, H(bf16)[M, F] = silu(gate) * up from the bf16-rounded values
  // (H is passed as r / ldr).  Each CTA-pair tile pairs gate columns
  // [128j, 128j+128) with up columns F + [128j, 128j+128).  CTA-pair kernel,
  // F % 128 == 0 only (gemm_swiglu_ok).
  EPI_BF16_SWIGLU = 6,
  // C(bf16) = acc over [q | k | v] with rotate-half RoPE applied to the q and
  // k columns (head_dim 128, R = float2 (cos, sin) table [M][64], ldr = 64,
  // from the bf16-rounded values as rope_qk does), and the k / v columns
  // also written to kc / vc (the KV cache rows of these tokens) when set.
  // CTA-pair kernel only (gemm_rope_ok).
  EPI_BF16_ROPE = 7,
  // Fused LM-head cross-entropy, forward (toy_model.hpp:320-331): nothing is
  // stored to C.  Per row and 256-column slab the epilogue writes the online
  // softmax partial (max, sum exp) to ce_part[row * ce_nparts + slab] and the
  // target column's logit to ce_tlogit[row]; ce_finish() combines them into
  // the row's log-sum-exp and loss.  No [T, V] logits ever reach HBM.
  EPI_CE_STATS = 8,
  // Fused LM-head cross-entropy, backward (toy_model.hpp:369-388): C(bf16) =
  // (exp(acc - ce_lse[row]) - [col == ce_tgt[row]]) * ce_scale, 0 for rows
  // without a target: dlogits recomputed from the saved LSE instead of being
  // kept from the forward.
  EPI_CE_GRAD = 9
};

struct GemmDesc {
  const void* a;  // bf16
  int64_t lda;
  int a_kmajor;   // 1: A[M,K] row-major; 0: A stored [K,M]
  const void* b;  // bf16
  int64_t ldb;
  int b_kmajor;   // 1: B[N,K] row-major; 0: B stored [K,N]
  void* c;
  int64_t ldc;
  const void* r;
  int64_t ldr;
  int64_t M, N, K;
  int epi;
  // EPI_BF16_ROPE: column where k starts / v starts, KV-cache copies
  int64_t col_k = 0, col_v = 0;
  void* kc = nullptr;
  void* vc = nullptr;
  int64_t cache_ld = 0;
  // EPI_CE_STATS / EPI_CE_GRAD
  const int32_t* ce_tgt = nullptr;  // [M] target column or -1
  float* ce_part = nullptr;         // [M][ce_nparts] float2 (max, sum)   STATS
  float* ce_tlogit = nullptr;       // [M] target logit                    STATS
  const float* ce_lse = nullptr;    // [M] log-sum-exp                      GRAD
  float ce_scale = 0.f;             // 1 / normalizer                       GRAD
};

// Partial-slab count of EPI_CE_STATS for N columns (one per 256 columns).
inline int64_t ce_nparts(int64_t N) { return (N + 255) / 256; }
// lse[row] = logsumexp over the row's partials; row_loss[row] = lse -
// tlogit[row] for rows with a target (0 otherwise).  One warp per row, fixed
// combine order (deterministic).
cudaError_t ce_finish(const float* part, int64_t nparts, const float* tlogit, const int32_t* tgt, int64_t M,
                      float* lse, float* row_loss, cudaStream_t st);

cudaError_t gemm(const GemmDesc& d, cudaStream_t st);
// Two EPI_F32_ACC GEMMs with the same operand majors in one CTA-pair launch
// (their tiles share the persistent grid's waves); falls back to two gemm()
// calls when either would not take the pair kernel.
cudaError_t gemm2(const GemmDesc& d0, const GemmDesc& d1, cudaStream_t st);
// Whether EPI_BF16_SWIGLU is available for this problem (else run EPI_BF16
// and the elementwise swiglu_fwd).
bool gemm_swiglu_ok(int64_t M, int64_t N, int64_t K);
// Whether EPI_BF16_ROPE is available ([q | k | v] of width N, head_dim dh,
// k at col_k, v at col_v; else run EPI_BF16 + rope_qk + kv_store).
bool gemm_rope_ok(int64_t M, int64_t N, int64_t K, int64_t dh, int64_t col_k, int64_t col_v);
int gemm_num_sms();
// 0 = auto (CTA-pair kernel for large GEMMs), 1 = single-CTA kernel only.
int gemm_mode();
void set_gemm_mode(int mode);

}  // namespace cfk
