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
  EPI_BF16_SWIGLU = 6
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
};

cudaError_t gemm(const GemmDesc& d, cudaStream_t st);
// Whether EPI_BF16_SWIGLU is available for this problem (else run EPI_BF16
// and the elementwise swiglu_fwd).
bool gemm_swiglu_ok(int64_t M, int64_t N, int64_t K);
int gemm_num_sms();
// 0 = auto (CTA-pair kernel for large GEMMs), 1 = single-CTA kernel only.
int gemm_mode();
void set_gemm_mode(int mode);

}  // namespace cfk
