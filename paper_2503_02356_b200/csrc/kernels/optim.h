// Fused AdamW over the flat fp32 gradient buffer (optim.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cfk {

// One storage piece of the model: its gradient elements are
// grads[goff, goff + n); the working weight (bf16, or fp32 for RMSNorm gains)
// is w[0, n) in the same element order.
struct AdamPiece {
  int64_t goff = 0, n = 0;
  void* w = nullptr;
  int32_t f32 = 0;    // working weight is fp32 (gain)
  int32_t decay = 1;  // decoupled weight decay applies
};

struct AdamHyper {
  float lr, b1, b2, eps, wd;
  float step_size;  // lr / (1 - b1^t)
  float sqrt_bc2;   // sqrt(1 - b2^t)
};

// Blocks the kernels use for n elements of one piece.
int64_t adam_blocks(int64_t n);
// coef[0] = min(1, max_norm / (||grads||_2 + 1e-6)) (1 when max_norm <= 0),
// norm_out[0] = the fp64 norm (may be null); scratch holds adam_blocks(n)
// floats.  Deterministic (fixed reduction order).
cudaError_t grad_clip_coef(const float* grads, int64_t n, float max_norm, float* scratch, float* coef,
                           double* norm_out, cudaStream_t st);
// AdamW over every piece (block_start: npieces + 1 prefix sums of
// adam_blocks(piece.n), device memory like `pieces`); clip (device, may be
// null) scales the gradient first.
cudaError_t adamw_step(const AdamPiece* pieces, int npieces, const int64_t* block_start, int64_t nblocks,
                       const float* grads, float* master, float* m, float* v, const float* clip, const AdamHyper& h,
                       cudaStream_t st);
// master = fp32 copy of the working weights.
cudaError_t master_from_weights(const AdamPiece* pieces, int npieces, const int64_t* block_start, int64_t nblocks,
                                float* master, cudaStream_t st);

}  // namespace cfk
