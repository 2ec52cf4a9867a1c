// Bandwidth-bound kernels of the chunk forward/backward (elementwise.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cfk {

using bf16 = __nv_bfloat16;

// Counter-based SplitMix64 init (toy_model.hpp:128-132): element (r, c) of a
// reference tensor takes draw number draw_base + r*cols + c of the stream
// seeded with `seed`; value (u*2-1)*scale computed in fp64, rounded to bf16.
cudaError_t init_uniform_bf16(bf16* dst, int64_t ld, int64_t rows, int64_t cols, uint64_t draw_base, uint64_t seed,
                              double scale, cudaStream_t st);
cudaError_t fill_f32(float* dst, int64_t n, float v, cudaStream_t st);
// x[t, :] = E[tok[t], :] (bf16 -> fp32)
cudaError_t embed_fwd(const int32_t* tok, const bf16* E, int64_t d, int64_t T, float* x, cudaStream_t st);
// y = bf16(x * rsqrt(mean(x^2) + eps) * gain)
cudaError_t rmsnorm_fwd(const float* x, const float* gain, int64_t T, int64_t d, float eps, bf16* y,
                        cudaStream_t st);
cudaError_t to_bf16(const float* x, bf16* y, int64_t n, cudaStream_t st);
// RoPE table [T, dh/2] of (cos, sin) at integer positions (fp64 angles).
cudaError_t rope_table(const int32_t* pos, int64_t T, int dh, double theta, float2* tab, cudaStream_t st);
// Rotate-half RoPE in place on the q heads (cols [0, H*dh)) and k heads
// (cols [col_k, col_k + KVH*dh)) of a [T, ld] bf16 buffer.
cudaError_t rope_qk(bf16* qkv, int64_t ld, int64_t T, int H, int KVH, int dh, int64_t col_k, const float2* tab,
                    cudaStream_t st);
// Copies k/v columns of T rows into the per-sequence KV cache rows.
cudaError_t kv_store(const bf16* qkv, int64_t ld, int64_t T, int64_t kvw, int64_t col_k, int64_t col_v, bf16* kc,
                     bf16* vc, int64_t cache_ld, cudaStream_t st);
cudaError_t swiglu_fwd(const bf16* gu, int64_t T, int64_t ffn, bf16* h, cudaStream_t st);
cudaError_t swiglu_bwd(const bf16* gu, const bf16* dh, int64_t T, int64_t ffn, bf16* dgu, cudaStream_t st);
// Per row: loss = lse(logits) - logits[target] (0 if target < 0);
// dlogits = (softmax - onehot) * inv_norm (zeros if target < 0; skipped if null).
cudaError_t ce_fwd_bwd(const float* logits, int64_t T, int64_t V, int64_t ld, const int32_t* targets, float inv_norm,
                       float* row_loss, bf16* dlogits, cudaStream_t st);
// out[0] = sum(v[0..n)) in fp64, fixed reduction order (deterministic).
cudaError_t sum_f64(const float* v, int64_t n, double* out, cudaStream_t st);
// dx = dres + d(rmsnorm)/dx^T dy  (dres may alias dx; may be null); writes rstd.
cudaError_t rmsnorm_bwd(const float* x, const float* gain, const float* dy, const float* dres, int64_t T, int64_t d,
                        float eps, float* dx, float* rstd, cudaStream_t st);
// Fused: dx = dres + d(rmsnorm)/dx^T dy (dres may alias dx; may be null),
// optional bf16 copy of dx, and dgain[c] += sum_t dy*x*rstd (fixed order:
// per-CTA row-range partials, then a column reduction).  Needs d % 4 == 0
// and d <= 8192 (rmsnorm_bwd_fused_ok).
cudaError_t rmsnorm_bwd_fused(const float* x, const float* gain, const float* dy, const float* dres, int64_t T,
                              int64_t d, float eps, float* dx, bf16* dx_bf16, float* dgain, cudaStream_t st);
bool rmsnorm_bwd_fused_ok(int64_t d);
// dgain[c] += sum_t dy[t,c] * x[t,c] * rstd[t]   (fixed order)
cudaError_t gain_grad(const float* x, const float* dy, const float* rstd, int64_t T, int64_t d, float* dgain,
                      cudaStream_t st);
// Own-row fp32 dK/dV accumulators -> bf16 columns of dqkv (RoPE-backward on
// dK when tab != null).
cudaError_t dkv_to_dqkv(const float* dk, const float* dv, int64_t acc_ld, int64_t T, int KVH, int dh,
                        const float2* tab, bf16* dqkv, int64_t ld, int64_t col_k, int64_t col_v, cudaStream_t st);
cudaError_t rope_bwd_q(bf16* dqkv, int64_t ld, int64_t T, int H, int dh, const float2* tab, cudaStream_t st);
cudaError_t scale_rows_f32(float* x, int64_t rows, int64_t cols, int64_t ld, float s, cudaStream_t st);
// dE[tok] += sum of dx rows listed in order[off[u] .. off[u+1]) for token uniq[u].
cudaError_t embed_bwd(const float* dx, int64_t d, const int32_t* order, const int32_t* uniq, const int32_t* off,
                      int64_t nuniq, float* dE, cudaStream_t st);
// Strided bf16 -> fp64 / fp64 -> bf16 copies used by parameter get/set.
cudaError_t bf16_to_f64(const bf16* src, int64_t ld, int64_t rows, int64_t cols, double* dst, cudaStream_t st);
cudaError_t f64_to_bf16(const double* src, int64_t rows, int64_t cols, bf16* dst, int64_t ld, cudaStream_t st);
cudaError_t f32_to_f64(const float* src, int64_t ld, int64_t rows, int64_t cols, double* dst, cudaStream_t st);
cudaError_t f64_to_f32(const double* src, int64_t rows, int64_t cols, float* dst, int64_t ld, cudaStream_t st);

}  // namespace cfk
