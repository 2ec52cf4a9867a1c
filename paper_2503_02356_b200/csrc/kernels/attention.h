// Chunked causal attention over packed segments with a KV prefix
// (reference: toy_model.hpp:263-302 forward, :436-486 backward).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cfk {

// One packed segment of a chunk.  Query i (0 <= i < len, chunk row
// q_start + i) sees keys [0, prefix + i] stored at K/V rows kv_row0 + key
// (bottom-right-aligned causal mask; prefix = start_token of a dependent
// chunk, 0 for standalone segments).
struct AttnSeg {
  int32_t q_start, len, kv_row0, prefix;
};
// Work tile: 64 queries (fwd/dq) or 64 keys (dkv) of one segment.
struct AttnTile {
  int32_t seg, first, count, pad;
};

struct AttnParams {
  const __nv_bfloat16* q;  // row t, head h at q + t*q_stride + h*dh
  int64_t q_stride;
  const __nv_bfloat16* k;  // key row r, kv head g at k + r*kv_stride + g*dh
  const __nv_bfloat16* v;
  int64_t kv_stride;
  __nv_bfloat16* o;  // [T, H*dh] (stride o_stride)
  int64_t o_stride;
  float* lse;  // [H, T]: natural-log sum-exp of the scaled scores
  const __nv_bfloat16* dout;
  int64_t dout_stride;
  float* dsum;  // [H, T]: rowsum(dO * O)
  __nv_bfloat16* dq;
  int64_t dq_stride;
  float* dk_acc;  // fp32 accumulators with the K/V row indexing
  float* dv_acc;
  int64_t acc_stride;
  const AttnSeg* segs;
  const AttnTile* tiles;
  int32_t num_tiles;
  int32_t T, H, KVH, dh;
  float scale;  // 1/sqrt(dh)
  // tcgen05 backward only (attention_tc_bwd.cu), optional:
  //   rope_tab: float2 (cos, sin) [T][dh/2]: dQ leaves the kernel with the
  //             inverse rotation applied (RoPE backward) — and so does dK
  //             when dkv_out is set
  //   dkv_out:  bf16 dK / dV written directly at dkv_out + row*dkv_out_ld +
  //             {col_k, col_v} + g*dh instead of being added into
  //             dk_acc / dv_acc (standalone chunks: every key row is owned by
  //             one CTA and nothing else accumulates into it)
  const float2* rope_tab = nullptr;
  __nv_bfloat16* dkv_out = nullptr;
  int64_t dkv_out_ld = 0, col_k = 0, col_v = 0;
  //   keys_per_query: the launch's attention pairs / T when the caller knows
  //             it (0 = unknown): long-context launches (>= 3072 keys per
  //             query on average) take the 128-key-tile dQ kernel
  double keys_per_query = 0;
};

cudaError_t attn_forward(const AttnParams& p, cudaStream_t st);
// dsum = rowsum(dO*O); then dQ (written) and dK/dV (added into the fp32
// accumulators; each key row is owned by one CTA, so the result is
// deterministic).  key_tiles: tiles over keys [0, prefix+len) per segment.
cudaError_t attn_backward(const AttnParams& p, const AttnTile* key_tiles, int32_t num_key_tiles,
                          cudaStream_t st);

}  // namespace cfk
