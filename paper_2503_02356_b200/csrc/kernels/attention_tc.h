// tcgen05 attention kernels (head_dim 128) — see attention_tc.cu.
#pragma once

#include "attention.h"

namespace cfk {

bool attn_tc_supported(const AttnParams& p);
// tiles128: 128-query tiles per segment; kv_rows: rows addressable in p.k/p.v.
cudaError_t attn_forward_tc(const AttnParams& p, const AttnTile* tiles128, int32_t ntiles, int64_t kv_rows,
                            cudaStream_t st);
// Ping-pong forward (attention_tc_fwd2.cu): one CTA = 128 queries x two q
// heads of one GQA group sharing the K/V stream; needs H/KVH even.
bool attn_fwd_pp_supported(const AttnParams& p);
cudaError_t attn_forward_tc_pp(const AttnParams& p, const AttnTile* tiles128, int32_t ntiles, int64_t kv_rows,
                               cudaStream_t st);
// dsum, then dQ (written) and dK/dV (added into the fp32 accumulators).
// Pipelined version (attention_tc_bwd.cu): 64-wide streamed sub-tiles,
// double-buffered S/dP in TMEM.
cudaError_t attn_backward_tc(const AttnParams& p, const AttnTile* qtiles128, int32_t nq, const AttnTile* ktiles128,
                             int32_t nk, int64_t kv_rows, cudaStream_t st);
// First version (attention_tc.cu): 128-wide tiles, serial MMA/softmax;
// kept selectable at operator level (cf_op_attention impl 2) for A/B tests.
cudaError_t attn_backward_tc_v1(const AttnParams& p, const AttnTile* qtiles128, int32_t nq,
                                const AttnTile* ktiles128, int32_t nk, int64_t kv_rows, cudaStream_t st);
// Testing: pseudo-random delays in every warp role of the pipelined
// backward kernels (cf_debug_set_attn_stress).
void set_attn_stress(int on);
// D = rowsum(dO * O) (shared with the warp-MMA path, attention.cu)
cudaError_t attn_dsum(const AttnParams& p, cudaStream_t st);

}  // namespace cfk
