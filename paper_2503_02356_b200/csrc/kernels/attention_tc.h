// tcgen05 attention kernels (head_dim 128) — see attention_tc.cu.
#pragma once

#include "attention.h"

namespace cfk {

bool attn_tc_supported(const AttnParams& p);
// tiles128: 128-query tiles per segment; kv_rows: rows addressable in p.k/p.v.
cudaError_t attn_forward_tc(const AttnParams& p, const AttnTile* tiles128, int32_t ntiles, int64_t kv_rows,
                            cudaStream_t st);

}  // namespace cfk
