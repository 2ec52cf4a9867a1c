// Fused AdamW step over the model's flat fp32 gradient buffer (SURVEY
// §8(f)-4; the reference stops at loss + gradients, so this is the B200
// runtime's own optimizer).  fp32 master weights, first and second moments
// live in the gradient buffer's layout; one pass reads g, m, v, master and
// writes m, v, master and the bf16 (or fp32 gain) working weight the
// forward reads — 4 + 4 + 4 + 4 B in, 4 + 4 + 4 + 2 B out per parameter, an
// HBM-bound stream.  Optional global-norm clipping is a deterministic
// two-kernel reduction (per-block fp32 partials, one fixed-order fp64 sum)
// whose coefficient stays on the device.
#include <cmath>

#include "common.cuh"
#include "ops.h"
#include "optim.h"

namespace cfk {
namespace {

constexpr int kThreads = 256;
constexpr int kVec = 4;                          // float4 per thread per step
constexpr int64_t kBlockElems = kThreads * kVec * 4;  // 4096 elements per block

__global__ void sumsq_partial_kernel(const float* __restrict__ g, int64_t n, float* __restrict__ part) {
  __shared__ float red[kThreads / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kBlockElems;
  float s = 0.f;
  for (int64_t i = base + static_cast<int64_t>(threadIdx.x) * kVec; i < min(base + kBlockElems, n);
       i += kThreads * kVec) {
    if (i + kVec <= n) {
      const float4 v = *reinterpret_cast<const float4*>(g + i);
      s = fmaf(v.x, v.x, s);
      s = fmaf(v.y, v.y, s);
      s = fmaf(v.z, v.z, s);
      s = fmaf(v.w, v.w, s);
    } else {
      for (int64_t j = i; j < n; ++j) s = fmaf(g[j], g[j], s);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// One block: fixed-order fp64 sum of the partials -> norm and clip coefficient
// (torch.nn.utils.clip_grad_norm_: coef = max_norm / (norm + 1e-6), <= 1).
__global__ void clip_coef_kernel(const float* __restrict__ part, int64_t nparts, float max_norm, float* coef,
                                 double* norm_out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < nparts; i += blockDim.x) s += static_cast<double>(part[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double norm = sqrt(red[0]);
    if (norm_out) *norm_out = norm;
    const double c = max_norm > 0.f ? static_cast<double>(max_norm) / (norm + 1e-6) : 1.0;
    *coef = static_cast<float>(c < 1.0 ? c : 1.0);
  }
}

// Blocks are laid out piece by piece (block_start[p] .. block_start[p+1]);
// a block finds its piece by binary search over the small piece table.
__global__ void __launch_bounds__(kThreads) adamw_kernel(const AdamPiece* __restrict__ pieces, int npieces,
                                                         const int64_t* __restrict__ block_start,
                                                         const float* __restrict__ grads, float* __restrict__ master,
                                                         float* __restrict__ m, float* __restrict__ v,
                                                         const float* __restrict__ clip, AdamHyper h) {
  int lo = 0, hi = npieces - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_start[mid] <= blockIdx.x)
      lo = mid;
    else
      hi = mid - 1;
  }
  const AdamPiece pc = pieces[lo];
  const float gscale = clip ? *clip : 1.f;
  const float decay = pc.decay ? h.lr * h.wd : 0.f;
  const int64_t first = (static_cast<int64_t>(blockIdx.x) - block_start[lo]) * kBlockElems;
  const int64_t last = first + kBlockElems < pc.n ? first + kBlockElems : pc.n;
  for (int64_t e = first + static_cast<int64_t>(threadIdx.x) * kVec; e < last; e += kThreads * kVec) {
    const int64_t gi = pc.goff + e;
    const int cnt = static_cast<int>(last - e < kVec ? last - e : kVec);
    float gg[kVec], mm[kVec], vv[kVec], ww[kVec];
    if (cnt == kVec) {
      const float4 a = *reinterpret_cast<const float4*>(grads + gi);
      const float4 b = *reinterpret_cast<const float4*>(m + gi);
      const float4 c = *reinterpret_cast<const float4*>(v + gi);
      const float4 d = *reinterpret_cast<const float4*>(master + gi);
      gg[0] = a.x; gg[1] = a.y; gg[2] = a.z; gg[3] = a.w;
      mm[0] = b.x; mm[1] = b.y; mm[2] = b.z; mm[3] = b.w;
      vv[0] = c.x; vv[1] = c.y; vv[2] = c.z; vv[3] = c.w;
      ww[0] = d.x; ww[1] = d.y; ww[2] = d.z; ww[3] = d.w;
    } else {
      for (int j = 0; j < kVec; ++j) {
        const bool in = j < cnt;
        gg[j] = in ? grads[gi + j] : 0.f;
        mm[j] = in ? m[gi + j] : 0.f;
        vv[j] = in ? v[gi + j] : 0.f;
        ww[j] = in ? master[gi + j] : 0.f;
      }
    }
#pragma unroll
    for (int j = 0; j < kVec; ++j) {
      // torch.optim.AdamW (decoupled decay, then the bias-corrected step)
      const float g = gg[j] * gscale;
      ww[j] -= decay * ww[j];
      mm[j] = h.b1 * mm[j] + (1.f - h.b1) * g;
      vv[j] = h.b2 * vv[j] + (1.f - h.b2) * g * g;
      const float denom = sqrtf(vv[j]) / h.sqrt_bc2 + h.eps;
      ww[j] -= h.step_size * mm[j] / denom;
    }
    if (cnt == kVec) {
      *reinterpret_cast<float4*>(m + gi) = make_float4(mm[0], mm[1], mm[2], mm[3]);
      *reinterpret_cast<float4*>(v + gi) = make_float4(vv[0], vv[1], vv[2], vv[3]);
      *reinterpret_cast<float4*>(master + gi) = make_float4(ww[0], ww[1], ww[2], ww[3]);
      if (pc.f32) {
        *reinterpret_cast<float4*>(static_cast<float*>(pc.w) + e) = make_float4(ww[0], ww[1], ww[2], ww[3]);
      } else {
        *reinterpret_cast<uint2*>(static_cast<bf16*>(pc.w) + e) =
            make_uint2(pack_bf16(ww[0], ww[1]), pack_bf16(ww[2], ww[3]));
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        m[gi + j] = mm[j];
        v[gi + j] = vv[j];
        master[gi + j] = ww[j];
        if (pc.f32)
          static_cast<float*>(pc.w)[e + j] = ww[j];
        else
          static_cast<bf16*>(pc.w)[e + j] = __float2bfloat16_rn(ww[j]);
      }
    }
  }
}

__global__ void master_from_weights_kernel(const AdamPiece* __restrict__ pieces, int npieces,
                                           const int64_t* __restrict__ block_start, float* __restrict__ master) {
  int lo = 0, hi = npieces - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_start[mid] <= blockIdx.x)
      lo = mid;
    else
      hi = mid - 1;
  }
  const AdamPiece pc = pieces[lo];
  const int64_t first = (static_cast<int64_t>(blockIdx.x) - block_start[lo]) * kBlockElems;
  const int64_t last = first + kBlockElems < pc.n ? first + kBlockElems : pc.n;
  for (int64_t e = first + threadIdx.x; e < last; e += kThreads)
    master[pc.goff + e] = pc.f32 ? static_cast<const float*>(pc.w)[e] : __bfloat162float(static_cast<const bf16*>(pc.w)[e]);
}

}  // namespace

int64_t adam_blocks(int64_t n) { return (n + kBlockElems - 1) / kBlockElems; }

cudaError_t grad_clip_coef(const float* grads, int64_t n, float max_norm, float* scratch, float* coef,
                           double* norm_out, cudaStream_t st) {
  const int64_t nb = adam_blocks(n);
  if (nb == 0) return cudaSuccess;
  sumsq_partial_kernel<<<static_cast<unsigned>(nb), kThreads, 0, st>>>(grads, n, scratch);
  clip_coef_kernel<<<1, 1024, 0, st>>>(scratch, nb, max_norm, coef, norm_out);
  return cudaGetLastError();
}

cudaError_t adamw_step(const AdamPiece* pieces, int npieces, const int64_t* block_start, int64_t nblocks,
                       const float* grads, float* master, float* m, float* v, const float* clip, const AdamHyper& h,
                       cudaStream_t st) {
  if (nblocks == 0) return cudaSuccess;
  adamw_kernel<<<static_cast<unsigned>(nblocks), kThreads, 0, st>>>(pieces, npieces, block_start, grads, master, m,
                                                                    v, clip, h);
  return cudaGetLastError();
}

cudaError_t master_from_weights(const AdamPiece* pieces, int npieces, const int64_t* block_start, int64_t nblocks,
                                float* master, cudaStream_t st) {
  if (nblocks == 0) return cudaSuccess;
  master_from_weights_kernel<<<static_cast<unsigned>(nblocks), kThreads, 0, st>>>(pieces, npieces, block_start,
                                                                                  master);
  return cudaGetLastError();
}

}  // namespace cfk
