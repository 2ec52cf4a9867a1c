// Chunked causal attention (packed segments + KV prefix + GQA) for sm_100a.
//
// Forward (reference toy_model.hpp:263-302): flash-style online softmax over
// 64-key tiles, bottom-right-aligned causal mask (query i of a segment sees
// keys [0, prefix + i]); writes O (bf16) and LSE (fp32, natural log).
// Backward (reference :436-486), deterministic by ownership:
//   dsum kernel   D = rowsum(dO * O)
//   dq kernel     one CTA per (64-query tile, q head): loops key tiles
//   dkv kernel    one CTA per (64-key tile, kv head): loops every q head of
//                 the GQA group and every query tile that sees the keys, and
//                 adds dK/dV into the fp32 KV-gradient store (each key row is
//                 owned by exactly one CTA -> no float atomics).
// First version: warp-level mma.sync m16n8k16 tiles with cp.async double
// buffering and an XOR-swizzled smem layout (ldmatrix conflict-free).
#include <cfloat>

#include "attention.h"
#include "common.cuh"

namespace cfk {
namespace {

using bf16 = __nv_bfloat16;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm4t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Element offset of (row, 16B-chunk) in a swizzled [64][DH] tile.
template <int DH>
__device__ __forceinline__ int sw(int row, int chunk) {
  return row * DH + ((chunk ^ (row & 7)) << 3);
}

// Loads rows [0, nvalid) of a 64 x dh tile (row stride `stride`), zero-fills
// the rest.  `safe` is any valid global address (source for zero-fills).
template <int DH>
__device__ __forceinline__ void load_tile(bf16* s, const bf16* base, int64_t stride, int nvalid, int dh, bool vec,
                                          const bf16* safe) {
  constexpr int CH = DH / 8;
  if (vec) {
    for (int i = threadIdx.x; i < 64 * CH; i += blockDim.x) {
      const int r = i / CH, c = i % CH;
      const bool ok = r < nvalid && c * 8 < dh;
      cp_async16(s + sw<DH>(r, c), ok ? base + static_cast<int64_t>(r) * stride + c * 8 : safe, ok ? 16 : 0);
    }
  } else {
    for (int i = threadIdx.x; i < 64 * DH; i += blockDim.x) {
      const int r = i / DH, e = i % DH;
      const bf16 v = (r < nvalid && e < dh) ? base[static_cast<int64_t>(r) * stride + e] : __float2bfloat16(0.f);
      s[sw<DH>(r, e >> 3) + (e & 7)] = v;
    }
  }
}

// A fragment (16 rows x 16 k) of a row-major swizzled tile at rows r0.
template <int DH>
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], const bf16* s, int r0, int ks, int lane) {
  ldsm4(a, s + sw<DH>(r0 + (lane & 15), 2 * ks + (lane >> 4)));
}
// B fragments for two 8-column n-tiles (rows n0..n0+15 of a [n][k] tile), k-step ks.
template <int DH>
__device__ __forceinline__ void frag_b(uint32_t (&b)[4], const bf16* s, int n0, int ks, int lane) {
  ldsm4(b, s + sw<DH>(n0 + ((lane >> 4) << 3) + (lane & 7), 2 * ks + ((lane >> 3) & 1)));
}
// B fragments from a [k][n] tile (transposed access): k rows k0..k0+15,
// n-chunks 2*np, 2*np+1.
template <int DH>
__device__ __forceinline__ void frag_bt(uint32_t (&b)[4], const bf16* s, int k0, int np, int lane) {
  ldsm4t(b, s + sw<DH>(k0 + (((lane >> 3) & 1) << 3) + (lane & 7), 2 * np + (lane >> 4)));
}

__device__ __forceinline__ bool vec_ok(const AttnParams& p) {
  return (p.dh % 8) == 0 && (p.q_stride % 8) == 0 && (p.kv_stride % 8) == 0 && (p.dout_stride % 8) == 0;
}

// ----------------------------------------------------------------- forward
template <int DH>
__global__ void __launch_bounds__(128) attn_fwd_kernel(AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sQ = reinterpret_cast<bf16*>(smem);
  bf16* sK = sQ + 64 * DH;
  bf16* sV = sK + 2 * 64 * DH;
  const AttnTile tl = p.tiles[blockIdx.x];
  const AttnSeg sg = p.segs[tl.seg];
  const int h = blockIdx.y, g = h / (p.H / p.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool vec = vec_ok(p);

  load_tile<DH>(sQ, p.q + static_cast<int64_t>(sg.q_start + tl.first) * p.q_stride + h * p.dh, p.q_stride, tl.count,
                p.dh, vec, p.q);
  const int kv_len = sg.prefix + tl.first + tl.count;
  const int nkt = (kv_len + 63) / 64;
  const bf16* kb = p.k + static_cast<int64_t>(sg.kv_row0) * p.kv_stride + g * p.dh;
  const bf16* vb = p.v + static_cast<int64_t>(sg.kv_row0) * p.kv_stride + g * p.dh;
  load_tile<DH>(sK, kb, p.kv_stride, min(64, kv_len), p.dh, vec, p.k);
  load_tile<DH>(sV, vb, p.kv_stride, min(64, kv_len), p.dh, vec, p.v);
  cp_commit();

  const int qi0 = tl.first + warp * 16 + (lane >> 2);
  const int lim0 = sg.prefix + min(qi0, sg.len - 1);
  const int lim1 = sg.prefix + min(qi0 + 8, sg.len - 1);
  const float sl2 = p.scale * kLog2e;
  float m0 = -FLT_MAX, m1 = -FLT_MAX, l0 = 0.f, l1 = 0.f;
  float o[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

  for (int kt = 0; kt < nkt; ++kt) {
    if (kt + 1 < nkt) {
      const int b = (kt + 1) & 1;
      const int r0 = (kt + 1) * 64;
      load_tile<DH>(sK + b * 64 * DH, kb + static_cast<int64_t>(r0) * p.kv_stride, p.kv_stride, min(64, kv_len - r0),
                    p.dh, vec, p.k);
      load_tile<DH>(sV + b * 64 * DH, vb + static_cast<int64_t>(r0) * p.kv_stride, p.kv_stride, min(64, kv_len - r0),
                    p.dh, vec, p.v);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* K_ = sK + (kt & 1) * 64 * DH;
    const bf16* V_ = sV + (kt & 1) * 64 * DH;
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      uint32_t a[4];
      frag_a<DH>(a, sQ, warp * 16, ks, lane);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b[4];
        frag_b<DH>(b, K_, np * 16, ks, lane);
        mma16816(s[2 * np], a, b[0], b[1]);
        mma16816(s[2 * np + 1], a, b[2], b[3]);
      }
    }
    const int key0 = kt * 64 + 2 * (lane & 3);
    float mx0 = -FLT_MAX, mx1 = -FLT_MAX;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = key0 + 8 * j + e;
        s[j][e] = key <= lim0 ? s[j][e] * sl2 : -FLT_MAX;
        s[j][2 + e] = key <= lim1 ? s[j][2 + e] * sl2 : -FLT_MAX;
        mx0 = fmaxf(mx0, s[j][e]);
        mx1 = fmaxf(mx1, s[j][2 + e]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float a0 = exp2f(m0 - mn0), a1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    float r0 = 0.f, r1 = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        s[j][e] = s[j][e] == -FLT_MAX ? 0.f : exp2f(s[j][e] - mn0);
        s[j][2 + e] = s[j][2 + e] == -FLT_MAX ? 0.f : exp2f(s[j][2 + e] - mn1);
        r0 += s[j][e];
        r1 += s[j][2 + e];
      }
    }
    l0 = l0 * a0 + r0;
    l1 = l1 * a1 + r1;
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
      o[j][0] *= a0;
      o[j][1] *= a0;
      o[j][2] *= a1;
      o[j][3] *= a1;
    }
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      uint32_t a[4] = {pack_bf16(s[2 * k2][0], s[2 * k2][1]), pack_bf16(s[2 * k2][2], s[2 * k2][3]),
                       pack_bf16(s[2 * k2 + 1][0], s[2 * k2 + 1][1]), pack_bf16(s[2 * k2 + 1][2], s[2 * k2 + 1][3])};
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        uint32_t b[4];
        frag_bt<DH>(b, V_, k2 * 16, np, lane);
        mma16816(o[2 * np], a, b[0], b[1]);
        mma16816(o[2 * np + 1], a, b[2], b[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int qi = qi0 + 8 * half;
    if (qi - tl.first >= tl.count || qi >= sg.len) continue;
    const int row = sg.q_start + qi;
    const float inv = half ? i1 : i0;
    bf16* orow = p.o + static_cast<int64_t>(row) * p.o_stride + h * p.dh;
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
      const int c = 8 * j + 2 * (lane & 3);
      if (c < p.dh) orow[c] = __float2bfloat16_rn(o[j][2 * half] * inv);
      if (c + 1 < p.dh) orow[c + 1] = __float2bfloat16_rn(o[j][2 * half + 1] * inv);
    }
    if ((lane & 3) == 0) p.lse[static_cast<int64_t>(h) * p.T + row] = ((half ? m1 : m0) + log2f(half ? l1 : l0)) * kLn2;
  }
}

// ------------------------------------------------------------- dsum (D)
__global__ void attn_dsum_kernel(AttnParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p.T * p.H) return;
  const int t = warp / p.H, h = warp % p.H;
  const bf16* a = p.dout + static_cast<int64_t>(t) * p.dout_stride + h * p.dh;
  const bf16* b = p.o + static_cast<int64_t>(t) * p.o_stride + h * p.dh;
  float s = 0.f;
  for (int c = lane; c < p.dh; c += 32) s += __bfloat162float(a[c]) * __bfloat162float(b[c]);
  s = warp_sum(s);
  if (lane == 0) p.dsum[static_cast<int64_t>(h) * p.T + t] = s;
}

// ------------------------------------------------------------------ dQ
template <int DH>
__global__ void __launch_bounds__(128) attn_dq_kernel(AttnParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sQ = reinterpret_cast<bf16*>(smem);
  bf16* sO = sQ + 64 * DH;  // dO
  bf16* sK = sO + 64 * DH;
  bf16* sV = sK + 2 * 64 * DH;
  const AttnTile tl = p.tiles[blockIdx.x];
  const AttnSeg sg = p.segs[tl.seg];
  const int h = blockIdx.y, g = h / (p.H / p.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool vec = vec_ok(p);
  const int64_t row0 = sg.q_start + tl.first;
  load_tile<DH>(sQ, p.q + row0 * p.q_stride + h * p.dh, p.q_stride, tl.count, p.dh, vec, p.q);
  load_tile<DH>(sO, p.dout + row0 * p.dout_stride + h * p.dh, p.dout_stride, tl.count, p.dh, vec, p.dout);
  const int kv_len = sg.prefix + tl.first + tl.count;
  const int nkt = (kv_len + 63) / 64;
  const bf16* kb = p.k + static_cast<int64_t>(sg.kv_row0) * p.kv_stride + g * p.dh;
  const bf16* vb = p.v + static_cast<int64_t>(sg.kv_row0) * p.kv_stride + g * p.dh;
  load_tile<DH>(sK, kb, p.kv_stride, min(64, kv_len), p.dh, vec, p.k);
  load_tile<DH>(sV, vb, p.kv_stride, min(64, kv_len), p.dh, vec, p.v);
  cp_commit();

  const int qi0 = tl.first + warp * 16 + (lane >> 2);
  const bool ok0 = qi0 < sg.len && qi0 - tl.first < tl.count;
  const bool ok1 = qi0 + 8 < sg.len && qi0 + 8 - tl.first < tl.count;
  const int lim0 = sg.prefix + min(qi0, sg.len - 1);
  const int lim1 = sg.prefix + min(qi0 + 8, sg.len - 1);
  const float sl2 = p.scale * kLog2e;
  const float lse0 = ok0 ? p.lse[static_cast<int64_t>(h) * p.T + sg.q_start + qi0] * kLog2e : 0.f;
  const float lse1 = ok1 ? p.lse[static_cast<int64_t>(h) * p.T + sg.q_start + qi0 + 8] * kLog2e : 0.f;
  const float D0 = ok0 ? p.dsum[static_cast<int64_t>(h) * p.T + sg.q_start + qi0] : 0.f;
  const float D1 = ok1 ? p.dsum[static_cast<int64_t>(h) * p.T + sg.q_start + qi0 + 8] : 0.f;
  float dq[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;

  for (int kt = 0; kt < nkt; ++kt) {
    if (kt + 1 < nkt) {
      const int b = (kt + 1) & 1;
      const int r0 = (kt + 1) * 64;
      load_tile<DH>(sK + b * 64 * DH, kb + static_cast<int64_t>(r0) * p.kv_stride, p.kv_stride, min(64, kv_len - r0),
                    p.dh, vec, p.k);
      load_tile<DH>(sV + b * 64 * DH, vb + static_cast<int64_t>(r0) * p.kv_stride, p.kv_stride, min(64, kv_len - r0),
                    p.dh, vec, p.v);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const bf16* K_ = sK + (kt & 1) * 64 * DH;
    const bf16* V_ = sV + (kt & 1) * 64 * DH;
    float s[8][4], dp[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
    }
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      uint32_t a[4], ad[4];
      frag_a<DH>(a, sQ, warp * 16, ks, lane);
      frag_a<DH>(ad, sO, warp * 16, ks, lane);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b[4];
        frag_b<DH>(b, K_, np * 16, ks, lane);
        mma16816(s[2 * np], a, b[0], b[1]);
        mma16816(s[2 * np + 1], a, b[2], b[3]);
        frag_b<DH>(b, V_, np * 16, ks, lane);
        mma16816(dp[2 * np], ad, b[0], b[1]);
        mma16816(dp[2 * np + 1], ad, b[2], b[3]);
      }
    }
    const int key0 = kt * 64 + 2 * (lane & 3);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = key0 + 8 * j + e;
        const float p0 = (ok0 && key <= lim0) ? exp2f(s[j][e] * sl2 - lse0) : 0.f;
        const float p1 = (ok1 && key <= lim1) ? exp2f(s[j][2 + e] * sl2 - lse1) : 0.f;
        s[j][e] = p0 * (dp[j][e] - D0);
        s[j][2 + e] = p1 * (dp[j][2 + e] - D1);
      }
    }
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      uint32_t a[4] = {pack_bf16(s[2 * k2][0], s[2 * k2][1]), pack_bf16(s[2 * k2][2], s[2 * k2][3]),
                       pack_bf16(s[2 * k2 + 1][0], s[2 * k2 + 1][1]), pack_bf16(s[2 * k2 + 1][2], s[2 * k2 + 1][3])};
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        uint32_t b[4];
        frag_bt<DH>(b, K_, k2 * 16, np, lane);
        mma16816(dq[2 * np], a, b[0], b[1]);
        mma16816(dq[2 * np + 1], a, b[2], b[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    if (!(half ? ok1 : ok0)) continue;
    const int row = sg.q_start + qi0 + 8 * half;
    bf16* out = p.dq + static_cast<int64_t>(row) * p.dq_stride + h * p.dh;
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
      const int c = 8 * j + 2 * (lane & 3);
      if (c < p.dh) out[c] = __float2bfloat16_rn(dq[j][2 * half] * p.scale);
      if (c + 1 < p.dh) out[c + 1] = __float2bfloat16_rn(dq[j][2 * half + 1] * p.scale);
    }
  }
}

// ------------------------------------------------------------- dK / dV
template <int DH>
__global__ void __launch_bounds__(128) attn_dkv_kernel(AttnParams p, const AttnTile* key_tiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* sK = reinterpret_cast<bf16*>(smem);
  bf16* sV = sK + 64 * DH;
  bf16* sQ = sV + 64 * DH;          // [2][64*DH]
  bf16* sO = sQ + 2 * 64 * DH;      // [2][64*DH] dO
  float* sL = reinterpret_cast<float*>(sO + 2 * 64 * DH);  // [2][64] lse*log2e
  float* sD = sL + 128;                                   // [2][64]
  const AttnTile tl = key_tiles[blockIdx.x];
  const AttnSeg sg = p.segs[tl.seg];
  const int g = blockIdx.y, per = p.H / p.KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool vec = vec_ok(p);
  const int key_first = tl.first;  // key index within [0, prefix+len)
  const int kv_len = sg.prefix + sg.len;
  load_tile<DH>(sK, p.k + static_cast<int64_t>(sg.kv_row0 + key_first) * p.kv_stride + g * p.dh, p.kv_stride,
                tl.count, p.dh, vec, p.k);
  load_tile<DH>(sV, p.v + static_cast<int64_t>(sg.kv_row0 + key_first) * p.kv_stride + g * p.dh, p.kv_stride,
                tl.count, p.dh, vec, p.v);

  const int i0 = max(0, key_first - sg.prefix);  // first query that sees any key here
  const int nqt = (sg.len - i0 + 63) / 64;
  const int iters = per * nqt;
  auto load_q = [&](int it, int b) {
    const int hq = g * per + it / nqt;
    const int q0 = i0 + (it % nqt) * 64;
    const int nq = min(64, sg.len - q0);
    const int64_t row0 = sg.q_start + q0;
    load_tile<DH>(sQ + b * 64 * DH, p.q + row0 * p.q_stride + hq * p.dh, p.q_stride, nq, p.dh, vec, p.q);
    load_tile<DH>(sO + b * 64 * DH, p.dout + row0 * p.dout_stride + hq * p.dh, p.dout_stride, nq, p.dh, vec, p.dout);
    for (int r = threadIdx.x; r < 64; r += blockDim.x) {
      const bool ok = r < nq;
      sL[b * 64 + r] = ok ? p.lse[static_cast<int64_t>(hq) * p.T + row0 + r] * kLog2e : 0.f;
      sD[b * 64 + r] = ok ? p.dsum[static_cast<int64_t>(hq) * p.T + row0 + r] : 0.f;
    }
  };
  if (iters > 0) load_q(0, 0);
  cp_commit();

  const int k_lo = key_first + warp * 16 + (lane >> 2);  // this thread's key rows k_lo, k_lo + 8
  const float sl2 = p.scale * kLog2e;
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) {
    dk[j][0] = dk[j][1] = dk[j][2] = dk[j][3] = 0.f;
    dv[j][0] = dv[j][1] = dv[j][2] = dv[j][3] = 0.f;
  }
  for (int it = 0; it < iters; ++it) {
    if (it + 1 < iters) {
      load_q(it + 1, (it + 1) & 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int b = it & 1;
    const bf16* Q_ = sQ + b * 64 * DH;
    const bf16* O_ = sO + b * 64 * DH;
    const float* L_ = sL + b * 64;
    const float* D_ = sD + b * 64;
    const int q0 = i0 + (it % nqt) * 64;
    float s[8][4], dp[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
      dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
    }
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      uint32_t ak[4], av[4];
      frag_a<DH>(ak, sK, warp * 16, ks, lane);
      frag_a<DH>(av, sV, warp * 16, ks, lane);
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t bq[4];
        frag_b<DH>(bq, Q_, np * 16, ks, lane);
        mma16816(s[2 * np], ak, bq[0], bq[1]);
        mma16816(s[2 * np + 1], ak, bq[2], bq[3]);
        frag_b<DH>(bq, O_, np * 16, ks, lane);
        mma16816(dp[2 * np], av, bq[0], bq[1]);
        mma16816(dp[2 * np + 1], av, bq[2], bq[3]);
      }
    }
    // s -> P^T, dp -> dS^T (rows = keys k_lo / k_lo+8, cols = queries)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int ql = 8 * j + 2 * (lane & 3) + e;  // query within tile
        const int qi = q0 + ql;
        const bool qok = qi < sg.len;
        const bool v0 = qok && k_lo < kv_len && k_lo <= sg.prefix + qi;
        const bool v1 = qok && k_lo + 8 < kv_len && k_lo + 8 <= sg.prefix + qi;
        const float p0 = v0 ? exp2f(s[j][e] * sl2 - L_[ql]) : 0.f;
        const float p1 = v1 ? exp2f(s[j][2 + e] * sl2 - L_[ql]) : 0.f;
        s[j][e] = p0;
        s[j][2 + e] = p1;
        dp[j][e] = p0 * (dp[j][e] - D_[ql]);
        dp[j][2 + e] = p1 * (dp[j][2 + e] - D_[ql]);
      }
    }
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      uint32_t ap[4] = {pack_bf16(s[2 * k2][0], s[2 * k2][1]), pack_bf16(s[2 * k2][2], s[2 * k2][3]),
                        pack_bf16(s[2 * k2 + 1][0], s[2 * k2 + 1][1]), pack_bf16(s[2 * k2 + 1][2], s[2 * k2 + 1][3])};
      uint32_t as[4] = {pack_bf16(dp[2 * k2][0], dp[2 * k2][1]), pack_bf16(dp[2 * k2][2], dp[2 * k2][3]),
                        pack_bf16(dp[2 * k2 + 1][0], dp[2 * k2 + 1][1]),
                        pack_bf16(dp[2 * k2 + 1][2], dp[2 * k2 + 1][3])};
#pragma unroll
      for (int np = 0; np < DH / 16; ++np) {
        uint32_t b[4];
        frag_bt<DH>(b, O_, k2 * 16, np, lane);
        mma16816(dv[2 * np], ap, b[0], b[1]);
        mma16816(dv[2 * np + 1], ap, b[2], b[3]);
        frag_bt<DH>(b, Q_, k2 * 16, np, lane);
        mma16816(dk[2 * np], as, b[0], b[1]);
        mma16816(dk[2 * np + 1], as, b[2], b[3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int key = k_lo + 8 * half;
    if (key >= kv_len || key - key_first >= tl.count) continue;
    const int64_t row = sg.kv_row0 + key;
    float* dkr = p.dk_acc + row * p.acc_stride + g * p.dh;
    float* dvr = p.dv_acc + row * p.acc_stride + g * p.dh;
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * j + 2 * (lane & 3) + e;
        if (c < p.dh) {
          dkr[c] += dk[j][2 * half + e] * p.scale;
          dvr[c] += dv[j][2 * half + e];
        }
      }
    }
  }
}

template <int DH>
cudaError_t fwd_t(const AttnParams& p, cudaStream_t st) {
  const size_t smem = 5 * 64 * DH * sizeof(bf16);
  // per (kernel, device), thread-safe
  cudaError_t attr = cudaSuccess;
  if (attr == cudaSuccess) attr = smem_optin(reinterpret_cast<const void*>(attn_fwd_kernel<DH>), static_cast<int>(smem));
  if (attr != cudaSuccess) return attr;
  attn_fwd_kernel<DH><<<dim3(p.num_tiles, p.H), 128, smem, st>>>(p);
  return cudaGetLastError();
}

template <int DH>
cudaError_t bwd_t(const AttnParams& p, const AttnTile* key_tiles, int32_t nkt, cudaStream_t st) {
  const size_t smem_dq = 6 * 64 * DH * sizeof(bf16);
  const size_t smem_dkv = 6 * 64 * DH * sizeof(bf16) + 4 * 64 * sizeof(float);
  // per (kernel, device), thread-safe
  cudaError_t attr = cudaSuccess;
  if (attr == cudaSuccess) attr = smem_optin(reinterpret_cast<const void*>(attn_dq_kernel<DH>), static_cast<int>(smem_dq));
  if (attr == cudaSuccess) attr = smem_optin(reinterpret_cast<const void*>(attn_dkv_kernel<DH>), static_cast<int>(smem_dkv));
  if (attr != cudaSuccess) return attr;
  const int64_t warps = static_cast<int64_t>(p.T) * p.H;
  attn_dsum_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(p);
  attn_dq_kernel<DH><<<dim3(p.num_tiles, p.H), 128, smem_dq, st>>>(p);
  if (nkt > 0) attn_dkv_kernel<DH><<<dim3(nkt, p.KVH), 128, smem_dkv, st>>>(p, key_tiles);
  return cudaGetLastError();
}

}  // namespace

cudaError_t attn_forward(const AttnParams& p, cudaStream_t st) {
  if (p.num_tiles == 0) return cudaSuccess;
  if (p.dh <= 64) return fwd_t<64>(p, st);
  if (p.dh <= 128) return fwd_t<128>(p, st);
  return cudaErrorInvalidValue;
}

cudaError_t attn_dsum(const AttnParams& p, cudaStream_t st) {
  const int64_t warps = static_cast<int64_t>(p.T) * p.H;
  attn_dsum_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t attn_backward(const AttnParams& p, const AttnTile* key_tiles, int32_t nkt, cudaStream_t st) {
  if (p.num_tiles == 0) return cudaSuccess;
  if (p.dh <= 64) return bwd_t<64>(p, key_tiles, nkt, st);
  if (p.dh <= 128) return bwd_t<128>(p, key_tiles, nkt, st);
  return cudaErrorInvalidValue;
}

}  // namespace cfk
