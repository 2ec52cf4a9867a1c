// Bandwidth-bound kernels (see ops.h): coalesced, vectorised where the row
// pitch allows, warp-shuffle reductions, and fixed reduction orders so every
// result is bitwise reproducible run to run (needed for the reference's
// recompute-loss check, plan_runner.hpp:232-241).
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "ops.h"

namespace cfk {
namespace {

constexpr int kThreads = 256;

inline unsigned blocks_for(int64_t n, int per = kThreads) {
  int64_t b = (n + per - 1) / per;
  if (b > 148 * 64) b = 148 * 64;
  return static_cast<unsigned>(b < 1 ? 1 : b);
}

__global__ void init_uniform_kernel(bf16* dst, int64_t ld, int64_t rows, int64_t cols, uint64_t base, uint64_t seed,
                                    double scale) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // state after (base + i + 1) increments of the golden gamma
    uint64_t z = seed + (base + static_cast<uint64_t>(i) + 1ull) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
    const int64_t r = i / cols, c = i % cols;
    dst[r * ld + c] = __double2bfloat16((u * 2.0 - 1.0) * scale);
  }
}

__global__ void fill_kernel(float* d, int64_t n, float v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d[i] = v;
}

// One warp per row.
__global__ void embed_kernel(const int32_t* tok, const bf16* E, int64_t d, int64_t T, float* x) {
  const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const bf16* e = E + static_cast<int64_t>(tok[row]) * d;
  float* o = x + row * d;
  if ((d & 7) == 0) {
    for (int64_t c = lane * 8; c < d; c += 256) {
      const uint4 v = *reinterpret_cast<const uint4*>(e + c);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
      float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]), f2 = __bfloat1622float2(h[2]),
             f3 = __bfloat1622float2(h[3]);
      *reinterpret_cast<float4*>(o + c) = make_float4(f0.x, f0.y, f1.x, f1.y);
      *reinterpret_cast<float4*>(o + c + 4) = make_float4(f2.x, f2.y, f3.x, f3.y);
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) o[c] = __bfloat162float(e[c]);
  }
}

__global__ void rmsnorm_fwd_kernel(const float* x, const float* gain, int64_t T, int64_t d, float eps, bf16* y) {
  const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const float* xr = x + row * d;
  bf16* yr = y + row * d;
  float ss = 0.f;
  const bool vec = (d & 3) == 0;
  if (vec) {
    for (int64_t c = lane * 4; c < d; c += 128) {
      const float4 v = *reinterpret_cast<const float4*>(xr + c);
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) ss += xr[c] * xr[c];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / static_cast<float>(d) + eps);
  if (vec) {
    for (int64_t c = lane * 4; c < d; c += 128) {
      const float4 v = *reinterpret_cast<const float4*>(xr + c);
      const float4 g = *reinterpret_cast<const float4*>(gain + c);
      uint2 o;
      o.x = pack_bf16(v.x * r * g.x, v.y * r * g.y);
      o.y = pack_bf16(v.z * r * g.z, v.w * r * g.w);
      *reinterpret_cast<uint2*>(yr + c) = o;
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) yr[c] = __float2bfloat16_rn(xr[c] * r * gain[c]);
  }
}

__global__ void to_bf16_kernel(const float* x, bf16* y, int64_t n) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    uint2 o;
    o.x = pack_bf16(v.x, v.y);
    o.y = pack_bf16(v.z, v.w);
    reinterpret_cast<uint2*>(y)[i] = o;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

__global__ void rope_table_kernel(const int32_t* pos, int64_t T, int half, int dh, double theta, float2* tab) {
  const int64_t n = T * half;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / half;
    const int j = static_cast<int>(i % half);
    const double f = pow(theta, -2.0 * static_cast<double>(j) / static_cast<double>(dh));
    double s, c;
    sincos(static_cast<double>(pos[t]) * f, &s, &c);
    tab[i] = make_float2(static_cast<float>(c), static_cast<float>(s));
  }
}

// grid-stride over (t, head, j) with j < half; heads [0,H) are q, [H, H+KVH) are k.
__global__ void rope_qk_kernel(bf16* qkv, int64_t ld, int64_t T, int H, int KVH, int dh, int64_t col_k,
                               const float2* tab, int inverse_q_only) {
  const int half = dh / 2;
  const int heads = inverse_q_only ? H : H + KVH;
  const int64_t n = T * heads * half;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i % half);
    const int64_t th = i / half;
    const int hh = static_cast<int>(th % heads);
    const int64_t t = th / heads;
    bf16* p = qkv + t * ld + (hh < H ? static_cast<int64_t>(hh) * dh : col_k + static_cast<int64_t>(hh - H) * dh);
    const float2 cs = tab[t * half + j];
    const float sn = inverse_q_only ? -cs.y : cs.y;
    const float x0 = __bfloat162float(p[j]), x1 = __bfloat162float(p[j + half]);
    p[j] = __float2bfloat16_rn(x0 * cs.x - x1 * sn);
    p[j + half] = __float2bfloat16_rn(x1 * cs.x + x0 * sn);
  }
}

__global__ void kv_store_kernel(const bf16* qkv, int64_t ld, int64_t T, int64_t kvw, int64_t col_k, int64_t col_v,
                                bf16* kc, bf16* vc, int64_t cache_ld) {
  const int64_t n = T * kvw;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / kvw, c = i % kvw;
    kc[t * cache_ld + c] = qkv[t * ld + col_k + c];
    vc[t * cache_ld + c] = qkv[t * ld + col_v + c];
  }
}


// 8 elements (16 bytes) per thread; ffn % 8 == 0 is validated at model creation.
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 p = __bfloat1622float2(h[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}

__global__ void swiglu_fwd_kernel(const bf16* gu, int64_t T, int64_t ffn, bf16* h) {
  const int64_t f8 = ffn / 8, n = T * f8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / f8, j = (i % f8) * 8;
    float g[8], u[8], o[8];
    unpack8(*reinterpret_cast<const uint4*>(gu + t * 2 * ffn + j), g);
    unpack8(*reinterpret_cast<const uint4*>(gu + t * 2 * ffn + ffn + j), u);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = g[e] * sigmoidf_(g[e]) * u[e];
    *reinterpret_cast<uint4*>(h + t * ffn + j) = pack8(o);
  }
}

__global__ void swiglu_bwd_kernel(const bf16* gu, const bf16* dh, int64_t T, int64_t ffn, bf16* dgu) {
  const int64_t f8 = ffn / 8, n = T * f8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / f8, j = (i % f8) * 8;
    float g[8], u[8], d[8], og[8], ou[8];
    unpack8(*reinterpret_cast<const uint4*>(gu + t * 2 * ffn + j), g);
    unpack8(*reinterpret_cast<const uint4*>(gu + t * 2 * ffn + ffn + j), u);
    unpack8(*reinterpret_cast<const uint4*>(dh + t * ffn + j), d);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float s = sigmoidf_(g[e]);
      og[e] = d[e] * u[e] * s * (1.f + g[e] * (1.f - s));
      ou[e] = d[e] * g[e] * s;
    }
    *reinterpret_cast<uint4*>(dgu + t * 2 * ffn + j) = pack8(og);
    *reinterpret_cast<uint4*>(dgu + t * 2 * ffn + ffn + j) = pack8(ou);
  }
}

// Row-resident RMSNorm: one 128-thread CTA per row, the row held in
// registers (NV float4 per thread, d <= NV*512), so x is read exactly once;
// block reduction through 4 warp partials (every thread sums them in the
// same order -> deterministic).
constexpr int kRowThreads = 128;
template <int NV>
__global__ __launch_bounds__(kRowThreads) void rmsnorm_row_kernel(const float* __restrict__ x,
                                                                   const float* __restrict__ gain, int d, float eps,
                                                                   bf16* __restrict__ y) {
  __shared__ float red[kRowThreads / 32];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * d;
  float4 v[NV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (threadIdx.x + i * kRowThreads) * 4;
    v[i] = c < d ? __ldcs(reinterpret_cast<const float4*>(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  ss = red[0] + red[1] + red[2] + red[3];
  const float r = rsqrtf(ss / static_cast<float>(d) + eps);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (threadIdx.x + i * kRowThreads) * 4;
    if (c < d) {
      const float4 g = *reinterpret_cast<const float4*>(gain + c);
      uint2 o;
      o.x = pack_bf16(v[i].x * r * g.x, v[i].y * r * g.y);
      o.y = pack_bf16(v[i].z * r * g.z, v[i].w * r * g.w);
      *reinterpret_cast<uint2*>(y + row * d + c) = o;
    }
  }
}

// Fused RMSNorm backward + gain gradient (+ bf16 copy of the result): a CTA
// owns a contiguous row range, holds its columns of the gain and of the
// gain-gradient partial in registers, and streams x / dy / dres once.
//   dx = dres + r*dy*g - x*r^3*<dy*g, x>/d,   part[cta][c] = sum_rows dy*x*r
constexpr int kBwdThreads = 256;
template <int NV>
__global__ __launch_bounds__(kBwdThreads) void rmsnorm_bwd_rows_kernel(
    const float* __restrict__ x, const float* __restrict__ gain, const float* __restrict__ dy, const float* dres,
    int64_t T, int d, float eps, int64_t rows_per_cta, float* dx, bf16* __restrict__ dx_bf16,
    float* __restrict__ part) {
  constexpr int W = kBwdThreads / 32;
  __shared__ float red[2][2][W];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 g[NV], acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (threadIdx.x + i * kBwdThreads) * 4;
    g[i] = c < d ? *reinterpret_cast<const float4*>(gain + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int64_t r0 = blockIdx.x * rows_per_cta, r1 = min(T, r0 + rows_per_cta);
  for (int64_t row = r0; row < r1; ++row) {
    const int par = static_cast<int>(row & 1);
    const float* xr = x + row * d;
    const float* gr = dy + row * d;
    float4 xv[NV], gv[NV], rv[NV];
    float ss = 0.f, dot = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (threadIdx.x + i * kBwdThreads) * 4;
      const bool in = c < d;
      xv[i] = in ? *reinterpret_cast<const float4*>(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      gv[i] = in ? __ldcs(reinterpret_cast<const float4*>(gr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      rv[i] = (in && dres) ? *reinterpret_cast<const float4*>(dres + row * d + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      ss += xv[i].x * xv[i].x + xv[i].y * xv[i].y + xv[i].z * xv[i].z + xv[i].w * xv[i].w;
      dot += gv[i].x * g[i].x * xv[i].x + gv[i].y * g[i].y * xv[i].y + gv[i].z * g[i].z * xv[i].z +
             gv[i].w * g[i].w * xv[i].w;
    }
    ss = warp_sum(ss);
    dot = warp_sum(dot);
    if (lane == 0) {
      red[par][0][w] = ss;
      red[par][1][w] = dot;
    }
    __syncthreads();
    ss = 0.f;
    dot = 0.f;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      ss += red[par][0][i];
      dot += red[par][1][i];
    }
    const float r = rsqrtf(ss / static_cast<float>(d) + eps);
    const float k = r * r * r * dot / static_cast<float>(d);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (threadIdx.x + i * kBwdThreads) * 4;
      if (c >= d) continue;
      float4 o = rv[i];
      o.x += r * gv[i].x * g[i].x - xv[i].x * k;
      o.y += r * gv[i].y * g[i].y - xv[i].y * k;
      o.z += r * gv[i].z * g[i].z - xv[i].z * k;
      o.w += r * gv[i].w * g[i].w - xv[i].w * k;
      __stcs(reinterpret_cast<float4*>(dx + row * d + c), o);
      if (dx_bf16) {
        uint2 b;
        b.x = pack_bf16(o.x, o.y);
        b.y = pack_bf16(o.z, o.w);
        *reinterpret_cast<uint2*>(dx_bf16 + row * d + c) = b;
      }
      acc[i].x += gv[i].x * xv[i].x * r;
      acc[i].y += gv[i].y * xv[i].y * r;
      acc[i].z += gv[i].z * xv[i].z * r;
      acc[i].w += gv[i].w * xv[i].w * r;
    }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (threadIdx.x + i * kBwdThreads) * 4;
    if (c < d) *reinterpret_cast<float4*>(part + blockIdx.x * static_cast<int64_t>(d) + c) = acc[i];
  }
}

// Column sums of the per-CTA gain partials, fixed order: block = 32
// columns x 8 row-groups (strided rows), then the 8 group sums in order.
__global__ void gain_reduce_cols_kernel(const float* __restrict__ part, int parts, int64_t d,
                                        float* __restrict__ dgain) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < d)
    for (int i = grp; i < parts; i += 8) s += part[i * d + c];
  red[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && c < d) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][lane];
    dgain[c] += t;
  }
}

// RoPE rotate-half, 8 consecutive frequency pairs per thread (16-byte loads
// of both halves); heads [0,H) are q, [H, H+KVH) are k.
__global__ void rope_qk_vec_kernel(bf16* qkv, int64_t ld, int64_t T, int H, int KVH, int dh, int64_t col_k,
                                   const float2* __restrict__ tab, int inverse_q_only) {
  const int half = dh / 2, g8 = half / 8;
  const int heads = inverse_q_only ? H : H + KVH;
  const int64_t n = T * heads * g8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i % g8) * 8;
    const int64_t th = i / g8;
    const int hh = static_cast<int>(th % heads);
    const int64_t t = th / heads;
    bf16* p = qkv + t * ld + (hh < H ? static_cast<int64_t>(hh) * dh : col_k + static_cast<int64_t>(hh - H) * dh);
    float a[8], b[8], oa[8], ob[8];
    unpack8(*reinterpret_cast<const uint4*>(p + j), a);
    unpack8(*reinterpret_cast<const uint4*>(p + j + half), b);
    const float4* tp = reinterpret_cast<const float4*>(tab + t * half + j);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 cs = tp[e];  // (cos, sin) of pairs j+2e, j+2e+1
      const float s0 = inverse_q_only ? -cs.y : cs.y, s1 = inverse_q_only ? -cs.w : cs.w;
      oa[2 * e] = a[2 * e] * cs.x - b[2 * e] * s0;
      ob[2 * e] = b[2 * e] * cs.x + a[2 * e] * s0;
      oa[2 * e + 1] = a[2 * e + 1] * cs.z - b[2 * e + 1] * s1;
      ob[2 * e + 1] = b[2 * e + 1] * cs.z + a[2 * e + 1] * s1;
    }
    *reinterpret_cast<uint4*>(p + j) = pack8(oa);
    *reinterpret_cast<uint4*>(p + j + half) = pack8(ob);
  }
}

// One 256-thread block per row.
__global__ void ce_kernel(const float* logits, int64_t V, int64_t ld, const int32_t* targets, float inv_norm, float* row_loss,
                          bf16* dlogits) {
  const int64_t row = blockIdx.x;
  const int32_t tgt = targets[row];
  const float* l = logits + row * ld;
  __shared__ float red_m[8], red_s[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (tgt < 0) {
    if (threadIdx.x == 0) row_loss[row] = 0.f;
    if (dlogits)
      for (int64_t c = threadIdx.x; c < V; c += blockDim.x) dlogits[row * ld + c] = __float2bfloat16(0.f);
    return;
  }
  float m = -INFINITY, s = 0.f;
  for (int64_t c = threadIdx.x; c < V; c += blockDim.x) {
    const float x = l[c];
    if (x > m) {
      s = s * __expf(m - x) + 1.f;
      m = x;
    } else {
      s += __expf(x - m);
    }
  }
  // combine (m, s) across the warp then the block
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mm));
    m = mm;
  }
  if (lane == 0) {
    red_m[warp] = m;
    red_s[warp] = s;
  }
  __syncthreads();
  float M = red_m[0];
  for (int w = 1; w < 8; ++w) M = fmaxf(M, red_m[w]);
  float S = 0.f;
  for (int w = 0; w < 8; ++w) S += red_s[w] * __expf(red_m[w] - M);
  const float lse = M + logf(S);
  if (threadIdx.x == 0) row_loss[row] = lse - l[tgt];
  if (dlogits) {
    const float invS = 1.f / S;
    for (int64_t c = threadIdx.x; c < V; c += blockDim.x) {
      const float p = __expf(l[c] - M) * invS - (c == tgt ? 1.f : 0.f);
      dlogits[row * ld + c] = __float2bfloat16_rn(p * inv_norm);
    }
  }
}

// Register-resident form: one 1024-thread block per row holds the whole row
// (NV float4 per thread, V <= 4096*NV), so the logits are read from HBM once
// (the strided kernel above reads them twice) with 16-byte loads and the
// bf16 gradient is written with 8-byte stores.
template <int NV>
__global__ void __launch_bounds__(1024, 1)
    ce_rows_kernel(const float* __restrict__ logits, int64_t V, int64_t ld, const int32_t* __restrict__ targets,
                   float inv_norm, float* __restrict__ row_loss, bf16* __restrict__ dlogits) {
  const int64_t row = blockIdx.x;
  const int32_t tgt = targets[row];
  const float4* l = reinterpret_cast<const float4*>(logits + row * ld);
  const int64_t nv = V / 4;
  __shared__ float red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (tgt < 0) {
    if (threadIdx.x == 0) row_loss[row] = 0.f;
    if (dlogits) {
      uint2* o = reinterpret_cast<uint2*>(dlogits + row * ld);
      for (int64_t c = threadIdx.x; c < nv; c += blockDim.x) o[c] = make_uint2(0u, 0u);
    }
    return;
  }
  float4 x[NV];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int64_t c = threadIdx.x + static_cast<int64_t>(i) * blockDim.x;
    x[i] = c < nv ? l[c] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    m = fmaxf(m, fmaxf(fmaxf(x[i].x, x[i].y), fmaxf(x[i].z, x[i].w)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  float M = red[0];
  for (int w = 1; w < 32; ++w) M = fmaxf(M, red[w]);
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    x[i].x = __expf(x[i].x - M);
    x[i].y = __expf(x[i].y - M);
    x[i].z = __expf(x[i].z - M);
    x[i].w = __expf(x[i].w - M);
    s += (x[i].x + x[i].y) + (x[i].z + x[i].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  float S = 0.f;
  for (int w = 0; w < 32; ++w) S += red[w];
  if (threadIdx.x == 0) row_loss[row] = M + logf(S) - logits[row * ld + tgt];
  if (dlogits) {
    const float scale = inv_norm / S;
    uint2* o = reinterpret_cast<uint2*>(dlogits + row * ld);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t c = threadIdx.x + static_cast<int64_t>(i) * blockDim.x;
      if (c >= nv) break;
      float4 p = make_float4(x[i].x * scale, x[i].y * scale, x[i].z * scale, x[i].w * scale);
      if (tgt >> 2 == c) {
        const int j = tgt & 3;
        if (j == 0) p.x -= inv_norm;
        if (j == 1) p.y -= inv_norm;
        if (j == 2) p.z -= inv_norm;
        if (j == 3) p.w -= inv_norm;
      }
      o[c] = make_uint2(pack_bf16(p.x, p.y), pack_bf16(p.z, p.w));
    }
  }
}

__global__ void sum_f64_kernel(const float* v, int64_t n, double* out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += static_cast<double>(v[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// One warp per row.
__global__ void rmsnorm_bwd_kernel(const float* x, const float* gain, const float* dy, const float* dres, int64_t T,
                                   int64_t d, float eps, float* dx, float* rstd) {
  const int64_t row = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const float* xr = x + row * d;
  const float* gr = dy + row * d;
  float ss = 0.f, dot = 0.f;
  // d % 8 == 0 (validated at model creation): float4 path
  for (int64_t c = lane * 4; c < d; c += 128) {
    const float4 xv = *reinterpret_cast<const float4*>(xr + c);
    const float4 gv = *reinterpret_cast<const float4*>(gr + c);
    const float4 w = *reinterpret_cast<const float4*>(gain + c);
    ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
    dot += gv.x * w.x * xv.x + gv.y * w.y * xv.y + gv.z * w.z * xv.z + gv.w * w.w * xv.w;
  }
  ss = warp_sum(ss);
  dot = warp_sum(dot);
  const float r = rsqrtf(ss / static_cast<float>(d) + eps);
  const float k = r * r * r * dot / static_cast<float>(d);
  for (int64_t c = lane * 4; c < d; c += 128) {
    const float4 xv = *reinterpret_cast<const float4*>(xr + c);
    const float4 gv = *reinterpret_cast<const float4*>(gr + c);
    const float4 w = *reinterpret_cast<const float4*>(gain + c);
    float4 o = dres ? *reinterpret_cast<const float4*>(dres + row * d + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    o.x += r * gv.x * w.x - xv.x * k;
    o.y += r * gv.y * w.y - xv.y * k;
    o.z += r * gv.z * w.z - xv.z * k;
    o.w += r * gv.w * w.w - xv.w * k;
    *reinterpret_cast<float4*>(dx + row * d + c) = o;
  }
  if (lane == 0 && rstd) rstd[row] = r;
}

// Stage 1: block (blockIdx.x: 128 columns, blockIdx.y: a contiguous row
// slice); each thread owns 4 adjacent columns (float4), warps stride rows.
// Partials [gridDim.y][d] are reduced in fixed order by stage 2.
constexpr int kGainSplit = 64;
__global__ void gain_grad_partial_kernel(const float* x, const float* dy, const float* rstd, int64_t T, int64_t d,
                                         float* part) {
  __shared__ float4 red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (blockIdx.x * 32 + lane) * 4;
  const int64_t rows = (T + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = blockIdx.y * rows, r1 = min(T, r0 + rows);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < d)
    for (int64_t t = r0 + w; t < r1; t += 8) {
      const float4 a = *reinterpret_cast<const float4*>(dy + t * d + c);
      const float4 b = *reinterpret_cast<const float4*>(x + t * d + c);
      const float r = rstd[t];
      s.x += a.x * b.x * r;
      s.y += a.y * b.y * r;
      s.z += a.z * b.z * r;
      s.w += a.w * b.w * r;
    }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < d) {
    float4 tot = red[0][lane];
    for (int i = 1; i < 8; ++i) {
      tot.x += red[i][lane].x;
      tot.y += red[i][lane].y;
      tot.z += red[i][lane].z;
      tot.w += red[i][lane].w;
    }
    *reinterpret_cast<float4*>(part + blockIdx.y * d + c) = tot;
  }
}
__global__ void gain_grad_reduce_kernel(const float* part, int splits, int64_t d, float* dgain) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= d) return;
  float s = 0.f;
  for (int i = 0; i < splits; ++i) s += part[i * d + c];
  dgain[c] += s;
}

__global__ void dkv_to_dqkv_kernel(const float* dk, const float* dv, int64_t acc_ld, int64_t T, int KVH, int dh,
                                   const float2* tab, bf16* dqkv, int64_t ld, int64_t col_k, int64_t col_v) {
  const int64_t kvw = static_cast<int64_t>(KVH) * dh;
  const int64_t n = T * kvw;
  const int half = dh / 2;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / kvw, c = i % kvw;
    dqkv[t * ld + col_v + c] = __float2bfloat16_rn(dv[t * acc_ld + c]);
    float val = dk[t * acc_ld + c];
    if (tab) {
      const int j = static_cast<int>(c % dh);
      const int64_t hb = c - j;
      const int jj = j < half ? j : j - half;
      const float2 cs = tab[t * half + jj];
      if (j < half) {  // dx0 = dy0 c + dy1 s
        val = val * cs.x + dk[t * acc_ld + hb + j + half] * cs.y;
      } else {  // dx1 = -dy0 s + dy1 c
        val = val * cs.x - dk[t * acc_ld + hb + jj] * cs.y;
      }
    }
    dqkv[t * ld + col_k + c] = __float2bfloat16_rn(val);
  }
}

// Vector form: 8 consecutive columns of one head-half per thread (two float4
// of dK, of its rotate-half partner and of dV; one 16-byte bf16 store each).
__global__ void dkv_to_dqkv_vec_kernel(const float* __restrict__ dk, const float* __restrict__ dv, int64_t acc_ld,
                                       int64_t T, int KVH, int dh, const float2* __restrict__ tab,
                                       bf16* __restrict__ dqkv, int64_t ld, int64_t col_k, int64_t col_v) {
  const int half = dh / 2, g8 = dh / 8;
  const int64_t n = T * KVH * g8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / (KVH * g8);
    const int64_t c = (i % (KVH * g8)) * 8;  // column within [0, kvw)
    const int j = static_cast<int>(c % dh);
    const float* kr = dk + t * acc_ld + c;
    const float* vr = dv + t * acc_ld + c;
    float kv[8], vv[8], out[8];
    *reinterpret_cast<float4*>(kv) = *reinterpret_cast<const float4*>(kr);
    *reinterpret_cast<float4*>(kv + 4) = *reinterpret_cast<const float4*>(kr + 4);
    *reinterpret_cast<float4*>(vv) = *reinterpret_cast<const float4*>(vr);
    *reinterpret_cast<float4*>(vv + 4) = *reinterpret_cast<const float4*>(vr + 4);
    if (tab) {
      const bool lo = j < half;
      const int jj = lo ? j : j - half;
      float pv[8];
      const float* pr = lo ? kr + half : kr - half;  // rotate-half partner
      *reinterpret_cast<float4*>(pv) = *reinterpret_cast<const float4*>(pr);
      *reinterpret_cast<float4*>(pv + 4) = *reinterpret_cast<const float4*>(pr + 4);
      const float4* tp = reinterpret_cast<const float4*>(tab + t * half + jj);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 cs = tp[e];  // (cos, sin) of pairs jj+2e, jj+2e+1
        // lo: dx0 = dy0 c + dy1 s;  hi: dx1 = dy1 c - dy0 s
        out[2 * e] = lo ? kv[2 * e] * cs.x + pv[2 * e] * cs.y : kv[2 * e] * cs.x - pv[2 * e] * cs.y;
        out[2 * e + 1] =
            lo ? kv[2 * e + 1] * cs.z + pv[2 * e + 1] * cs.w : kv[2 * e + 1] * cs.z - pv[2 * e + 1] * cs.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) out[e] = kv[e];
    }
    *reinterpret_cast<uint4*>(dqkv + t * ld + col_k + c) = pack8(out);
    *reinterpret_cast<uint4*>(dqkv + t * ld + col_v + c) = pack8(vv);
  }
}

__global__ void scale_rows_kernel(float* x, int64_t rows, int64_t cols, int64_t ld, float s) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[(i / cols) * ld + i % cols] *= s;
}

__global__ void embed_bwd_kernel(const float* dx, int64_t d, const int32_t* order, const int32_t* uniq,
                                 const int32_t* off, float* dE) {
  const int u = blockIdx.x;
  const int32_t b = off[u], e = off[u + 1];
  float* dst = dE + static_cast<int64_t>(uniq[u]) * d;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    for (int32_t i = b; i < e; ++i) s += dx[static_cast<int64_t>(order[i]) * d + c];
    dst[c] += s;
  }
}

__global__ void bf16_to_f64_kernel(const bf16* src, int64_t ld, int64_t rows, int64_t cols, double* dst) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<double>(__bfloat162float(src[(i / cols) * ld + i % cols]));
}
__global__ void f64_to_bf16_kernel(const double* src, int64_t rows, int64_t cols, bf16* dst, int64_t ld) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[(i / cols) * ld + i % cols] = __double2bfloat16(src[i]);
}
__global__ void f32_to_f64_kernel(const float* src, int64_t ld, int64_t rows, int64_t cols, double* dst) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<double>(src[(i / cols) * ld + i % cols]);
}
__global__ void f64_to_f32_kernel(const double* src, int64_t rows, int64_t cols, float* dst, int64_t ld) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[(i / cols) * ld + i % cols] = static_cast<float>(src[i]);
}

}  // namespace

cudaError_t init_uniform_bf16(bf16* dst, int64_t ld, int64_t rows, int64_t cols, uint64_t draw_base, uint64_t seed,
                              double scale, cudaStream_t st) {
  init_uniform_kernel<<<blocks_for(rows * cols), kThreads, 0, st>>>(dst, ld, rows, cols, draw_base, seed, scale);
  return cudaGetLastError();
}
cudaError_t fill_f32(float* dst, int64_t n, float v, cudaStream_t st) {
  fill_kernel<<<blocks_for(n), kThreads, 0, st>>>(dst, n, v);
  return cudaGetLastError();
}
cudaError_t embed_fwd(const int32_t* tok, const bf16* E, int64_t d, int64_t T, float* x, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  embed_kernel<<<static_cast<unsigned>((T * 32 + 255) / 256), 256, 0, st>>>(tok, E, d, T, x);
  return cudaGetLastError();
}
template <int MaxNV = 16, class F>
bool dispatch_nv(int64_t d, F&& f) {
  const int64_t nv = (d + 4 * kRowThreads - 1) / (4 * kRowThreads);
  if (nv > MaxNV) return false;
  switch (nv) {
    case 1: f(std::integral_constant<int, 1>()); return true;
    case 2: f(std::integral_constant<int, 2>()); return true;
    case 4: f(std::integral_constant<int, 4>()); return true;
    case 6: f(std::integral_constant<int, 6>()); return true;
    case 8: f(std::integral_constant<int, 8>()); return true;
    case 10: f(std::integral_constant<int, 10>()); return true;
    case 12: f(std::integral_constant<int, 12>()); return true;
    case 16: f(std::integral_constant<int, 16>()); return true;
    default: return false;
  }
}

cudaError_t rmsnorm_fwd(const float* x, const float* gain, int64_t T, int64_t d, float eps, bf16* y,
                        cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  const bool row_kernel = (d % 4) == 0 && dispatch_nv(d, [&](auto nv) {
    rmsnorm_row_kernel<decltype(nv)::value><<<static_cast<unsigned>(T), kRowThreads, 0, st>>>(
        x, gain, static_cast<int>(d), eps, y);
  });
  if (!row_kernel)
    rmsnorm_fwd_kernel<<<static_cast<unsigned>((T * 32 + 255) / 256), 256, 0, st>>>(x, gain, T, d, eps, y);
  return cudaGetLastError();
}
cudaError_t to_bf16(const float* x, bf16* y, int64_t n, cudaStream_t st) {
  to_bf16_kernel<<<blocks_for(n / 4 + 1), kThreads, 0, st>>>(x, y, n);
  return cudaGetLastError();
}
cudaError_t rope_table(const int32_t* pos, int64_t T, int dh, double theta, float2* tab, cudaStream_t st) {
  rope_table_kernel<<<blocks_for(T * (dh / 2)), kThreads, 0, st>>>(pos, T, dh / 2, dh, theta, tab);
  return cudaGetLastError();
}
// 16-byte vector path when the half head width is a multiple of 8 and every
// row / column base is 16-byte aligned.
inline bool rope_vec_ok(const void* p, int64_t ld, int dh, int64_t col_k) {
  return (dh / 2) % 8 == 0 && ld % 8 == 0 && col_k % 8 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}
cudaError_t rope_qk(bf16* qkv, int64_t ld, int64_t T, int H, int KVH, int dh, int64_t col_k, const float2* tab,
                    cudaStream_t st) {
  if (rope_vec_ok(qkv, ld, dh, col_k))
    rope_qk_vec_kernel<<<blocks_for(T * (H + KVH) * (dh / 16)), kThreads, 0, st>>>(qkv, ld, T, H, KVH, dh, col_k,
                                                                                  tab, 0);
  else
    rope_qk_kernel<<<blocks_for(T * (H + KVH) * (dh / 2)), kThreads, 0, st>>>(qkv, ld, T, H, KVH, dh, col_k, tab, 0);
  return cudaGetLastError();
}
cudaError_t rope_bwd_q(bf16* dqkv, int64_t ld, int64_t T, int H, int dh, const float2* tab, cudaStream_t st) {
  if (rope_vec_ok(dqkv, ld, dh, 0))
    rope_qk_vec_kernel<<<blocks_for(T * H * (dh / 16)), kThreads, 0, st>>>(dqkv, ld, T, H, 0, dh, 0, tab, 1);
  else
    rope_qk_kernel<<<blocks_for(T * H * (dh / 2)), kThreads, 0, st>>>(dqkv, ld, T, H, 0, dh, 0, tab, 1);
  return cudaGetLastError();
}
cudaError_t kv_store(const bf16* qkv, int64_t ld, int64_t T, int64_t kvw, int64_t col_k, int64_t col_v, bf16* kc,
                     bf16* vc, int64_t cache_ld, cudaStream_t st) {
  kv_store_kernel<<<blocks_for(T * kvw), kThreads, 0, st>>>(qkv, ld, T, kvw, col_k, col_v, kc, vc, cache_ld);
  return cudaGetLastError();
}
cudaError_t swiglu_fwd(const bf16* gu, int64_t T, int64_t ffn, bf16* h, cudaStream_t st) {
  swiglu_fwd_kernel<<<blocks_for(T * ffn / 8), kThreads, 0, st>>>(gu, T, ffn, h);
  return cudaGetLastError();
}
cudaError_t swiglu_bwd(const bf16* gu, const bf16* dh, int64_t T, int64_t ffn, bf16* dgu, cudaStream_t st) {
  swiglu_bwd_kernel<<<blocks_for(T * ffn / 8), kThreads, 0, st>>>(gu, dh, T, ffn, dgu);
  return cudaGetLastError();
}
cudaError_t ce_fwd_bwd(const float* logits, int64_t T, int64_t V, int64_t ld, const int32_t* targets, float inv_norm,
                       float* row_loss, bf16* dlogits, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  const bool vec = V % 4 == 0 && ld % 4 == 0 && V <= 4096 * 8 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dlogits) & 7) == 0;
  if (!vec) {
    ce_kernel<<<static_cast<unsigned>(T), 256, 0, st>>>(logits, V, ld, targets, inv_norm, row_loss, dlogits);
  } else if (V <= 4096 * 2) {
    ce_rows_kernel<2><<<static_cast<unsigned>(T), 1024, 0, st>>>(logits, V, ld, targets, inv_norm, row_loss, dlogits);
  } else if (V <= 4096 * 4) {
    ce_rows_kernel<4><<<static_cast<unsigned>(T), 1024, 0, st>>>(logits, V, ld, targets, inv_norm, row_loss, dlogits);
  } else {
    ce_rows_kernel<8><<<static_cast<unsigned>(T), 1024, 0, st>>>(logits, V, ld, targets, inv_norm, row_loss, dlogits);
  }
  return cudaGetLastError();
}
cudaError_t sum_f64(const float* v, int64_t n, double* out, cudaStream_t st) {
  sum_f64_kernel<<<1, 1024, 0, st>>>(v, n, out);
  return cudaGetLastError();
}
cudaError_t rmsnorm_bwd(const float* x, const float* gain, const float* dy, const float* dres, int64_t T, int64_t d,
                        float eps, float* dx, float* rstd, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  rmsnorm_bwd_kernel<<<static_cast<unsigned>((T * 32 + 255) / 256), 256, 0, st>>>(x, gain, dy, dres, T, d, eps, dx,
                                                                                    rstd);
  return cudaGetLastError();
}
cudaError_t rmsnorm_bwd_fused(const float* x, const float* gain, const float* dy, const float* dres, int64_t T,
                              int64_t d, float eps, float* dx, bf16* dx_bf16, float* dgain, cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  if (d % 4) return cudaErrorInvalidValue;
  // one wave at the occupancy the register footprint allows (row state and
  // gain partial live in registers: ~20 regs per float4 column group)
  const int64_t nv = (d + 4 * kBwdThreads - 1) / (4 * kBwdThreads);
  // one wave at the occupancy the register footprint allows (the row and
  // the gain partial live in registers); the row split depends only on T
  // and d, so the reduction order is fixed
  float* part = nullptr;
  int64_t rows = 0, grid = 0;
  cudaError_t e = cudaSuccess;
  bool ok = true;
  auto go = [&](auto nvc) {
    auto* kern = rmsnorm_bwd_rows_kernel<decltype(nvc)::value>;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBwdThreads, 0);
    const int64_t ctas = std::min<int64_t>(T, 148 * std::max(1, per_sm));
    rows = (T + ctas - 1) / ctas;
    grid = (T + rows - 1) / rows;
    e = cudaMallocAsync(&part, static_cast<size_t>(grid * d) * 4, st);
    if (e != cudaSuccess) return;
    kern<<<static_cast<unsigned>(grid), kBwdThreads, 0, st>>>(x, gain, dy, dres, T, static_cast<int>(d), eps, rows,
                                                             dx, dx_bf16, part);
  };
  switch (nv) {
    case 1: go(std::integral_constant<int, 1>()); break;
    case 2: go(std::integral_constant<int, 2>()); break;
    case 3: go(std::integral_constant<int, 3>()); break;
    case 4: go(std::integral_constant<int, 4>()); break;
    case 5: go(std::integral_constant<int, 5>()); break;
    case 6: go(std::integral_constant<int, 6>()); break;
    default: ok = false;
  }
  if (!ok) return cudaErrorInvalidValue;
  if (e != cudaSuccess) return e;
  gain_reduce_cols_kernel<<<static_cast<unsigned>((d + 31) / 32), 256, 0, st>>>(part, static_cast<int>(grid), d,
                                                                               dgain);
  e = cudaGetLastError();
  cudaFreeAsync(part, st);
  return e;
}
bool rmsnorm_bwd_fused_ok(int64_t d) {
  return d % 4 == 0 && d <= 6 * 4 * kBwdThreads;
}
cudaError_t gain_grad(const float* x, const float* dy, const float* rstd, int64_t T, int64_t d, float* dgain,
                      cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  const int splits = static_cast<int>(std::min<int64_t>(kGainSplit, (T + 7) / 8));
  float* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, static_cast<size_t>(splits) * d * 4, st);
  if (e != cudaSuccess) return e;
  gain_grad_partial_kernel<<<dim3(static_cast<unsigned>((d / 4 + 31) / 32), splits), 256, 0, st>>>(x, dy, rstd, T,
                                                                                                     d, part);
  gain_grad_reduce_kernel<<<static_cast<unsigned>((d + 255) / 256), 256, 0, st>>>(part, splits, d, dgain);
  e = cudaGetLastError();
  cudaFreeAsync(part, st);
  return e;
}
cudaError_t dkv_to_dqkv(const float* dk, const float* dv, int64_t acc_ld, int64_t T, int KVH, int dh,
                        const float2* tab, bf16* dqkv, int64_t ld, int64_t col_k, int64_t col_v, cudaStream_t st) {
  const bool vec = dh % 16 == 0 && acc_ld % 4 == 0 && ld % 8 == 0 && col_k % 8 == 0 && col_v % 8 == 0 &&
                   (reinterpret_cast<uintptr_t>(dk) & 15) == 0 && (reinterpret_cast<uintptr_t>(dv) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dqkv) & 15) == 0;
  if (vec)
    dkv_to_dqkv_vec_kernel<<<blocks_for(T * KVH * (dh / 8)), kThreads, 0, st>>>(dk, dv, acc_ld, T, KVH, dh, tab, dqkv,
                                                                               ld, col_k, col_v);
  else
    dkv_to_dqkv_kernel<<<blocks_for(T * KVH * dh), kThreads, 0, st>>>(dk, dv, acc_ld, T, KVH, dh, tab, dqkv, ld,
                                                                     col_k, col_v);
  return cudaGetLastError();
}
cudaError_t scale_rows_f32(float* x, int64_t rows, int64_t cols, int64_t ld, float s, cudaStream_t st) {
  scale_rows_kernel<<<blocks_for(rows * cols), kThreads, 0, st>>>(x, rows, cols, ld, s);
  return cudaGetLastError();
}
cudaError_t embed_bwd(const float* dx, int64_t d, const int32_t* order, const int32_t* uniq, const int32_t* off,
                      int64_t nuniq, float* dE, cudaStream_t st) {
  if (nuniq == 0) return cudaSuccess;
  embed_bwd_kernel<<<static_cast<unsigned>(nuniq), 256, 0, st>>>(dx, d, order, uniq, off, dE);
  return cudaGetLastError();
}
cudaError_t bf16_to_f64(const bf16* src, int64_t ld, int64_t rows, int64_t cols, double* dst, cudaStream_t st) {
  bf16_to_f64_kernel<<<blocks_for(rows * cols), kThreads, 0, st>>>(src, ld, rows, cols, dst);
  return cudaGetLastError();
}
cudaError_t f64_to_bf16(const double* src, int64_t rows, int64_t cols, bf16* dst, int64_t ld, cudaStream_t st) {
  f64_to_bf16_kernel<<<blocks_for(rows * cols), kThreads, 0, st>>>(src, rows, cols, dst, ld);
  return cudaGetLastError();
}
cudaError_t f32_to_f64(const float* src, int64_t ld, int64_t rows, int64_t cols, double* dst, cudaStream_t st) {
  f32_to_f64_kernel<<<blocks_for(rows * cols), kThreads, 0, st>>>(src, ld, rows, cols, dst);
  return cudaGetLastError();
}
cudaError_t f64_to_f32(const double* src, int64_t rows, int64_t cols, float* dst, int64_t ld, cudaStream_t st) {
  f64_to_f32_kernel<<<blocks_for(rows * cols), kThreads, 0, st>>>(src, rows, cols, dst, ld);
  return cudaGetLastError();
}

}  // namespace cfk
