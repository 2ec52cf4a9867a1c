// Pipelined tcgen05 attention backward for head_dim 128 (sm_100a).
//
// Same math as the first version (attention_tc.cu: dQ kernel + dK/dV-owner
// kernel, deterministic, reference toy_model.hpp:436-486), restructured so
// the tensor core never waits for the softmax warps: the streamed dimension
// is cut into 64-wide sub-tiles, S/dP live in double-buffered TMEM
// (2 x 64 columns each), and the MMA issuer runs one sub-tile ahead:
//
//   MMA:     S/dP(i+1)  |  [P/dS(i) ready] dQ or dV,dK(i)  |  S/dP(i+2) ...
//   softmax:      P/dS(i) from TMEM -> bf16 -> swizzled smem  |  P/dS(i+1)
//
// TMEM: S0 S1 dP0 dP1 (4 x 64 cols) + accumulators (dQ: 128; dV + dK: 256).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "attention.h"
#include "attention_tc.h"
#include "common.cuh"

namespace cfk {
namespace {

constexpr int DH = 128;
constexpr int SUB = 64;                     // streamed sub-tile (keys for dQ, queries for dK/dV)
#ifndef CF_BWD_DIAG  // diagnostics only: 1 = softmax math skipped, 2 = softmax side skipped
#define CF_BWD_DIAG 0
#endif
#ifndef CF_DQ_KS
#define CF_DQ_KS 4
#endif
#ifndef CF_DQ_VS
#define CF_DQ_VS 4
#endif
#ifndef CF_DKV_QS
#define CF_DKV_QS 3
#endif
// diagnostics 4 / 5: no operand loads / half of them (MMAs read stale smem)
#if CF_BWD_DIAG == 4
#define TMA_TX(x) 0u
#define TMA_A(...) ((void)0)
#define TMA_B(...) ((void)0)
#elif CF_BWD_DIAG == 5
#define TMA_TX(x) ((x) / 2)
#define TMA_A(...) tma_load_2d(__VA_ARGS__)
#define TMA_B(...) ((void)0)
#else
#define TMA_TX(x) (x)
#define TMA_A(...) tma_load_2d(__VA_ARGS__)
#define TMA_B(...) tma_load_2d(__VA_ARGS__)
#endif
constexpr int KS = CF_DQ_KS, VS = CF_DQ_VS;  // dQ kernel: K / V ring depths
constexpr int QS = CF_DKV_QS;                // dK/dV kernel: Q/dO ring depth
constexpr uint32_t kBox128 = 128 * 64 * 2;  // [128 rows][64 cols] bf16
constexpr uint32_t kBox64 = 64 * 64 * 2;    // [64 rows][64 cols]
constexpr float kLog2e = 1.4426950408889634f;
// CF_ATTN_TRACE=1 (diagnostic builds only): CTA 0 of the persistent dQ
// kernel stamps clock64 at its pipeline events (role 0 = MMA issuer, 1 =
// softmax warp 0, 2 = TMA producer); the host writes them to $CF_TRACE_OUT.
#ifndef CF_ATTN_TRACE
#define CF_ATTN_TRACE 0
#endif
#if CF_ATTN_TRACE
__device__ unsigned long long g_trace[3][8192];
__device__ int g_trace_n[3];
#define TR(role, ev, J)                                                                                  \
  do {                                                                                                 \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) {                                                  \
      const int i_ = g_trace_n[role]++;                                                                \
      if (i_ < 8192)                                                                                   \
        g_trace[role][i_] = (static_cast<unsigned long long>(clock64()) << 20) | ((ev) << 16) | ((J) & 0xffff); \
    }                                                                                                  \
  } while (0)
#else
#define TR(role, ev, J) ((void)0)
#endif

struct Args {
  const AttnSeg* segs;
  const AttnTile* tiles;  // 128-row tiles (queries for dQ, keys for dK/dV)
  // raw rows for the per-CTA-invariant operands staged into TMEM
  const __nv_bfloat16* q;
  int64_t q_stride;
  const __nv_bfloat16* dout;
  int64_t dout_stride;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  int64_t kv_stride;
  const float* lse;
  float* dsum;               // D = rowsum(dO * O): written by the dQ kernel, read by dK/dV
  const __nv_bfloat16* o;    // attention output O (for D)
  int64_t o_stride;
  __nv_bfloat16* dq;
  int64_t dq_stride;
  float* dk_acc;
  float* dv_acc;
  int64_t acc_stride;
  int32_t T, H, KVH;
  float sl2, scale;
  const float2* rope_tab;   // RoPE backward on dQ (and dK with dkv_out)
  __nv_bfloat16* dkv_out;   // direct bf16 dK / dV (standalone chunks)
  int64_t dkv_out_ld, col_k, col_v;
  int32_t stress;  // cf_debug_set_attn_stress: pseudo-random delays in every warp role
};

// Synchronisation stress (testing): a pseudo-random 0-2 us sleep keyed on
// (site, iteration, CTA, warp) so producer, MMA issuer and softmax warps
// reach every mbarrier in perturbed orders; results must stay bitwise equal.
__device__ __forceinline__ void stress_delay(int32_t on, uint32_t site, uint32_t it) {
  if (on) {
    const uint32_t h = (site * 0x9E3779B1u) ^ (it * 0x85EBCA77u) ^ (blockIdx.x * 0xC2B2AE3Du) ^
                       (blockIdx.y * 0x27D4EB2Fu) ^ ((threadIdx.x >> 5) * 0x165667B1u);
    __nanosleep((h >> 21) & 2047u);
  }
}

// Inverse rotate-half of 32 (a, b) pairs (a = columns c0.., b = c0+64..)
// with (cos, sin) pairs tab[c0 .. c0+32): the RoPE backward rope_qk applies.
__device__ __forceinline__ void rope_inverse32(const float2* tab, float (&a)[32], float (&b)[32]) {
  const float4* tp = reinterpret_cast<const float4*>(tab);
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const float4 cs = tp[e];
    const float s0 = -cs.y, s1 = -cs.w;
    const float a0 = a[2 * e], b0 = b[2 * e], a1 = a[2 * e + 1], b1 = b[2 * e + 1];
    a[2 * e] = a0 * cs.x - b0 * s0;
    b[2 * e] = b0 * cs.x + a0 * s0;
    a[2 * e + 1] = a1 * cs.z - b1 * s1;
    b[2 * e + 1] = b1 * cs.z + a1 * s1;
  }
}
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32]) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    d4[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                       pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}
// rope_inverse32 / store_bf16x32 on 16 (a, b) pairs / 16 values
__device__ __forceinline__ void rope_inverse16(const float2* tab, float (&a)[16], float (&b)[16]) {
  const float4* tp = reinterpret_cast<const float4*>(tab);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const float4 cs = tp[e];
    const float s0 = -cs.y, s1 = -cs.w;
    const float a0 = a[2 * e], b0 = b[2 * e], a1 = a[2 * e + 1], b1 = b[2 * e + 1];
    a[2 * e] = a0 * cs.x - b0 * s0;
    b[2 * e] = b0 * cs.x + a0 * s0;
    a[2 * e + 1] = a1 * cs.z - b1 * s1;
    b[2 * e + 1] = b1 * cs.z + a1 * s1;
  }
}
__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst, const float (&v)[16]) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 2; ++q)
    d4[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                       pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}
// bf16 round trip (the unfused path rotates the stored bf16 dQ)
__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One thread = one TMEM lane (row): copies 64 bf16 (this half's columns) of a
// global row into 32 TMEM columns at `taddr` (A-operand layout: element k of
// the row in column k/2).  Rows that do not exist are zero-filled.  With
// `dot_with` set, also returns sum_k row[k] * dot_with[k] (the D = dO.O
// softmax-statistic reduction, fused into the dQ kernel's staging).
__device__ __forceinline__ float stage_row_tmem(uint32_t taddr, const __nv_bfloat16* src, bool ok,
                                                const __nv_bfloat16* dot_with = nullptr) {
  uint32_t w[32];
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 v = ok ? __ldg(s4 + c) : make_uint4(0u, 0u, 0u, 0u);
    w[4 * c] = v.x;
    w[4 * c + 1] = v.y;
    w[4 * c + 2] = v.z;
    w[4 * c + 3] = v.w;
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]),
      "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]),
      "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
      : "memory");
  float acc = 0.f;
  if (dot_with && ok) {
    const uint4* o4 = reinterpret_cast<const uint4*>(dot_with);
    float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 ov = __ldg(o4 + c);
      const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 a2 = *reinterpret_cast<const __nv_bfloat162*>(&w[4 * c + e]);
        const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&ow[e]);
        part[e] = fmaf(__low2float(a2), __low2float(b2), part[e]);
        part[e] = fmaf(__high2float(a2), __high2float(b2), part[e]);
      }
    }
    acc = (part[0] + part[1]) + (part[2] + part[3]);
  }
  return acc;
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st32w(uint32_t taddr, const uint32_t (&w)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]),
      "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]),
      "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
      : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
// 32 rows x 64 bf16 of a row-major bf16 matrix (row i at base + i * stride;
// rows >= valid read as zero) into registers with lane i holding row i
// (out[c] = 16-byte chunk c).  Read coalesced -- 8 lanes per 128-byte
// half-row, 4 rows per load -- and transposed through a 4 KB per-warp smem
// scratch whose 16-byte chunks are XOR-swizzled by row (4 wavefronts per
// 512-byte access, the minimum).  A lane-per-row global read instead touches
// 32 cache lines per load instruction: staging a short-chunk dQ item that way
// took ~7,900 cycles, 38 % of the kernel (tools/attn_trace.py).
__device__ __forceinline__ void rows_to_lanes(uint32_t scr, const __nv_bfloat16* base, int64_t stride, int valid,
                                              uint4 (&out)[8]) {
  const int lane = threadIdx.x & 31, c = lane & 7;
  uint4 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = 4 * k + (lane >> 3);
    v[k] = i < valid ? __ldg(reinterpret_cast<const uint4*>(base + i * stride) + c) : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = 4 * k + (lane >> 3);
    sts128(scr + i * 128 + ((c ^ (i & 7)) << 4), v[k]);
  }
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) out[cc] = lds128(scr + lane * 128 + ((cc ^ (lane & 7)) << 4));
  __syncwarp();
}
// rows_to_lanes for 32 bf16 (64 bytes) per row: 4 lanes per row, 8 rows per
// load, a 2 KB scratch with chunks swizzled by (row >> 1) & 3 so the 8 lanes
// of each read wavefront hit distinct bank groups.
__device__ __forceinline__ void rows_to_lanes64(uint32_t scr, const __nv_bfloat16* base, int64_t stride, int valid,
                                                uint4 (&out)[4]) {
  const int lane = threadIdx.x & 31, c = lane & 3;
  uint4 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = 8 * k + (lane >> 2);
    v[k] = i < valid ? __ldg(reinterpret_cast<const uint4*>(base + i * stride) + c) : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = 8 * k + (lane >> 2);
    sts128(scr + i * 64 + ((c ^ ((i >> 1) & 3)) << 4), v[k]);
  }
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < 4; ++cc) out[cc] = lds128(scr + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4));
  __syncwarp();
}
__device__ __forceinline__ void words_of(const uint4 (&x)[8], uint32_t (&w)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    w[4 * c] = x[c].x;
    w[4 * c + 1] = x[c].y;
    w[4 * c + 2] = x[c].z;
    w[4 * c + 3] = x[c].w;
  }
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
constexpr int kThreads = 320;
// dK/dV kernel: 16 softmax-side warps (4 per TMEM lane quarter, 16 query
// columns each) + TMA + MMA; 576 threads cap registers at 96 per thread
constexpr int kDkvThreads = 576;

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
// stage_row_tmem for 32 bf16 (16 TMEM columns)
__device__ __forceinline__ void stage_row_tmem16(uint32_t taddr, const __nv_bfloat16* src, bool ok) {
  uint32_t w[16];
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 v = ok ? __ldg(s4 + c) : make_uint4(0u, 0u, 0u, 0u);
    w[4 * c] = v.x;
    w[4 * c + 1] = v.y;
    w[4 * c + 2] = v.z;
    w[4 * c + 3] = v.w;
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
      : "memory");
}

// 16-byte chunk c (0..7) of row r in a [rows][64] SW128 box
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
  return static_cast<uint32_t>(r * 128 + ((c ^ (r & 7)) << 4));
}
// K-major operand made of boxes of `box` bytes along K (64 elements each)
__device__ __forceinline__ uint64_t kdesc(uint32_t base, uint32_t box, int ks) {
  return umma_desc_sw128(base + (ks >> 2) * box + (ks & 3) * 32, 16, 1024);
}
// MN-major view: N = 128 (two 64-col slabs `box` bytes apart), K = rows
__device__ __forceinline__ uint64_t mndesc(uint32_t base, uint32_t box, int ks) {
  return umma_desc_sw128(base + ks * 2048, box, 1024);
}

// ------------------------------------------------------------------ dQ
// CTA = 128 queries x one q head; keys streamed in 64-key sub-tiles.
__global__ void __launch_bounds__(kThreads, 1)
    dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO,
              const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // Q and dO (per-CTA invariant A operands of S and dP) live in TMEM.
  // K is held until dQ of its sub-tile (late), V only until dP (early):
  // separate rings, KS and VS deep, so loads are issued >= 2 sub-tiles ahead.
  uint8_t* sK = sm;                    // KS stages x 2 x [64][64]
  uint8_t* sV = sK + KS * 2 * kBox64;  // VS stages
  uint8_t* sS = sV + VS * 2 * kBox64;  // 2 x [128 q][64 keys] (dS)
  float* sRowD = reinterpret_cast<float*>(sS + 2 * kBox128);  // [2 half][128 rows]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRowD + 256);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;              // [KS]
  uint64_t* k_empty = k_full + KS;         // [KS]
  uint64_t* v_full = k_empty + KS;         // [VS]
  uint64_t* v_empty = v_full + VS;         // [VS]
  uint64_t* s_full = v_empty + VS;         // [2]
  uint64_t* s_free = s_full + 2;           // [2]
  uint64_t* ds_full = s_free + 2;          // [2]
  uint64_t* ds_free = ds_full + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ds_free + 2);

  const AttnTile tl = a.tiles[blockIdx.x];
  const AttnSeg sg = a.segs[tl.seg];
  const int h = blockIdx.y, g = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_row0 = sg.q_start + tl.first;
  const int kv_len = sg.prefix + tl.first + tl.count;
  const int nkt = (kv_len + SUB - 1) / SUB;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmO);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 8);  // softmax warps staging Q / dO into TMEM
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);   // one arrive per softmax warp
      mbar_init(&ds_full[i], 8);
      mbar_init(&ds_free[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // S[b] at tmem + 64b, dP[b] at tmem + 128 + 64b
  const uint32_t tQ = tmem + 256;     // dQ accumulator
  const uint32_t tAq = tmem + 384;    // Q  (A operand, 64 columns)
  const uint32_t tAo = tmem + 448;    // dO (A operand, 64 columns)

  if (warp == 8) {
    if (lane == 0) {
      for (int j = 0; j < nkt; ++j) {
        const int sk = j % KS, sv = j % VS;
        const int krow = sg.kv_row0 + j * SUB;
        stress_delay(a.stress, 1, j);
        mbar_wait(&v_empty[sv], ((j / VS) & 1) ^ 1);
        mbar_expect_tx(&v_full[sv], TMA_TX(2 * kBox64));
        TMA_A(sV + sv * 2 * kBox64, &tmV, &v_full[sv], g * DH, krow);
        TMA_B(sV + sv * 2 * kBox64 + kBox64, &tmV, &v_full[sv], g * DH + 64, krow);
        mbar_wait(&k_empty[sk], ((j / KS) & 1) ^ 1);
        mbar_expect_tx(&k_full[sk], TMA_TX(2 * kBox64));
        TMA_A(sK + sk * 2 * kBox64, &tmK, &k_full[sk], g * DH, krow);
        TMA_B(sK + sk * 2 * kBox64 + kBox64, &tmK, &k_full[sk], g * DH + 64, krow);
      }
    }
  } else if (warp == 9) {
    // whole warp, convergent (elect.sync inside the issue helpers)
    constexpr uint32_t idS = umma_idesc_bf16(128, SUB, 0, 0);  // S, dP: N = 64 keys
    constexpr uint32_t idQ = umma_idesc_bf16(128, 128, 0, 1);  // dQ: N = dh, B = K (MN-major view)
    const uint32_t sK0 = smem_u32(sK), sV0 = smem_u32(sV), sS0 = smem_u32(sS);
    const uint32_t bKf = smem_u32(k_full), bKe = smem_u32(k_empty), bVf = smem_u32(v_full),
                   bVe = smem_u32(v_empty), bSf = smem_u32(s_full), bSr = smem_u32(s_free),
                   bDf = smem_u32(ds_full), bDr = smem_u32(ds_free);
    int ik = 0, iv = 0, ck = 0;  // ring slots: K/V for the next S/dP issue, K for the next dQ
    uint32_t pk = 0, pv = 0;
    auto issue_s = [&](int j) {
      const uint32_t b = j & 1;
      mbar_wait_s(bKf + ik * 8, pk);
      mbar_wait_s(bVf + iv * 8, pv);
      mbar_wait_s(bSr + b * 8, ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t k0 = sK0 + ik * 2 * kBox64, v0 = sV0 + iv * 2 * kBox64;
      // K = dh in two 4-MMA chains (one 64-column box each): A columns step 8,
      // B descriptors step 32 bytes inside a box
      umma4_ts_w<8, 2>(tmem + b * 64, tAq, kdesc(k0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tmem + b * 64, tAq + 32, kdesc(k0, kBox64, 4), idS, 1u);
      umma4_ts_w<8, 2>(tmem + 128 + b * 64, tAo, kdesc(v0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tmem + 128 + b * 64, tAo + 32, kdesc(v0, kBox64, 4), idS, 1u);
      umma_commit_w(bVe + iv * 8);
      umma_commit_w(bSf + b * 8);
      if (++ik == KS) { ik = 0; pk ^= 1; }
      if (++iv == VS) { iv = 0; pv ^= 1; }
    };
    mbar_wait(q_full, 0);  // Q / dO staged into TMEM by the softmax warps
    tc_fence_after();
    issue_s(0);
    for (int j = 0; j < nkt; ++j) {
      stress_delay(a.stress, 2, j);
      if (j + 1 < nkt) issue_s(j + 1);
      const uint32_t b = j & 1;
      mbar_wait_s(bDf + b * 8, (j >> 1) & 1);
      tc_fence_after();
      const uint32_t s0 = sS0 + b * kBox128, k0 = sK0 + ck * 2 * kBox64;
#if CF_BWD_DIAG < 3
      umma4_ss_w<2, 128>(tQ, kdesc(s0, kBox128, 0), mndesc(k0, kBox64, 0), idQ, j > 0 ? 1u : 0u);
#endif
      umma_commit_w(bKe + ck * 8);
      umma_commit_w(bDr + b * 8);
      if (++ck == KS) ck = 0;
    }
  } else {
    const int quarter = warp & 3, half = warp >> 2;  // half: which 32 of the 64 key columns
    const int row = quarter * 32 + lane;
    const int qi = tl.first + row;
    const bool ok = qi < sg.len && row < tl.count;
    const int lim = sg.prefix + min(qi, sg.len - 1);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float lse2 = ok ? a.lse[static_cast<int64_t>(h) * a.T + q_row0 + row] * kLog2e : 0.f;
    float D;
    {
      const bool rok = row < tl.count;
      const int64_t r = q_row0 + row;
      stage_row_tmem(tAq + lane_off + half * 32, a.q + r * a.q_stride + static_cast<int64_t>(h) * DH + half * 64, rok);
      const float dpart = stage_row_tmem(
          tAo + lane_off + half * 32, a.dout + r * a.dout_stride + static_cast<int64_t>(h) * DH + half * 64, ok,
          a.o + r * a.o_stride + static_cast<int64_t>(h) * DH + half * 64);
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(q_full);
      // D = rowsum(dO * O): the two half-rows meet in smem (fixed order)
      sRowD[half * 128 + row] = dpart;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      D = sRowD[row] + sRowD[128 + row];
      if (ok && half == 0) a.dsum[static_cast<int64_t>(h) * a.T + q_row0 + row] = D;
    }
    const uint32_t bSf = smem_u32(s_full), bSr = smem_u32(s_free), bDf = smem_u32(ds_full),
                   bDr = smem_u32(ds_free), sS0 = smem_u32(sS);
    const int klim = ok ? lim : -1;  // last visible key of this query row (-1: row absent)
    const int tile_lim = sg.prefix + tl.first;  // smallest row limit of the tile
    uint32_t dst_off[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) dst_off[c] = sw_off(row, half * 4 + c);
    for (int j = 0; j < nkt; ++j) {
      const uint32_t b = j & 1;
      mbar_wait_s(bSf + b * 8, (j >> 1) & 1);
      tc_fence_after();
#if CF_BWD_DIAG >= 2
      warp_arrive_s(bSr + b * 8);
      if (j >= 2) mbar_wait_s(bDr + b * 8, ((j >> 1) & 1) ^ 1);
      warp_arrive_s(bDf + b * 8);
      continue;
#endif
      uint32_t rs[32], rp[32];
      tmem_ld32(tmem + b * 64 + lane_off + half * 32, rs);
      tmem_ld32(tmem + 128 + b * 64 + lane_off + half * 32, rp);
      tmem_ld_wait();
      tc_fence_before();
      warp_arrive_s(bSr + b * 8);
      uint32_t pk[16];
      // dS = P * (dP - D); P masked only on sub-tiles that cross the causal
      // diagonal or the end of the segment (two separately compiled bodies)
      // pairs in FFMA2 / FADD2 / FMUL2: x = s * sl2 - lse2, dS = P (dP - D)
      const float2 sl2v = make_float2(a.sl2, a.sl2), nl = make_float2(-lse2, -lse2), nD = make_float2(-D, -D);
      auto body = [&](auto masked) {
        const int key0 = j * SUB + half * 32;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = ffma2(make_float2(__uint_as_float(rs[2 * e]), __uint_as_float(rs[2 * e + 1])), sl2v, nl);
          float2 p = make_float2(ex2(x.x), ex2(x.y));
          if constexpr (decltype(masked)::value) {
            p.x = key0 + 2 * e <= klim ? p.x : 0.f;
            p.y = key0 + 2 * e + 1 <= klim ? p.y : 0.f;
          }
          const float2 ds =
              fmul2(p, fadd2(make_float2(__uint_as_float(rp[2 * e]), __uint_as_float(rp[2 * e + 1])), nD));
          pk[e] = pack_bf16(ds.x, ds.y);
        }
      };
#if CF_BWD_DIAG == 1
      for (int e = 0; e < 16; ++e) pk[e] = rs[e] ^ rp[e];
#else
      if (j * SUB + SUB - 1 <= tile_lim)  // uniform: every row of the tile sees every key
        body(std::false_type{});
      else
        body(std::true_type{});
#endif
      stress_delay(a.stress, 3, j);
      if (j >= 2) mbar_wait_s(bDr + b * 8, ((j >> 1) & 1) ^ 1);
      const uint32_t dst = sS0 + b * kBox128;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        sts128(dst + dst_off[c], make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
      fence_async_smem();
      warp_arrive_s(bDf + b * 8);
    }
    const int last = nkt - 1;
    mbar_wait(&ds_free[last & 1], (last >> 1) & 1);
    tc_fence_after();
    __nv_bfloat16* out = a.dq + static_cast<int64_t>(q_row0 + row) * a.dq_stride + h * DH;
    if (a.rope_tab) {  // this half takes rotate-half partners: chunks (half, half + 2)
      uint32_t ra[32], rb[32];
      tmem_ld32(tQ + lane_off + half * 32, ra);
      tmem_ld32(tQ + lane_off + (half + 2) * 32, rb);
      tmem_ld_wait();
      if (ok) {
        float fa[32], fb[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          fa[e] = bf16_round(__uint_as_float(ra[e]) * a.scale);
          fb[e] = bf16_round(__uint_as_float(rb[e]) * a.scale);
        }
        rope_inverse32(a.rope_tab + static_cast<int64_t>(q_row0 + row) * (DH / 2) + half * 32, fa, fb);
        store_bf16x32(out + half * 32, fa);
        store_bf16x32(out + (half + 2) * 32, fb);
      }
    } else {
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int c = half * 2 + cc;  // 32-column chunk of dQ
      uint32_t r[32];
      tmem_ld32(tQ + lane_off + c * 32, r);
      tmem_ld_wait();
      if (ok) {
        uint4* d4 = reinterpret_cast<uint4*>(out + c * 32);
        const float sc = a.scale;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          d4[q] = make_uint4(pack_bf16(__uint_as_float(r[8 * q]) * sc, __uint_as_float(r[8 * q + 1]) * sc),
                             pack_bf16(__uint_as_float(r[8 * q + 2]) * sc, __uint_as_float(r[8 * q + 3]) * sc),
                             pack_bf16(__uint_as_float(r[8 * q + 4]) * sc, __uint_as_float(r[8 * q + 5]) * sc),
                             pack_bf16(__uint_as_float(r[8 * q + 6]) * sc, __uint_as_float(r[8 * q + 7]) * sc));
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// ------------------------------------------------------- dQ, persistent
// dq_kernel's math and 64-key sub-tiles for packed short segments, with one
// CTA per SM looping over (128-query tile, q head) items (item = blockIdx.x
// + k * gridDim.x): TMEM and barriers are set up once, the producer streams
// the next item's K/V while the current one drains, and the softmax warps
// stage the next item's Q / dO into TMEM (the A operands are free once the
// item's last MMA has completed) before reading out the current dQ, so the
// MMA issuer starts the next item while the dQ row stores run.  Ring slots
// and the S / dP buffer parity run on counters that continue across items.
__device__ __forceinline__ void item_of(const Args& a, int nq, int item, AttnTile& tl, AttnSeg& sg, int& h) {
  h = item / nq;
  tl = a.tiles[item - h * nq];
  sg = a.segs[tl.seg];
}
__global__ void __launch_bounds__(kThreads, 1)
    dq_persist_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Args a,
                      int nq) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;                    // KS stages x 2 x [64][64]
  uint8_t* sV = sK + KS * 2 * kBox64;  // VS stages
  uint8_t* sS = sV + VS * 2 * kBox64;  // 2 x [128 q][64 keys] (dS)
  float* sRowD = reinterpret_cast<float*>(sS + 2 * kBox128);  // [2 half][128 rows]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRowD + 256);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;              // [KS]
  uint64_t* k_empty = k_full + KS;         // [KS]
  uint64_t* v_full = k_empty + KS;         // [VS]
  uint64_t* v_empty = v_full + VS;         // [VS]
  uint64_t* s_full = v_empty + VS;         // [2]
  uint64_t* s_free = s_full + 2;           // [2]
  uint64_t* ds_full = s_free + 2;          // [2]
  uint64_t* ds_free = ds_full + 2;         // [2]
  uint64_t* dq_done = ds_free + 2;         // MMA: the item's last MMA completed
  uint64_t* dq_free = dq_done + 1;         // softmax: the item's dQ read out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_free + 1);

  const int items = nq * a.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = a.H / a.KVH;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 8);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&ds_full[i], 8);
      mbar_init(&ds_free[i], 1);
    }
    mbar_init(dq_done, 1);
    mbar_init(dq_free, 8);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tQ = tmem + 256, tAq = tmem + 384, tAo = tmem + 448;

  if (warp == 8) {
    if (lane == 0) {
      int jj = 0;  // sub-tiles loaded so far (ring position)
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        AttnTile tl;
        AttnSeg sg;
        int h;
        item_of(a, nq, item, tl, sg, h);
        const int g = h / per;
        const int nkt = (sg.prefix + tl.first + tl.count + SUB - 1) / SUB;
        for (int j = 0; j < nkt; ++j, ++jj) {
          const int sk = jj % KS, sv = jj % VS;
          const int krow = sg.kv_row0 + j * SUB;
          stress_delay(a.stress, 1, jj);
          mbar_wait(&v_empty[sv], ((jj / VS) & 1) ^ 1);
          TR(2, 1, jj);
          mbar_expect_tx(&v_full[sv], 2 * kBox64);
          tma_load_2d(sV + sv * 2 * kBox64, &tmV, &v_full[sv], g * DH, krow);
          tma_load_2d(sV + sv * 2 * kBox64 + kBox64, &tmV, &v_full[sv], g * DH + 64, krow);
          mbar_wait(&k_empty[sk], ((jj / KS) & 1) ^ 1);
          mbar_expect_tx(&k_full[sk], 2 * kBox64);
          tma_load_2d(sK + sk * 2 * kBox64, &tmK, &k_full[sk], g * DH, krow);
          tma_load_2d(sK + sk * 2 * kBox64 + kBox64, &tmK, &k_full[sk], g * DH + 64, krow);
        }
      }
    }
  } else if (warp == 9) {
    constexpr uint32_t idS = umma_idesc_bf16(128, SUB, 0, 0);
    constexpr uint32_t idQ = umma_idesc_bf16(128, 128, 0, 1);
    const uint32_t sK0 = smem_u32(sK), sV0 = smem_u32(sV), sS0 = smem_u32(sS);
    const uint32_t bKf = smem_u32(k_full), bKe = smem_u32(k_empty), bVf = smem_u32(v_full),
                   bVe = smem_u32(v_empty), bSf = smem_u32(s_full), bSr = smem_u32(s_free),
                   bDf = smem_u32(ds_full), bDr = smem_u32(ds_free), bQf = smem_u32(q_full),
                   bQd = smem_u32(dq_done), bQr = smem_u32(dq_free);
    int ik = 0, iv = 0, ck = 0;
    uint32_t pk = 0, pv = 0;
    auto issue_s = [&](int J) {
      const uint32_t b = J & 1;
      TR(0, 1, J);
      mbar_wait_s(bKf + ik * 8, pk);
      mbar_wait_s(bVf + iv * 8, pv);
      TR(0, 2, J);
      mbar_wait_s(bSr + b * 8, ((J >> 1) & 1) ^ 1);
      tc_fence_after();
      TR(0, 3, J);
      const uint32_t k0 = sK0 + ik * 2 * kBox64, v0 = sV0 + iv * 2 * kBox64;
      umma4_ts_w<8, 2>(tmem + b * 64, tAq, kdesc(k0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tmem + b * 64, tAq + 32, kdesc(k0, kBox64, 4), idS, 1u);
      umma4_ts_w<8, 2>(tmem + 128 + b * 64, tAo, kdesc(v0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tmem + 128 + b * 64, tAo + 32, kdesc(v0, kBox64, 4), idS, 1u);
      umma_commit_w(bVe + iv * 8);
      umma_commit_w(bSf + b * 8);
      if (++ik == KS) { ik = 0; pk ^= 1; }
      if (++iv == VS) { iv = 0; pv ^= 1; }
    };
    int J0 = 0, n = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
      AttnTile tl;
      AttnSeg sg;
      int h;
      item_of(a, nq, item, tl, sg, h);
      const int nkt = (sg.prefix + tl.first + tl.count + SUB - 1) / SUB;
      TR(0, 4, J0);
      mbar_wait_s(bQf, n & 1);  // this item's Q / dO staged
      tc_fence_after();
      TR(0, 5, J0);
      issue_s(J0);
      for (int j = 0; j < nkt; ++j) {
        const int J = J0 + j;
        stress_delay(a.stress, 2, J);
        if (j + 1 < nkt) issue_s(J + 1);
        const uint32_t b = J & 1;
        mbar_wait_s(bDf + b * 8, (J >> 1) & 1);
        TR(0, 6, J);
        if (j == 0 && n > 0) mbar_wait_s(bQr, (n - 1) & 1);  // previous item's dQ read out
        tc_fence_after();
        TR(0, 7, J);
        const uint32_t s0 = sS0 + b * kBox128, k0 = sK0 + ck * 2 * kBox64;
        umma4_ss_w<2, 128>(tQ, kdesc(s0, kBox128, 0), mndesc(k0, kBox64, 0), idQ, j > 0 ? 1u : 0u);
        umma_commit_w(bKe + ck * 8);
        umma_commit_w(bDr + b * 8);
        if (++ck == KS) ck = 0;
      }
      umma_commit_w(bQd);
      J0 += nkt;
    }
  } else {
    const int quarter = warp & 3, half = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t bSf = smem_u32(s_full), bSr = smem_u32(s_free), bDf = smem_u32(ds_full),
                   bDr = smem_u32(ds_free), sS0 = smem_u32(sS), bQd = smem_u32(dq_done), bQr = smem_u32(dq_free);
    uint32_t dst_off[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) dst_off[c] = sw_off(row, half * 4 + c);
    // stage item `it`'s Q / dO rows into TMEM and return D = rowsum(dO * O)
    // per-warp transpose scratch: the dS buffers, free whenever staging runs
    // (before the first item, and after dq_done: every MMA of the previous
    // item, the dQ GEMMs that read dS included, has completed)
    const uint32_t scr = smem_u32(sS) + warp * 4096;
    auto stage = [&](int it, int rnd) -> float {
      AttnTile tl;
      AttnSeg sg;
      int h;
      item_of(a, nq, it, tl, sg, h);
      const int qi = tl.first + row;
      const bool ok = qi < sg.len && row < tl.count;
      const int vq = tl.count - quarter * 32;                             // rows with Q
      const int vo = min(tl.count, sg.len - tl.first) - quarter * 32;     // rows with dO / O
      const int64_t r0 = sg.q_start + tl.first + quarter * 32;            // this warp's first row
      const int64_t hc = static_cast<int64_t>(h) * DH + half * 64;
      float dpart = 0.f;
      {
        uint4 x[8];
        uint32_t w[32];
        rows_to_lanes(scr, a.q + r0 * a.q_stride + hc, a.q_stride, vq, x);
        words_of(x, w);
        tmem_st32w(tAq + lane_off + half * 32, w);
      }
      {
        uint4 xd[8], xo[8];
        uint32_t w[32];
        rows_to_lanes(scr, a.dout + r0 * a.dout_stride + hc, a.dout_stride, vo, xd);
        words_of(xd, w);
        tmem_st32w(tAo + lane_off + half * 32, w);
        rows_to_lanes(scr, a.o + r0 * a.o_stride + hc, a.o_stride, vo, xo);
        if (ok) {  // D partial: same arithmetic order as stage_row_tmem
          float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t ow[4] = {xo[c].x, xo[c].y, xo[c].z, xo[c].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const __nv_bfloat162 a2 = *reinterpret_cast<const __nv_bfloat162*>(&w[4 * c + e]);
              const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&ow[e]);
              part[e] = fmaf(__low2float(a2), __low2float(b2), part[e]);
              part[e] = fmaf(__high2float(a2), __high2float(b2), part[e]);
            }
          }
          dpart = (part[0] + part[1]) + (part[2] + part[3]);
        }
      }
      const int64_t r = sg.q_start + tl.first + row;
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(q_full);
      // the two half-rows meet in smem (fixed order); rnd alternates the
      // buffer so a fast warp pair cannot overwrite a slot still being read
      sRowD[half * 128 + row] = dpart;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      const float D = sRowD[row] + sRowD[128 + row];
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      if (ok && half == 0) a.dsum[static_cast<int64_t>(h) * a.T + r] = D;
      (void)rnd;
      return D;
    };
    int J0 = 0, n = 0;
    float D = blockIdx.x < items ? stage(blockIdx.x, 0) : 0.f;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
      AttnTile tl;
      AttnSeg sg;
      int h;
      item_of(a, nq, item, tl, sg, h);
      const int q_row0 = sg.q_start + tl.first;
      const int nkt = (sg.prefix + tl.first + tl.count + SUB - 1) / SUB;
      const int qi = tl.first + row;
      const bool ok = qi < sg.len && row < tl.count;
      const int lim = sg.prefix + min(qi, sg.len - 1);
      const float lse2 = ok ? a.lse[static_cast<int64_t>(h) * a.T + q_row0 + row] * kLog2e : 0.f;
      const int klim = ok ? lim : -1;
      const int tile_lim = sg.prefix + tl.first;
      {
        // pull the next item's Q / dO / O half-rows into L2 now, so staging
        // them after this item's last MMA waits on L2, not HBM
        const int nx = item + gridDim.x;
        if (nx < items) {
          AttnTile tn;
          AttnSeg sn;
          int hn;
          item_of(a, nq, nx, tn, sn, hn);
          if (row < tn.count) {
            const int64_t r = sn.q_start + tn.first + row;
            const int64_t hc = static_cast<int64_t>(hn) * DH + half * 64;
            prefetch_l2(a.q + r * a.q_stride + hc);
            prefetch_l2(a.dout + r * a.dout_stride + hc);
            prefetch_l2(a.o + r * a.o_stride + hc);
          }
        }
      }
      const float2 sl2v = make_float2(a.sl2, a.sl2), nl = make_float2(-lse2, -lse2), nD = make_float2(-D, -D);
      for (int j = 0; j < nkt; ++j) {
        const int J = J0 + j;
        const uint32_t b = J & 1;
        if (warp == 0) TR(1, 1, J);
        mbar_wait_s(bSf + b * 8, (J >> 1) & 1);
        tc_fence_after();
        if (warp == 0) TR(1, 2, J);
        uint32_t rs[32], rp[32];
        tmem_ld32(tmem + b * 64 + lane_off + half * 32, rs);
        tmem_ld32(tmem + 128 + b * 64 + lane_off + half * 32, rp);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive_s(bSr + b * 8);
        uint32_t pk[16];
        auto body = [&](auto masked) {
          const int key0 = j * SUB + half * 32;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 x = ffma2(make_float2(__uint_as_float(rs[2 * e]), __uint_as_float(rs[2 * e + 1])), sl2v, nl);
            float2 p = make_float2(ex2(x.x), ex2(x.y));
            if constexpr (decltype(masked)::value) {
              p.x = key0 + 2 * e <= klim ? p.x : 0.f;
              p.y = key0 + 2 * e + 1 <= klim ? p.y : 0.f;
            }
            const float2 ds =
                fmul2(p, fadd2(make_float2(__uint_as_float(rp[2 * e]), __uint_as_float(rp[2 * e + 1])), nD));
            pk[e] = pack_bf16(ds.x, ds.y);
          }
        };
        if (j * SUB + SUB - 1 <= tile_lim)
          body(std::false_type{});
        else
          body(std::true_type{});
        stress_delay(a.stress, 3, J);
        if (warp == 0) TR(1, 3, J);
        if (J >= 2) mbar_wait_s(bDr + b * 8, ((J >> 1) & 1) ^ 1);
        if (warp == 0) TR(1, 4, J);
        const uint32_t dst = sS0 + b * kBox128;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          sts128(dst + dst_off[c], make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
        fence_async_smem();
        warp_arrive_s(bDf + b * 8);
      }
      J0 += nkt;
      mbar_wait_s(bQd, n & 1);  // every MMA of this item done: Q / dO / dQ settled
      tc_fence_after();
      if (warp == 0) TR(1, 5, J0);
      // the next item's Q / dO go into TMEM now, so its S / dP overlap this
      // item's dQ read-out
      const int next = item + gridDim.x;
      const float Dn = next < items ? stage(next, n + 1) : 0.f;
      if (warp == 0) TR(1, 6, J0);
      __nv_bfloat16* out = a.dq + static_cast<int64_t>(q_row0 + row) * a.dq_stride + h * DH;
      if (a.rope_tab) {
        uint32_t ra[32], rb[32];
        tmem_ld32(tQ + lane_off + half * 32, ra);
        tmem_ld32(tQ + lane_off + (half + 2) * 32, rb);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive_s(bQr);
        if (ok) {
          float fa[32], fb[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            fa[e] = bf16_round(__uint_as_float(ra[e]) * a.scale);
            fb[e] = bf16_round(__uint_as_float(rb[e]) * a.scale);
          }
          rope_inverse32(a.rope_tab + static_cast<int64_t>(q_row0 + row) * (DH / 2) + half * 32, fa, fb);
          store_bf16x32(out + half * 32, fa);
          store_bf16x32(out + (half + 2) * 32, fb);
        }
      } else {
        uint32_t r0[32], r1[32];
        tmem_ld32(tQ + lane_off + (half * 2) * 32, r0);
        tmem_ld32(tQ + lane_off + (half * 2 + 1) * 32, r1);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive_s(bQr);
        if (ok) {
          const float sc = a.scale;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const uint32_t* r = cc ? r1 : r0;
            uint4* d4 = reinterpret_cast<uint4*>(out + (half * 2 + cc) * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              d4[q] = make_uint4(pack_bf16(__uint_as_float(r[8 * q]) * sc, __uint_as_float(r[8 * q + 1]) * sc),
                                 pack_bf16(__uint_as_float(r[8 * q + 2]) * sc, __uint_as_float(r[8 * q + 3]) * sc),
                                 pack_bf16(__uint_as_float(r[8 * q + 4]) * sc, __uint_as_float(r[8 * q + 5]) * sc),
                                 pack_bf16(__uint_as_float(r[8 * q + 6]) * sc, __uint_as_float(r[8 * q + 7]) * sc));
          }
        }
      }
      if (warp == 0) TR(1, 7, J0);
      D = Dn;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}


// --------------------------------------------------- dQ, persistent + TMA
// dq_persist_kernel with the per-item staging taken off the critical path:
// the clock64 trace (profiles/round2_dq_persist_trace.txt) has the MMA issuer
// waiting ~32 % of the time for the softmax warps to fetch the next item's
// Q / dO / O rows from global memory.  Here
//   * D = rowsum(dO * O) comes from dsum_rows_kernel, launched just before;
//   * the producer TMA-loads the next item's Q and dO tiles into a 64 KB smem
//     buffer (qo_tma) once the current item's copy has left it (qo_free);
//   * the softmax warps copy them into the Q / dO TMEM A operands (smem ->
//     tcgen05.st) as soon as the s_full of the item's last sub-tile certifies
//     its last S / dP MMAs, and the MMA issuer queues the next item's first
//     S / dP ahead of the current item's last dQ GEMM;
//   * the next item's LSE and D are read at that point too.
// Items and the per-item math are dq_persist_kernel's.
__global__ void __launch_bounds__(kThreads, 1)
    dq_persist_tma_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO, Args a,
                          int nq) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;                    // KS stages x 2 x [64][64]
  uint8_t* sV = sK + KS * 2 * kBox64;  // VS stages
  uint8_t* sS = sV + VS * 2 * kBox64;  // 2 x [128 q][64 keys] (dS)
  uint8_t* sQO = sS + 2 * kBox128;     // next item's Q, dO: 2 x 2 x [128 rows][64 dh]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sQO + 4 * kBox128);
  uint64_t* q_full = bar;                  // Q / dO in TMEM (8 warp arrivals)
  uint64_t* k_full = bar + 1;              // [KS]
  uint64_t* k_empty = k_full + KS;         // [KS]
  uint64_t* v_full = k_empty + KS;         // [VS]
  uint64_t* v_empty = v_full + VS;         // [VS]
  uint64_t* s_full = v_empty + VS;         // [2]
  uint64_t* s_free = s_full + 2;           // [2]
  uint64_t* ds_full = s_free + 2;          // [2]
  uint64_t* ds_free = ds_full + 2;         // [2]
  uint64_t* dq_done = ds_free + 2;         // the item's last MMA completed
  uint64_t* dq_free = dq_done + 1;         // the item's dQ read out (8 warp arrivals)
  uint64_t* qo_tma = dq_free + 1;          // Q / dO landed in sQO
  uint64_t* qo_free = qo_tma + 1;          // sQO copied to TMEM (8 warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qo_free + 1);

  const int items = nq * a.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmQ);
    tma_prefetch(&tmO);
    mbar_init(q_full, 8);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&ds_full[i], 8);
      mbar_init(&ds_free[i], 1);
    }
    mbar_init(dq_done, 1);
    mbar_init(dq_free, 8);
    mbar_init(qo_tma, 1);
    mbar_init(qo_free, 8);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tQ = tmem + 256, tAq = tmem + 384, tAo = tmem + 448;

  if (warp == 8) {
    if (lane == 0) {
      auto load_qo = [&](int it) {
        AttnTile tl;
        AttnSeg sg;
        int h;
        item_of(a, nq, it, tl, sg, h);
        const int qrow = sg.q_start + tl.first;
        mbar_expect_tx(qo_tma, 4 * kBox128);
        tma_load_2d(sQO, &tmQ, qo_tma, h * DH, qrow);
        tma_load_2d(sQO + kBox128, &tmQ, qo_tma, h * DH + 64, qrow);
        tma_load_2d(sQO + 2 * kBox128, &tmO, qo_tma, h * DH, qrow);
        tma_load_2d(sQO + 3 * kBox128, &tmO, qo_tma, h * DH + 64, qrow);
      };
      if (blockIdx.x < items) load_qo(blockIdx.x);
      int jj = 0, n = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
        AttnTile tl;
        AttnSeg sg;
        int h;
        item_of(a, nq, item, tl, sg, h);
        const int g = h / (a.H / a.KVH);
        const int nkt = (sg.prefix + tl.first + tl.count + SUB - 1) / SUB;
        for (int j = 0; j < nkt; ++j, ++jj) {
          const int sk = jj % KS, sv = jj % VS;
          const int krow = sg.kv_row0 + j * SUB;
          stress_delay(a.stress, 1, jj);
          mbar_wait(&v_empty[sv], ((jj / VS) & 1) ^ 1);
          mbar_expect_tx(&v_full[sv], 2 * kBox64);
          tma_load_2d(sV + sv * 2 * kBox64, &tmV, &v_full[sv], g * DH, krow);
          tma_load_2d(sV + sv * 2 * kBox64 + kBox64, &tmV, &v_full[sv], g * DH + 64, krow);
          mbar_wait(&k_empty[sk], ((jj / KS) & 1) ^ 1);
          mbar_expect_tx(&k_full[sk], 2 * kBox64);
          tma_load_2d(sK + sk * 2 * kBox64, &tmK, &k_full[sk], g * DH, krow);
          tma_load_2d(sK + sk * 2 * kBox64 + kBox64, &tmK, &k_full[sk], g * DH + 64, krow);
        }
        // the next item's Q / dO, once this item's copy has left sQO
        if (item + static_cast<int>(gridDim.x) < items) {
          mbar_wait(qo_free, n & 1);
          load_qo(item + gridDim.x);
        }
      }
    }
  } else if (warp == 9) {
    constexpr uint32_t idS = umma_idesc_bf16(128, SUB, 0, 0);
    constexpr uint32_t idQ = umma_idesc_bf16(128, 128, 0, 1);
    const uint32_t sK0 = smem_u32(sK), sV0 = smem_u32(sV), sS0 = smem_u32(sS);
    const uint32_t bKf = smem_u32(k_full), bKe = smem_u32(k_empty), bVf = smem_u32(v_full),
                   bVe = smem_u32(v_empty), bSf = smem_u32(s_full), bSr = smem_u32(s_free),
                   bDf = smem_u32(ds_full), bDr = smem_u32(ds_free), bQf = smem_u32(q_full),
                   bQd = smem_u32(dq_done), bQr = smem_u32(dq_free);
    int ik = 0, iv = 0, ck = 0;
    uint32_t pk = 0, pv = 0;
    auto issue_s = [&](int J) {
      const uint32_t b = J & 1;
      mbar_wait_s(bKf + ik * 8, pk);
      mbar_wait_s(bVf + iv * 8, pv);
      mbar_wait_s(bSr + b * 8, ((J >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t k0 = sK0 + ik * 2 * kBox64, v0 = sV0 + iv * 2 * kBox64;
      umma4_ts_w<8, 2>(tmem + b * 64, tAq, kdesc(k0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tmem + b * 64, tAq + 32, kdesc(k0, kBox64, 4), idS, 1u);
      umma4_ts_w<8, 2>(tmem + 128 + b * 64, tAo, kdesc(v0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tmem + 128 + b * 64, tAo + 32, kdesc(v0, kBox64, 4), idS, 1u);
      umma_commit_w(bVe + iv * 8);
      umma_commit_w(bSf + b * 8);
      if (++ik == KS) { ik = 0; pk ^= 1; }
      if (++iv == VS) { iv = 0; pv ^= 1; }
    };
    int J0 = 0, n = 0;
    if (blockIdx.x < items) {
      mbar_wait_s(bQf, 0);
      tc_fence_after();
      issue_s(0);
    }
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
      AttnTile tl;
      AttnSeg sg;
      int h;
      item_of(a, nq, item, tl, sg, h);
      const int nkt = (sg.prefix + tl.first + tl.count + SUB - 1) / SUB;
      for (int j = 0; j < nkt; ++j) {
        const int J = J0 + j;
        stress_delay(a.stress, 2, J);
        if (j + 1 < nkt) {
          issue_s(J + 1);
        } else if (item + static_cast<int>(gridDim.x) < items) {
          mbar_wait_s(bQf, (n + 1) & 1);  // the next item's Q / dO are in TMEM
          tc_fence_after();
          issue_s(J + 1);
        }
        const uint32_t b = J & 1;
        mbar_wait_s(bDf + b * 8, (J >> 1) & 1);
        if (j == 0 && n > 0) mbar_wait_s(bQr, (n - 1) & 1);  // previous item's dQ read out
        tc_fence_after();
        const uint32_t s0 = sS0 + b * kBox128, k0 = sK0 + ck * 2 * kBox64;
        umma4_ss_w<2, 128>(tQ, kdesc(s0, kBox128, 0), mndesc(k0, kBox64, 0), idQ, j > 0 ? 1u : 0u);
        umma_commit_w(bKe + ck * 8);
        umma_commit_w(bDr + b * 8);
        if (++ck == KS) ck = 0;
      }
      umma_commit_w(bQd);
      J0 += nkt;
    }
  } else {
    const int quarter = warp & 3, half = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t bSf = smem_u32(s_full), bSr = smem_u32(s_free), bDf = smem_u32(ds_full),
                   bDr = smem_u32(ds_free), sS0 = smem_u32(sS), bQd = smem_u32(dq_done), bQr = smem_u32(dq_free),
                   sQO0 = smem_u32(sQO);
    uint32_t dst_off[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) dst_off[c] = sw_off(row, half * 4 + c);
    // sQO -> the Q / dO TMEM A operands (this warp's 32 rows, dh columns
    // [64 half, 64 half + 64) = box `half`, 128B-swizzled by row); returns
    // the item's LSE (log2 units) and D for this row
    auto copy_qo = [&](int it, uint32_t phase, float& lse2, float& D) {
      AttnTile tl;
      AttnSeg sg;
      int h;
      item_of(a, nq, it, tl, sg, h);
      const bool ok = tl.first + row < sg.len && row < tl.count;
      const int64_t r = static_cast<int64_t>(h) * a.T + sg.q_start + tl.first + row;
      lse2 = ok ? __ldg(a.lse + r) * kLog2e : 0.f;
      D = ok ? __ldg(a.dsum + r) : 0.f;
      mbar_wait(qo_tma, phase);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint32_t base = sQO0 + (2 * t + half) * kBox128 + row * 128;
        uint32_t w[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 x = lds128(base + ((c ^ (row & 7)) << 4));
          w[4 * c] = x.x, w[4 * c + 1] = x.y, w[4 * c + 2] = x.z, w[4 * c + 3] = x.w;
        }
        tmem_st32w((t ? tAo : tAq) + lane_off + half * 32, w);
      }
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(q_full);
      warp_arrive(qo_free);
    };
    int J0 = 0, n = 0;
    float lse2 = 0.f, D = 0.f, lse2n = 0.f, Dn = 0.f;
    if (blockIdx.x < items) copy_qo(blockIdx.x, 0, lse2, D);
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
      AttnTile tl;
      AttnSeg sg;
      int h;
      item_of(a, nq, item, tl, sg, h);
      const int q_row0 = sg.q_start + tl.first;
      const int nkt = (sg.prefix + tl.first + tl.count + SUB - 1) / SUB;
      const int qi = tl.first + row;
      const bool ok = qi < sg.len && row < tl.count;
      const int lim = sg.prefix + min(qi, sg.len - 1);
      const int klim = ok ? lim : -1;
      const int tile_lim = sg.prefix + tl.first;
      const bool next = item + static_cast<int>(gridDim.x) < items;
      const float2 sl2v = make_float2(a.sl2, a.sl2), nl = make_float2(-lse2, -lse2), nD = make_float2(-D, -D);
      for (int j = 0; j < nkt; ++j) {
        const int J = J0 + j;
        const uint32_t b = J & 1;
        mbar_wait_s(bSf + b * 8, (J >> 1) & 1);
        tc_fence_after();
        // the item's last S / dP completed: Q / dO TMEM free for the next item
        if (j + 1 == nkt && next) copy_qo(item + gridDim.x, (n + 1) & 1, lse2n, Dn);
        uint32_t rs[32], rp[32];
        tmem_ld32(tmem + b * 64 + lane_off + half * 32, rs);
        tmem_ld32(tmem + 128 + b * 64 + lane_off + half * 32, rp);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive_s(bSr + b * 8);
        uint32_t pk[16];
        auto body = [&](auto masked) {
          const int key0 = j * SUB + half * 32;
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 x = ffma2(make_float2(__uint_as_float(rs[2 * e]), __uint_as_float(rs[2 * e + 1])), sl2v, nl);
            float2 p = make_float2(ex2(x.x), ex2(x.y));
            if constexpr (decltype(masked)::value) {
              p.x = key0 + 2 * e <= klim ? p.x : 0.f;
              p.y = key0 + 2 * e + 1 <= klim ? p.y : 0.f;
            }
            const float2 ds =
                fmul2(p, fadd2(make_float2(__uint_as_float(rp[2 * e]), __uint_as_float(rp[2 * e + 1])), nD));
            pk[e] = pack_bf16(ds.x, ds.y);
          }
        };
        if (j * SUB + SUB - 1 <= tile_lim)
          body(std::false_type{});
        else
          body(std::true_type{});
        stress_delay(a.stress, 3, J);
        if (J >= 2) mbar_wait_s(bDr + b * 8, ((J >> 1) & 1) ^ 1);
        const uint32_t dst = sS0 + b * kBox128;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          sts128(dst + dst_off[c], make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
        fence_async_smem();
        warp_arrive_s(bDf + b * 8);
      }
      J0 += nkt;
      mbar_wait_s(bQd, n & 1);  // every MMA of this item done: dQ settled
      tc_fence_after();
      __nv_bfloat16* out = a.dq + static_cast<int64_t>(q_row0 + row) * a.dq_stride + h * DH;
      if (a.rope_tab) {
        uint32_t ra[32], rb[32];
        tmem_ld32(tQ + lane_off + half * 32, ra);
        tmem_ld32(tQ + lane_off + (half + 2) * 32, rb);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive_s(bQr);
        if (ok) {
          float fa[32], fb[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            fa[e] = bf16_round(__uint_as_float(ra[e]) * a.scale);
            fb[e] = bf16_round(__uint_as_float(rb[e]) * a.scale);
          }
          rope_inverse32(a.rope_tab + static_cast<int64_t>(q_row0 + row) * (DH / 2) + half * 32, fa, fb);
          store_bf16x32(out + half * 32, fa);
          store_bf16x32(out + (half + 2) * 32, fb);
        }
      } else {
        uint32_t r0[32], r1[32];
        tmem_ld32(tQ + lane_off + (half * 2) * 32, r0);
        tmem_ld32(tQ + lane_off + (half * 2 + 1) * 32, r1);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive_s(bQr);
        if (ok) {
          const float sc = a.scale;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const uint32_t* rr = cc ? r1 : r0;
            uint4* d4 = reinterpret_cast<uint4*>(out + (half * 2 + cc) * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              d4[q] = make_uint4(pack_bf16(__uint_as_float(rr[8 * q]) * sc, __uint_as_float(rr[8 * q + 1]) * sc),
                                 pack_bf16(__uint_as_float(rr[8 * q + 2]) * sc, __uint_as_float(rr[8 * q + 3]) * sc),
                                 pack_bf16(__uint_as_float(rr[8 * q + 4]) * sc, __uint_as_float(rr[8 * q + 5]) * sc),
                                 pack_bf16(__uint_as_float(rr[8 * q + 6]) * sc, __uint_as_float(rr[8 * q + 7]) * sc));
          }
        }
      }
      lse2 = lse2n;
      D = Dn;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// D = rowsum(dO * O) per (q head, row) for dq_persist_tma_kernel and the
// dK/dV kernel: one 256-thread CTA per row, 16-byte coalesced reads, each
// head's 16 chunks reduced across a half-warp in a fixed order.  HBM-bound:
// 4 bytes read per element of dO and O.
__global__ void __launch_bounds__(256) dsum_rows_kernel(Args a) {
  const int t = blockIdx.x, lane = threadIdx.x & 31;
  const int chunks = a.H * (DH / 8);
  const uint4* d4 = reinterpret_cast<const uint4*>(a.dout + static_cast<int64_t>(t) * a.dout_stride);
  const uint4* o4 = reinterpret_cast<const uint4*>(a.o + static_cast<int64_t>(t) * a.o_stride);
  // whole warps iterate together (the shuffles need every lane)
  for (int k0 = threadIdx.x - lane; k0 < chunks; k0 += blockDim.x) {
    const int k = k0 + lane;
    float acc = 0.f;
    if (k < chunks) {
      const uint4 dv = __ldg(d4 + k), ov = __ldg(o4 + k);
      const uint32_t dw[4] = {dv.x, dv.y, dv.z, dv.w}, ow[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&dw[e]);
        const __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(&ow[e]);
        acc = fmaf(__low2float(x), __low2float(y), acc);
        acc = fmaf(__high2float(x), __high2float(y), acc);
      }
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (k < chunks && (k & 15) == 0) a.dsum[static_cast<int64_t>(k >> 4) * a.T + t] = acc;
  }
}

// ------------------------------------------------------------- dQ, wide
// CTA = 128 queries x one q head, keys streamed in 128-key tiles so the S /
// dP MMAs are N = 128 (a tcgen05.mma with N <= 64 pays a ~45-cycle floor,
// profiles/round2_mma_probe.txt).  TMEM: S [0,128) dP [128,256) dQ
// [256,384) Q [384,448) dO [448,512) — S / dP single-buffered; the MMA
// issuer covers their read-out with the previous tile's dQ GEMM:
//   S(j) dP(j) | dQ(j-1) | S(j+1) dP(j+1) | dQ(j) | ...
// 16 softmax warps: lane quarter (warp & 3) x 32-key column quarter (warp >> 2).
constexpr int kWKS = 3, kWVS = 2;        // K / V ring depths (128-key tiles)
constexpr int kDqWideThreads = 576;      // 16 softmax warps + TMA + MMA
__global__ void __launch_bounds__(kDqWideThreads, 1)
    dq_wide_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;                            // kWKS x 2 x [128][64]
  uint8_t* sV = sK + kWKS * 2 * kBox128;       // kWVS x 2 x [128][64]
  uint8_t* sS = sV + kWVS * 2 * kBox128;       // 2 x 2 x [128 q][64 keys] (dS)
  float* sRowD = reinterpret_cast<float*>(sS); // [4][128] D partials, before dS(0) exists
  uint64_t* bar = reinterpret_cast<uint64_t*>(sS + 4 * kBox128);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;              // [kWKS]
  uint64_t* k_empty = k_full + kWKS;       // [kWKS]
  uint64_t* v_full = k_empty + kWKS;       // [kWVS]
  uint64_t* v_empty = v_full + kWVS;       // [kWVS]
  uint64_t* s_full = v_empty + kWVS;
  uint64_t* s_free = s_full + 1;
  uint64_t* ds_full = s_free + 1;          // [2]
  uint64_t* ds_free = ds_full + 2;         // [2]
  uint64_t* dq_done = ds_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);

  const AttnTile tl = a.tiles[blockIdx.x];
  const AttnSeg sg = a.segs[tl.seg];
  const int h = blockIdx.y, g = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_row0 = sg.q_start + tl.first;
  const int kv_len = sg.prefix + tl.first + tl.count;
  const int nkt = (kv_len + 127) / 128;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 16);
    for (int i = 0; i < kWKS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kWVS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 16);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ds_full[i], 16);
      mbar_init(&ds_free[i], 1);
    }
    mbar_init(dq_done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256, tAq = tmem + 384, tAo = tmem + 448;

  if (warp == 16) {
    if (lane == 0) {
      for (int j = 0; j < nkt; ++j) {
        const int sk = j % kWKS, sv = j % kWVS;
        const int krow = sg.kv_row0 + j * 128;
        stress_delay(a.stress, 1, j);
        mbar_wait(&v_empty[sv], ((j / kWVS) & 1) ^ 1);
        mbar_expect_tx(&v_full[sv], 2 * kBox128);
        tma_load_2d(sV + sv * 2 * kBox128, &tmV, &v_full[sv], g * DH, krow);
        tma_load_2d(sV + sv * 2 * kBox128 + kBox128, &tmV, &v_full[sv], g * DH + 64, krow);
        mbar_wait(&k_empty[sk], ((j / kWKS) & 1) ^ 1);
        mbar_expect_tx(&k_full[sk], 2 * kBox128);
        tma_load_2d(sK + sk * 2 * kBox128, &tmK, &k_full[sk], g * DH, krow);
        tma_load_2d(sK + sk * 2 * kBox128 + kBox128, &tmK, &k_full[sk], g * DH + 64, krow);
      }
    }
  } else if (warp == 17) {
    // whole warp, convergent (elect.sync inside the issue helpers)
    constexpr uint32_t idS = umma_idesc_bf16(128, 128, 0, 0);  // S, dP: N = 128 keys
    constexpr uint32_t idQ = umma_idesc_bf16(128, 128, 0, 1);  // dQ: N = dh, B = K (MN-major view)
    const uint32_t sK0 = smem_u32(sK), sV0 = smem_u32(sV), sS0 = smem_u32(sS);
    const uint32_t bKf = smem_u32(k_full), bKe = smem_u32(k_empty), bVf = smem_u32(v_full),
                   bVe = smem_u32(v_empty), bSf = smem_u32(s_full), bSr = smem_u32(s_free),
                   bDf = smem_u32(ds_full), bDr = smem_u32(ds_free), bQd = smem_u32(dq_done);
    auto issue_s = [&](int j) {
      const int sk = j % kWKS, sv = j % kWVS;
      mbar_wait_s(bKf + sk * 8, (j / kWKS) & 1);
      mbar_wait_s(bVf + sv * 8, (j / kWVS) & 1);
      tc_fence_after();
      const uint32_t k0 = sK0 + sk * 2 * kBox128, v0 = sV0 + sv * 2 * kBox128;
      umma4_ts_w<8, 2>(tS, tAq, kdesc(k0, kBox128, 0), idS, 0u);
      umma4_ts_w<8, 2>(tS, tAq + 32, kdesc(k0, kBox128, 4), idS, 1u);
      umma4_ts_w<8, 2>(tP, tAo, kdesc(v0, kBox128, 0), idS, 0u);
      umma4_ts_w<8, 2>(tP, tAo + 32, kdesc(v0, kBox128, 4), idS, 1u);
      umma_commit_w(bVe + sv * 8);
      umma_commit_w(bSf);
    };
    auto issue_dq = [&](int j) {
      const uint32_t b = j & 1;
      mbar_wait_s(bDf + b * 8, (j >> 1) & 1);
      tc_fence_after();
      const uint32_t s0 = sS0 + b * 2 * kBox128, k0 = sK0 + (j % kWKS) * 2 * kBox128;
      // dQ += dS K: K = 128 keys in two 64-key boxes of dS (4 MMAs each)
      umma4_ss_w<2, 128>(tQ, kdesc(s0, kBox128, 0), mndesc(k0, kBox128, 0), idQ, j > 0 ? 1u : 0u);
      umma4_ss_w<2, 128>(tQ, kdesc(s0, kBox128, 4), mndesc(k0, kBox128, 4), idQ, 1u);
      umma_commit_w(bKe + (j % kWKS) * 8);
      umma_commit_w(bDr + b * 8);
    };
    mbar_wait(q_full, 0);  // Q / dO staged into TMEM by the softmax warps
    tc_fence_after();
    issue_s(0);
    for (int j = 0; j < nkt; ++j) {
      stress_delay(a.stress, 2, j);
      if (j >= 1) issue_dq(j - 1);
      if (j + 1 < nkt) {
        mbar_wait_s(bSr, j & 1);  // S(j) / dP(j) read out: the columns are free
        tc_fence_after();
        issue_s(j + 1);
      }
    }
    issue_dq(nkt - 1);
    umma_commit_w(bQd);
  } else {
    const int quarter = warp & 3, cq = warp >> 2;  // TMEM lane quarter, 32-key column quarter
    const int row = quarter * 32 + lane;
    const int qi = tl.first + row;
    const bool ok = qi < sg.len && row < tl.count;
    const int lim = sg.prefix + min(qi, sg.len - 1);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float lse2 = ok ? a.lse[static_cast<int64_t>(h) * a.T + q_row0 + row] * kLog2e : 0.f;
    float D;
    {
      // this warp stages dh columns [32 cq, 32 cq + 32) of Q and dO (16 TMEM
      // columns each) and the matching part of D = rowsum(dO * O)
      const bool rok = row < tl.count;
      const int64_t r = q_row0 + row;
      stage_row_tmem16(tAq + lane_off + cq * 16, a.q + r * a.q_stride + static_cast<int64_t>(h) * DH + cq * 32, rok);
      stage_row_tmem16(tAo + lane_off + cq * 16, a.dout + r * a.dout_stride + static_cast<int64_t>(h) * DH + cq * 32,
                       ok);
      float dpart = 0.f;
      if (ok) {
        const uint4* d4 = reinterpret_cast<const uint4*>(a.dout + r * a.dout_stride + static_cast<int64_t>(h) * DH + cq * 32);
        const uint4* o4 = reinterpret_cast<const uint4*>(a.o + r * a.o_stride + static_cast<int64_t>(h) * DH + cq * 32);
        float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 dv = __ldg(d4 + c), ov = __ldg(o4 + c);
          const uint32_t dw[4] = {dv.x, dv.y, dv.z, dv.w}, ow[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __nv_bfloat162 a2 = *reinterpret_cast<const __nv_bfloat162*>(&dw[e]);
            const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&ow[e]);
            part[e] = fmaf(__low2float(a2), __low2float(b2), part[e]);
            part[e] = fmaf(__high2float(a2), __high2float(b2), part[e]);
          }
        }
        dpart = (part[0] + part[1]) + (part[2] + part[3]);
      }
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(q_full);
      // the four column quarters of a row meet in smem (fixed order)
      sRowD[cq * 128 + row] = dpart;
      asm volatile("bar.sync %0, 128;" ::"r"(1 + quarter) : "memory");
      D = (sRowD[row] + sRowD[128 + row]) + (sRowD[256 + row] + sRowD[384 + row]);
      if (ok && cq == 0) a.dsum[static_cast<int64_t>(h) * a.T + q_row0 + row] = D;
    }
    const uint32_t bSf = smem_u32(s_full), bSr = smem_u32(s_free), bDf = smem_u32(ds_full),
                   bDr = smem_u32(ds_free), sS0 = smem_u32(sS);
    const int klim = ok ? lim : -1;
    const int tile_lim = sg.prefix + tl.first;
    // dS row `row`, keys [32 cq, 32 cq + 32): box cq >> 1, 16-byte chunks
    // 4 (cq & 1) .. 4 (cq & 1) + 3
    uint32_t dst_off[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) dst_off[c] = (cq >> 1) * kBox128 + sw_off(row, (cq & 1) * 4 + c);
    const float2 sl2v = make_float2(a.sl2, a.sl2), nl = make_float2(-lse2, -lse2), nD = make_float2(-D, -D);
    // the D exchange above used the dS buffers' memory: every softmax warp
    // is past it before any dS store
    asm volatile("bar.sync %0, 512;" ::"r"(5) : "memory");
    for (int j = 0; j < nkt; ++j) {
      const uint32_t b = j & 1;
      mbar_wait_s(bSf, j & 1);
      tc_fence_after();
      uint32_t rs[32], rp[32];
      tmem_ld32(tS + lane_off + cq * 32, rs);
      tmem_ld32(tP + lane_off + cq * 32, rp);
      tmem_ld_wait();
      tc_fence_before();
      warp_arrive_s(bSr);
      uint32_t pk[16];
      auto body = [&](auto masked) {
        const int key0 = j * 128 + cq * 32;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = ffma2(make_float2(__uint_as_float(rs[2 * e]), __uint_as_float(rs[2 * e + 1])), sl2v, nl);
          float2 p = make_float2(ex2(x.x), ex2(x.y));
          if constexpr (decltype(masked)::value) {
            p.x = key0 + 2 * e <= klim ? p.x : 0.f;
            p.y = key0 + 2 * e + 1 <= klim ? p.y : 0.f;
          }
          const float2 ds =
              fmul2(p, fadd2(make_float2(__uint_as_float(rp[2 * e]), __uint_as_float(rp[2 * e + 1])), nD));
          pk[e] = pack_bf16(ds.x, ds.y);
        }
      };
      if (j * 128 + 127 <= tile_lim)
        body(std::false_type{});
      else
        body(std::true_type{});
      stress_delay(a.stress, 3, j);
      if (j >= 2) mbar_wait_s(bDr + b * 8, ((j >> 1) & 1) ^ 1);
      const uint32_t dst = sS0 + b * 2 * kBox128;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        sts128(dst + dst_off[c], make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]));
      fence_async_smem();
      warp_arrive_s(bDf + b * 8);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    __nv_bfloat16* out = a.dq + static_cast<int64_t>(q_row0 + row) * a.dq_stride + h * DH;
    if (a.rope_tab) {  // column quarters 0, 1 take rotate-half partner chunks (cq, cq + 2)
      if (cq < 2) {
        uint32_t ra[32], rb[32];
        tmem_ld32(tQ + lane_off + cq * 32, ra);
        tmem_ld32(tQ + lane_off + (cq + 2) * 32, rb);
        tmem_ld_wait();
        if (ok) {
          float fa[32], fb[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            fa[e] = bf16_round(__uint_as_float(ra[e]) * a.scale);
            fb[e] = bf16_round(__uint_as_float(rb[e]) * a.scale);
          }
          rope_inverse32(a.rope_tab + static_cast<int64_t>(q_row0 + row) * (DH / 2) + cq * 32, fa, fb);
          store_bf16x32(out + cq * 32, fa);
          store_bf16x32(out + (cq + 2) * 32, fb);
        }
      }
    } else {
      uint32_t r[32];
      tmem_ld32(tQ + lane_off + cq * 32, r);
      tmem_ld_wait();
      if (ok) {
        uint4* d4 = reinterpret_cast<uint4*>(out + cq * 32);
        const float sc = a.scale;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          d4[q] = make_uint4(pack_bf16(__uint_as_float(r[8 * q]) * sc, __uint_as_float(r[8 * q + 1]) * sc),
                             pack_bf16(__uint_as_float(r[8 * q + 2]) * sc, __uint_as_float(r[8 * q + 3]) * sc),
                             pack_bf16(__uint_as_float(r[8 * q + 4]) * sc, __uint_as_float(r[8 * q + 5]) * sc),
                             pack_bf16(__uint_as_float(r[8 * q + 6]) * sc, __uint_as_float(r[8 * q + 7]) * sc));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// ------------------------------------------------------------- dK / dV
// CTA = 128 keys x one kv head (sole owner of those rows); queries streamed
// in 64-query sub-tiles over every q head of the GQA group.
__global__ void __launch_bounds__(kDkvThreads, 1)
    dkv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // K and V (per-CTA invariant A operands of S^T and dP^T) live in TMEM;
  // S^T / dP^T are single-buffered (their readers release them right after
  // tcgen05.ld), which leaves room for K, V next to the dV / dK accumulators.
  uint8_t* sQ = sm;                      // QS stages x 2 x [64][64]
  uint8_t* sdO = sQ + QS * 2 * kBox64;   // QS stages x 2 x [64][64]
  uint8_t* sP = sdO + QS * 2 * kBox64;   // 2 x [128 keys][64 q]
  uint8_t* sS = sP + 2 * kBox128;        // 2 x [128 keys][64 q]
  uint8_t* sLD = sS + 2 * kBox128;       // QS stages x {LSE[64], D[64]} fp32 (staged with Q / dO)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sLD + QS * 512);
  uint64_t* kv_full = bar;               // K / V staged into TMEM (256 arrivals)
  uint64_t* q_full = bar + 1;            // [QS]
  uint64_t* q_empty = q_full + QS;       // [QS]
  uint64_t* s_full = q_empty + QS;       // [1]
  uint64_t* s_free = s_full + 1;         // [1]
  uint64_t* pds_full = s_free + 1;       // [2]
  uint64_t* pds_free = pds_full + 2;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pds_free + 2);

  const AttnTile tl = a.tiles[blockIdx.x];
  const AttnSeg sg = a.segs[tl.seg];
  const int g = blockIdx.y, per = a.H / a.KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int key_first = tl.first;
  const int kv_len = sg.prefix + sg.len;
  const int i0 = max(0, key_first - sg.prefix);
  const int nqt = (sg.len - i0 + SUB - 1) / SUB;
  const int iters = per * nqt;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmO);
    mbar_init(kv_full, 16);  // one arrive per softmax-side warp
    for (int i = 0; i < QS; ++i) {
      mbar_init(&q_full[i], 2);  // TMA expect_tx arrive + LSE / D staged arrive
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 16);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pds_full[i], 16);
      mbar_init(&pds_free[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 64;  // S^T, dP^T (64 columns each)
  const uint32_t tdV = tmem + 128, tdK = tmem + 256;
  const uint32_t tAk = tmem + 384, tAv = tmem + 448;  // K, V A operands (64 columns each)
  const uint32_t sQ0 = smem_u32(sQ), sO0 = smem_u32(sdO), sP0 = smem_u32(sP), sS0 = smem_u32(sS),
                 sLD0 = smem_u32(sLD);
  const uint32_t bQf = smem_u32(q_full), bQe = smem_u32(q_empty), bSf = smem_u32(s_full),
                 bSr = smem_u32(s_free), bPf = smem_u32(pds_full), bPr = smem_u32(pds_free);

  if (warp == 16) {
    // whole warp: lane 0 issues the Q / dO TMA, every lane stages two of the
    // 64 LSE / D values (plain loads: segment starts are not 16B-aligned)
    int qs = 0, hi = 0, qi = 0;  // ring slot, q head within the group, query sub-tile
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      const int hq = g * per + hi;
      const int qt0 = i0 + qi * SUB;
      const int qrow = sg.q_start + qt0;
      stress_delay(a.stress, 4, it);
      mbar_wait_s(bQe + qs * 8, ph ^ 1);
      if (lane == 0) {
        mbar_expect_tx(&q_full[qs], TMA_TX(4 * kBox64));
        uint8_t* q = sQ + qs * 2 * kBox64;
        uint8_t* o = sdO + qs * 2 * kBox64;
        TMA_A(q, &tmQ, &q_full[qs], hq * DH, qrow);
        TMA_B(q + kBox64, &tmQ, &q_full[qs], hq * DH + 64, qrow);
        TMA_A(o, &tmO, &q_full[qs], hq * DH, qrow);
        TMA_B(o + kBox64, &tmO, &q_full[qs], hq * DH + 64, qrow);
      }
      const int64_t base = static_cast<int64_t>(hq) * a.T + qrow;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int c = lane + 32 * h2;
        const bool in = qt0 + c < sg.len;  // past the segment: masked by the consumer
        sts_f32(sLD0 + qs * 512 + c * 4, in ? __ldg(a.lse + base + c) : 0.f);
        sts_f32(sLD0 + qs * 512 + 256 + c * 4, in ? __ldg(a.dsum + base + c) : 0.f);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_s(bQf + qs * 8);
      if (++qi == nqt) { qi = 0; ++hi; }
      if (++qs == QS) { qs = 0; ph ^= 1; }
    }
  } else if (warp == 17) {
    // whole warp, convergent (elect.sync inside the issue helpers)
    constexpr uint32_t idS = umma_idesc_bf16(128, SUB, 0, 0);  // S^T, dP^T: N = 64 queries
    constexpr uint32_t idG = umma_idesc_bf16(128, 128, 0, 1);  // dV, dK: N = dh, B MN-major view
    int is = 0, cs = 0;  // ring slot of the next S^T issue / of the next dV,dK issue
    uint32_t ps = 0;
    auto issue_s = [&](int it) {
      mbar_wait_s(bQf + is * 8, ps);
      mbar_wait_s(bSr, (it & 1) ^ 1);
      tc_fence_after();
      const uint32_t q0 = sQ0 + is * 2 * kBox64, o0 = sO0 + is * 2 * kBox64;
      umma4_ts_w<8, 2>(tS, tAk, kdesc(q0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tS, tAk + 32, kdesc(q0, kBox64, 4), idS, 1u);
      umma4_ts_w<8, 2>(tP, tAv, kdesc(o0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tP, tAv + 32, kdesc(o0, kBox64, 4), idS, 1u);
      umma_commit_w(bSf);
      if (++is == QS) { is = 0; ps ^= 1; }
    };
    mbar_wait(kv_full, 0);
    tc_fence_after();
    issue_s(0);
    for (int it = 0; it < iters; ++it) {
      stress_delay(a.stress, 5, it);
      if (it + 1 < iters) issue_s(it + 1);
      const uint32_t b = it & 1;
      mbar_wait_s(bPf + b * 8, (it >> 1) & 1);
      tc_fence_after();
      const uint32_t q0 = sQ0 + cs * 2 * kBox64, o0 = sO0 + cs * 2 * kBox64;
      const uint32_t p0 = sP0 + b * kBox128, s0 = sS0 + b * kBox128;
#if CF_BWD_DIAG < 3
      umma4_ss_w<2, 128>(tdV, kdesc(p0, kBox128, 0), mndesc(o0, kBox64, 0), idG, it > 0 ? 1u : 0u);
      umma4_ss_w<2, 128>(tdK, kdesc(s0, kBox128, 0), mndesc(q0, kBox64, 0), idG, it > 0 ? 1u : 0u);
#endif
      umma_commit_w(bQe + cs * 8);
      umma_commit_w(bPr + b * 8);
      if (++cs == QS) cs = 0;
    }
  } else {
    const int quarter = warp & 3, part = warp >> 2;  // part: which 16 of the 64 query columns
    const int row = quarter * 32 + lane;                // key row within the tile
    const int key = key_first + row;
    const bool kok = row < tl.count && key < kv_len;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    {
      // K and V quarter-rows, read coalesced through a per-warp scratch in
      // the P / dS buffers (unused until the first S^T completes)
      const int valid = min(tl.count, kv_len - key_first) - quarter * 32;
      const int64_t r0 = sg.kv_row0 + key_first + quarter * 32;
      const int64_t off = r0 * a.kv_stride + static_cast<int64_t>(g) * DH + part * 32;
      const uint32_t scr = smem_u32(sP) + warp * 2048;
      uint4 xk[4], xv[4];
      rows_to_lanes64(scr, a.k + off, a.kv_stride, valid, xk);
      rows_to_lanes64(scr, a.v + off, a.kv_stride, valid, xv);
      uint32_t wk[16], wv[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        wk[4 * c] = xk[c].x, wk[4 * c + 1] = xk[c].y, wk[4 * c + 2] = xk[c].z, wk[4 * c + 3] = xk[c].w;
        wv[4 * c] = xv[c].x, wv[4 * c + 1] = xv[c].y, wv[4 * c + 2] = xv[c].z, wv[4 * c + 3] = xv[c].w;
      }
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tAk + lane_off + part * 16),
          "r"(wk[0]), "r"(wk[1]), "r"(wk[2]), "r"(wk[3]), "r"(wk[4]), "r"(wk[5]), "r"(wk[6]), "r"(wk[7]), "r"(wk[8]),
          "r"(wk[9]), "r"(wk[10]), "r"(wk[11]), "r"(wk[12]), "r"(wk[13]), "r"(wk[14]), "r"(wk[15])
          : "memory");
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tAv + lane_off + part * 16),
          "r"(wv[0]), "r"(wv[1]), "r"(wv[2]), "r"(wv[3]), "r"(wv[4]), "r"(wv[5]), "r"(wv[6]), "r"(wv[7]), "r"(wv[8]),
          "r"(wv[9]), "r"(wv[10]), "r"(wv[11]), "r"(wv[12]), "r"(wv[13]), "r"(wv[14]), "r"(wv[15])
          : "memory");
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(kv_full);
    }
    // query index range this key row sees: [qlo, len) (qlo = INT_MAX: row absent)
    const int qlo = kok ? key - sg.prefix : INT_MAX;
    uint32_t dst_off[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) dst_off[c] = sw_off(row, part * 2 + c);
    int qs = 0, qi = 0;
    uint32_t qph = 0;
    for (int it = 0; it < iters; ++it) {
      const uint32_t b = it & 1;
      const int qt0 = i0 + qi * SUB;
      mbar_wait_s(bSf, it & 1);
      tc_fence_after();
#if CF_BWD_DIAG >= 2
      warp_arrive_s(bSr);
      if (it >= 2) mbar_wait_s(bPr + b * 8, ((it >> 1) & 1) ^ 1);
      warp_arrive_s(bPf + b * 8);
      if (++qi == nqt) qi = 0;
      if (++qs == QS) { qs = 0; qph ^= 1; }
      continue;
#endif
      uint32_t rs[16], rp[16];
      tmem_ld16(tS + lane_off + part * 16, rs);
      tmem_ld16(tP + lane_off + part * 16, rp);
      tmem_ld_wait();
      tc_fence_before();
      warp_arrive_s(bSr);
      stress_delay(a.stress, 6, it);
      mbar_wait_s(bQf + qs * 8, qph);  // LSE / D of this slot (already complete: S^T waited on it)
      const uint32_t lrow = sLD0 + qs * 512 + part * 64;
      uint32_t pp[8], pd[8];
      auto body = [&](auto masked) {
        // pairs in FFMA2 / FADD2 / FMUL2: x = s * sl2 - LSE * log2e,
        // dS = P (dP - D), per-column LSE / D
        const float2 sl2v = make_float2(a.sl2, a.sl2), nlg = make_float2(-kLog2e, -kLog2e),
                     m1 = make_float2(-1.f, -1.f);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const float4 L = lds_f32x4(lrow + c4 * 16);
          const float4 Dv = lds_f32x4(lrow + 256 + c4 * 16);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int col = c4 * 4 + 2 * h2;
            const float2 nl = fmul2(h2 ? make_float2(L.z, L.w) : make_float2(L.x, L.y), nlg);
            const float2 nd = fmul2(h2 ? make_float2(Dv.z, Dv.w) : make_float2(Dv.x, Dv.y), m1);
            const float2 x = ffma2(make_float2(__uint_as_float(rs[col]), __uint_as_float(rs[col + 1])), sl2v, nl);
            float2 p = make_float2(ex2(x.x), ex2(x.y));
            float2 ds = fmul2(p, fadd2(make_float2(__uint_as_float(rp[col]), __uint_as_float(rp[col + 1])), nd));
            if constexpr (decltype(masked)::value) {
              // masked entries are selected away (never multiplied), so
              // whatever LSE / D a slot holds past the segment cannot leak
              const int qq = qt0 + part * 16 + col;
              const bool in0 = qq >= qlo && qq < sg.len, in1 = qq + 1 >= qlo && qq + 1 < sg.len;
              p = make_float2(in0 ? p.x : 0.f, in1 ? p.y : 0.f);
              ds = make_float2(in0 ? ds.x : 0.f, in1 ? ds.y : 0.f);
            }
            pp[2 * c4 + h2] = pack_bf16(p.x, p.y);
            pd[2 * c4 + h2] = pack_bf16(ds.x, ds.y);
          }
        }
      };
      // uniform: every key of the tile sees every query of the sub-tile
#if CF_BWD_DIAG == 1
      for (int e = 0; e < 8; ++e) { pp[e] = rs[e] ^ rp[e]; pd[e] = rs[e + 8] ^ rp[e + 8]; }
#else
      if (key_first + 127 < kv_len && key_first + 127 <= sg.prefix + qt0 && qt0 + SUB <= sg.len)
        body(std::false_type{});
      else
        body(std::true_type{});
#endif
      stress_delay(a.stress, 7, it);
      if (it >= 2) mbar_wait_s(bPr + b * 8, ((it >> 1) & 1) ^ 1);
      const uint32_t dP_ = sP0 + b * kBox128, dS_ = sS0 + b * kBox128;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        sts128(dP_ + dst_off[c], make_uint4(pp[4 * c], pp[4 * c + 1], pp[4 * c + 2], pp[4 * c + 3]));
        sts128(dS_ + dst_off[c], make_uint4(pd[4 * c], pd[4 * c + 1], pd[4 * c + 2], pd[4 * c + 3]));
      }
      fence_async_smem();
      warp_arrive_s(bPf + b * 8);
      if (++qi == nqt) qi = 0;
      if (++qs == QS) { qs = 0; qph ^= 1; }
    }
    const int last = iters - 1;
    mbar_wait(&pds_free[last & 1], (last >> 1) & 1);
    tc_fence_after();
    if (a.dkv_out) {
      // parts 0, 1: dK chunks (part, part + 2), rotated back; parts 2, 3: dV
      // chunks (part - 2, part); bf16 straight into dq|dk|dv
      const bool is_k = part < 2;
      const int c0 = part & 1;
      uint32_t ra[32], rb[32];
      tmem_ld32((is_k ? tdK : tdV) + lane_off + c0 * 32, ra);
      tmem_ld32((is_k ? tdK : tdV) + lane_off + (c0 + 2) * 32, rb);
      tmem_ld_wait();
      if (kok) {
        const int64_t r = sg.kv_row0 + key;
        float fa[32], fb[32];
        const float sc = is_k ? a.scale : 1.f;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          fa[e] = __uint_as_float(ra[e]) * sc;
          fb[e] = __uint_as_float(rb[e]) * sc;
        }
        if (is_k && a.rope_tab) rope_inverse32(a.rope_tab + r * (DH / 2) + c0 * 32, fa, fb);
        __nv_bfloat16* dst = a.dkv_out + r * a.dkv_out_ld + (is_k ? a.col_k : a.col_v) + g * DH;
        store_bf16x32(dst + c0 * 32, fa);
        store_bf16x32(dst + (c0 + 2) * 32, fb);
      }
    } else {
    float* dkr = a.dk_acc + static_cast<int64_t>(sg.kv_row0 + key) * a.acc_stride + g * DH;
    float* dvr = a.dv_acc + static_cast<int64_t>(sg.kv_row0 + key) * a.acc_stride + g * DH;
    {
      const int c = part;  // 32-column chunk of dK / dV
      uint32_t rk[32], rv[32];
      tmem_ld32(tdK + lane_off + c * 32, rk);
      tmem_ld32(tdV + lane_off + c * 32, rv);
      tmem_ld_wait();
      if (kok) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 k4 = reinterpret_cast<float4*>(dkr + c * 32)[q];
          k4.x += __uint_as_float(rk[4 * q]) * a.scale;
          k4.y += __uint_as_float(rk[4 * q + 1]) * a.scale;
          k4.z += __uint_as_float(rk[4 * q + 2]) * a.scale;
          k4.w += __uint_as_float(rk[4 * q + 3]) * a.scale;
          reinterpret_cast<float4*>(dkr + c * 32)[q] = k4;
          float4 v4 = reinterpret_cast<float4*>(dvr + c * 32)[q];
          v4.x += __uint_as_float(rv[4 * q]);
          v4.y += __uint_as_float(rv[4 * q + 1]);
          v4.z += __uint_as_float(rv[4 * q + 2]);
          v4.w += __uint_as_float(rv[4 * q + 3]);
          reinterpret_cast<float4*>(dvr + c * 32)[q] = v4;
        }
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// The item a persistent CTA takes in round r: boustrophedon order over the
// grid (even rounds ascending, odd rounds descending), so with items sorted
// by decreasing work each CTA's total stays close to the mean (plain
// round-robin hands CTA 0 the heaviest item of every round).
__device__ __forceinline__ int snake_item(int r) {
  const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
  return r * G + ((r & 1) ? G - 1 - b : b);
}
// -------------------------------------------------- dK / dV, persistent
// dkv_kernel's math with one CTA per SM looping over (128-key tile, kv head)
// items (item = blockIdx.x + k * gridDim.x, tile-major: heaviest tiles
// first).  Ring positions and barrier phases run on counters that continue
// across items, and the item boundary is overlapped:
//   * the producer TMA-loads the next item's K / V tiles into a smem buffer
//     once it has issued this item's last Q / dO sub-tile;
//   * the softmax warps copy them into the K / V TMEM A operands as soon as
//     this item's last S^T / dP^T MMAs have completed (the s_full of its last
//     sub-tile), so the MMA issuer queues the next item's first S^T / dP^T
//     ahead of this item's last dV / dK GEMMs;
//   * the next item's first dV / dK GEMMs overwrite the accumulators, so they
//     wait for dkv_free: the softmax warps' read-out of this item's dK / dV,
//     whose global stores then overlap the next item's MMAs.
// Per item every value is computed in dkv_kernel's order (bitwise equal).
__global__ void __launch_bounds__(kDkvThreads, 1)
    dkv_persist_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO,
                       const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, Args a,
                       int nk) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                      // QS stages x 2 x [64][64]
  uint8_t* sdO = sQ + QS * 2 * kBox64;   // QS stages x 2 x [64][64]
  uint8_t* sP = sdO + QS * 2 * kBox64;   // 2 x [128 keys][64 q]
  uint8_t* sS = sP + 2 * kBox128;        // 2 x [128 keys][64 q]
  uint8_t* sKV = sS + 2 * kBox128;       // next item's K, V: 2 x 2 x [128 keys][64 dh]
  uint8_t* sLD = sKV + 4 * kBox128;      // QS stages x {LSE[64], D[64]} fp32
  uint64_t* bar = reinterpret_cast<uint64_t*>(sLD + QS * 512);
  uint64_t* kv_full = bar;               // K / V in TMEM (16 warp arrivals)
  uint64_t* q_full = bar + 1;            // [QS]
  uint64_t* q_empty = q_full + QS;       // [QS]
  uint64_t* s_full = q_empty + QS;       // [1]
  uint64_t* s_free = s_full + 1;         // [1]
  uint64_t* pds_full = s_free + 1;       // [2]
  uint64_t* pds_free = pds_full + 2;     // [2]
  uint64_t* kv_tma = pds_free + 2;       // K / V landed in sKV (TMA)
  uint64_t* kv_smem_free = kv_tma + 1;   // sKV copied to TMEM (16 warp arrivals)
  uint64_t* dkv_done = kv_smem_free + 1; // the item's last dV / dK GEMMs completed
  uint64_t* dkv_free = dkv_done + 1;     // the item's dK / dV read out (16 warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dkv_free + 1);

  const int items = nk * a.KVH;
  const int per = a.H / a.KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // item -> (key tile, kv head) and its loop extent
  auto item_of = [&](int it, AttnTile& tl, AttnSeg& sg, int& g, int& i0, int& nqt) {
    const int t = it / a.KVH;
    g = it - t * a.KVH;
    tl = a.tiles[t];
    sg = a.segs[tl.seg];
    i0 = max(0, tl.first - sg.prefix);
    nqt = (sg.len - i0 + SUB - 1) / SUB;
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmO);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(kv_full, 16);
    for (int i = 0; i < QS; ++i) {
      mbar_init(&q_full[i], 2);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 16);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&pds_full[i], 16);
      mbar_init(&pds_free[i], 1);
    }
    mbar_init(kv_tma, 1);
    mbar_init(kv_smem_free, 16);
    mbar_init(dkv_done, 1);
    mbar_init(dkv_free, 16);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 64;
  const uint32_t tdV = tmem + 128, tdK = tmem + 256;
  const uint32_t tAk = tmem + 384, tAv = tmem + 448;
  const uint32_t sQ0 = smem_u32(sQ), sO0 = smem_u32(sdO), sP0 = smem_u32(sP), sS0 = smem_u32(sS),
                 sLD0 = smem_u32(sLD), sKV0 = smem_u32(sKV);
  const uint32_t bQf = smem_u32(q_full), bQe = smem_u32(q_empty), bSf = smem_u32(s_full),
                 bSr = smem_u32(s_free), bPf = smem_u32(pds_full), bPr = smem_u32(pds_free);

  if (warp == 16) {
    int qs = 0, n = 0;
    uint32_t ph = 0;
    auto load_kv = [&](int it) {  // lane 0: the item's K / V tiles into sKV
      AttnTile tl;
      AttnSeg sg;
      int g, i0, nqt;
      item_of(it, tl, sg, g, i0, nqt);
      const int krow = sg.kv_row0 + tl.first;
      mbar_expect_tx(kv_tma, 4 * kBox128);
      tma_load_2d(sKV, &tmK, kv_tma, g * DH, krow);
      tma_load_2d(sKV + kBox128, &tmK, kv_tma, g * DH + 64, krow);
      tma_load_2d(sKV + 2 * kBox128, &tmV, kv_tma, g * DH, krow);
      tma_load_2d(sKV + 3 * kBox128, &tmV, kv_tma, g * DH + 64, krow);
    };
    if (lane == 0 && blockIdx.x < items) load_kv(blockIdx.x);
    for (int item = snake_item(0); item < items; item = snake_item(++n)) {
      AttnTile tl;
      AttnSeg sg;
      int g, i0, nqt;
      item_of(item, tl, sg, g, i0, nqt);
      const int iters = per * nqt;
      int hi = 0, qi = 0;
      for (int it = 0; it < iters; ++it) {
        const int hq = g * per + hi;
        const int qt0 = i0 + qi * SUB;
        const int qrow = sg.q_start + qt0;
        // LSE / D of the sub-tile fetched before the slot wait (their latency
        // overlaps it)
        const int64_t base = static_cast<int64_t>(hq) * a.T + qrow;
        float lv[2], dv[2];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c = lane + 32 * h2;
          const bool in = qt0 + c < sg.len;
          lv[h2] = in ? __ldg(a.lse + base + c) : 0.f;
          dv[h2] = in ? __ldg(a.dsum + base + c) : 0.f;
        }
        stress_delay(a.stress, 4, it);
        mbar_wait_s(bQe + qs * 8, ph ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&q_full[qs], 4 * kBox64);
          uint8_t* q = sQ + qs * 2 * kBox64;
          uint8_t* o = sdO + qs * 2 * kBox64;
          tma_load_2d(q, &tmQ, &q_full[qs], hq * DH, qrow);
          tma_load_2d(q + kBox64, &tmQ, &q_full[qs], hq * DH + 64, qrow);
          tma_load_2d(o, &tmO, &q_full[qs], hq * DH, qrow);
          tma_load_2d(o + kBox64, &tmO, &q_full[qs], hq * DH + 64, qrow);
        }
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c = lane + 32 * h2;
          sts_f32(sLD0 + qs * 512 + c * 4, lv[h2]);
          sts_f32(sLD0 + qs * 512 + 256 + c * 4, dv[h2]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_s(bQf + qs * 8);
        if (++qi == nqt) { qi = 0; ++hi; }
        if (++qs == QS) { qs = 0; ph ^= 1; }
      }
      // the next item's K / V, once this item's copy has left sKV
      if (lane == 0 && snake_item(n + 1) < items) {
        mbar_wait(kv_smem_free, n & 1);
        load_kv(snake_item(n + 1));
      }
    }
  } else if (warp == 17) {
    constexpr uint32_t idS = umma_idesc_bf16(128, SUB, 0, 0);
    constexpr uint32_t idG = umma_idesc_bf16(128, 128, 0, 1);
    int is = 0, cs = 0, J = 0, n = 0;  // ring slots, sub-tiles so far, items so far
    uint32_t ps = 0;
    auto issue_s = [&](int Js) {
      mbar_wait_s(bQf + is * 8, ps);
      mbar_wait_s(bSr, (Js & 1) ^ 1);
      tc_fence_after();
      const uint32_t q0 = sQ0 + is * 2 * kBox64, o0 = sO0 + is * 2 * kBox64;
      umma4_ts_w<8, 2>(tS, tAk, kdesc(q0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tS, tAk + 32, kdesc(q0, kBox64, 4), idS, 1u);
      umma4_ts_w<8, 2>(tP, tAv, kdesc(o0, kBox64, 0), idS, 0u);
      umma4_ts_w<8, 2>(tP, tAv + 32, kdesc(o0, kBox64, 4), idS, 1u);
      umma_commit_w(bSf);
      if (++is == QS) { is = 0; ps ^= 1; }
    };
    if (blockIdx.x < items) {
      mbar_wait(kv_full, 0);
      tc_fence_after();
      issue_s(0);
    }
    for (int item = snake_item(0); item < items; item = snake_item(++n)) {
      AttnTile tl;
      AttnSeg sg;
      int g, i0, nqt;
      item_of(item, tl, sg, g, i0, nqt);
      const int iters = per * nqt;
      for (int it = 0; it < iters; ++it, ++J) {
        stress_delay(a.stress, 5, J);
        if (it + 1 < iters) {
          issue_s(J + 1);
        } else if (snake_item(n + 1) < items) {
          // the next item's K / V are in TMEM: its first S^T / dP^T go ahead
          // of this item's last dV / dK GEMMs
          mbar_wait(kv_full, (n + 1) & 1);
          tc_fence_after();
          issue_s(J + 1);
        }
        const uint32_t b = J & 1;
        mbar_wait_s(bPf + b * 8, (J >> 1) & 1);
        if (it == 0 && n > 0) mbar_wait(dkv_free, (n - 1) & 1);  // previous item's dK / dV read out
        tc_fence_after();
        const uint32_t q0 = sQ0 + cs * 2 * kBox64, o0 = sO0 + cs * 2 * kBox64;
        const uint32_t p0 = sP0 + b * kBox128, s0 = sS0 + b * kBox128;
        umma4_ss_w<2, 128>(tdV, kdesc(p0, kBox128, 0), mndesc(o0, kBox64, 0), idG, it > 0 ? 1u : 0u);
        umma4_ss_w<2, 128>(tdK, kdesc(s0, kBox128, 0), mndesc(q0, kBox64, 0), idG, it > 0 ? 1u : 0u);
        umma_commit_w(bQe + cs * 8);
        umma_commit_w(bPr + b * 8);
        if (++cs == QS) cs = 0;
      }
      umma_commit_w(smem_u32(dkv_done));
    }
  } else {
    const int quarter = warp & 3, part = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    uint32_t dst_off[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) dst_off[c] = sw_off(row, part * 2 + c);
    // sKV -> the K / V TMEM A operands: this warp's 32 rows, dh columns
    // [32 part, 32 part + 32) of each (16-byte chunks (part & 1) * 4 .. + 3
    // of box part >> 1, 128B-swizzled by row)
    auto copy_kv = [&](uint32_t phase) {
      mbar_wait(kv_tma, phase);
      uint32_t wk[16], wv[16];
      const uint32_t bk = sKV0 + (part >> 1) * kBox128 + row * 128;
      const uint32_t bv = bk + 2 * kBox128;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ch = ((part & 1) * 4 + c) ^ (row & 7);
        const uint4 x = lds128(bk + (ch << 4));
        const uint4 y = lds128(bv + (ch << 4));
        wk[4 * c] = x.x, wk[4 * c + 1] = x.y, wk[4 * c + 2] = x.z, wk[4 * c + 3] = x.w;
        wv[4 * c] = y.x, wv[4 * c + 1] = y.y, wv[4 * c + 2] = y.z, wv[4 * c + 3] = y.w;
      }
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tAk + lane_off + part * 16),
          "r"(wk[0]), "r"(wk[1]), "r"(wk[2]), "r"(wk[3]), "r"(wk[4]), "r"(wk[5]), "r"(wk[6]), "r"(wk[7]), "r"(wk[8]),
          "r"(wk[9]), "r"(wk[10]), "r"(wk[11]), "r"(wk[12]), "r"(wk[13]), "r"(wk[14]), "r"(wk[15])
          : "memory");
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tAv + lane_off + part * 16),
          "r"(wv[0]), "r"(wv[1]), "r"(wv[2]), "r"(wv[3]), "r"(wv[4]), "r"(wv[5]), "r"(wv[6]), "r"(wv[7]), "r"(wv[8]),
          "r"(wv[9]), "r"(wv[10]), "r"(wv[11]), "r"(wv[12]), "r"(wv[13]), "r"(wv[14]), "r"(wv[15])
          : "memory");
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(kv_full);
      warp_arrive(kv_smem_free);
    };
    if (blockIdx.x < items) copy_kv(0);
    int qs = 0, J = 0, n = 0;
    uint32_t qph = 0;
    for (int item = snake_item(0); item < items; item = snake_item(++n)) {
      // per-item loop state kept small (96 registers at 576 threads): the
      // rows / head are re-read from the tile table for the epilogue
      int iters, i0, qend, seg_len, qlo, full_lo;
      {
        AttnTile tl;
        AttnSeg sg;
        int g, nqt;
        item_of(item, tl, sg, g, i0, nqt);
        iters = per * nqt;
        qend = i0 + nqt * SUB;
        seg_len = sg.len;
        const int kv_len = sg.prefix + sg.len;
        const int key = tl.first + row;
        qlo = row < tl.count && key < kv_len ? key - sg.prefix : INT_MAX;
        // sub-tiles from query full_lo on see every key of the tile (uniform body)
        full_lo = tl.first + 127 < kv_len ? tl.first + 127 - sg.prefix : INT_MAX;
      }
      const bool next = snake_item(n + 1) < items;
      int qt0 = i0;
      for (int it = 0; it < iters; ++it, ++J) {
        const uint32_t b = J & 1;
        mbar_wait_s(bSf, J & 1);
        tc_fence_after();
        // this s_full certifies the item's last S^T / dP^T: the K / V A
        // operands are free for the next item's
        if (it + 1 == iters && next) copy_kv((n + 1) & 1);
        uint32_t rs[16], rp[16];
        tmem_ld16(tS + lane_off + part * 16, rs);
        tmem_ld16(tP + lane_off + part * 16, rp);
        tmem_ld_wait();
        tc_fence_before();
        warp_arrive_s(bSr);
        stress_delay(a.stress, 6, J);
        mbar_wait_s(bQf + qs * 8, qph);
        const uint32_t lrow = sLD0 + qs * 512 + part * 64;
        uint32_t pp[8], pd[8];
        auto body = [&](auto masked) {
          const float2 sl2v = make_float2(a.sl2, a.sl2), nlg = make_float2(-kLog2e, -kLog2e),
                       m1 = make_float2(-1.f, -1.f);
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 L = lds_f32x4(lrow + c4 * 16);
            const float4 Dv = lds_f32x4(lrow + 256 + c4 * 16);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              const int col = c4 * 4 + 2 * h2;
              const float2 nl = fmul2(h2 ? make_float2(L.z, L.w) : make_float2(L.x, L.y), nlg);
              const float2 nd = fmul2(h2 ? make_float2(Dv.z, Dv.w) : make_float2(Dv.x, Dv.y), m1);
              const float2 x = ffma2(make_float2(__uint_as_float(rs[col]), __uint_as_float(rs[col + 1])), sl2v, nl);
              float2 p = make_float2(ex2(x.x), ex2(x.y));
              float2 ds = fmul2(p, fadd2(make_float2(__uint_as_float(rp[col]), __uint_as_float(rp[col + 1])), nd));
              if constexpr (decltype(masked)::value) {
                const int qq = qt0 + part * 16 + col;
                const bool in0 = qq >= qlo && qq < seg_len, in1 = qq + 1 >= qlo && qq + 1 < seg_len;
                p = make_float2(in0 ? p.x : 0.f, in1 ? p.y : 0.f);
                ds = make_float2(in0 ? ds.x : 0.f, in1 ? ds.y : 0.f);
              }
              pp[2 * c4 + h2] = pack_bf16(p.x, p.y);
              pd[2 * c4 + h2] = pack_bf16(ds.x, ds.y);
            }
          }
        };
        if (full_lo <= qt0 && qt0 + SUB <= seg_len)
          body(std::false_type{});
        else
          body(std::true_type{});
        stress_delay(a.stress, 7, J);
        if (J >= 2) mbar_wait_s(bPr + b * 8, ((J >> 1) & 1) ^ 1);
        const uint32_t dP_ = sP0 + b * kBox128, dS_ = sS0 + b * kBox128;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          sts128(dP_ + dst_off[c], make_uint4(pp[4 * c], pp[4 * c + 1], pp[4 * c + 2], pp[4 * c + 3]));
          sts128(dS_ + dst_off[c], make_uint4(pd[4 * c], pd[4 * c + 1], pd[4 * c + 2], pd[4 * c + 3]));
        }
        fence_async_smem();
        warp_arrive_s(bPf + b * 8);
        qt0 += SUB;
        if (qt0 == qend) qt0 = i0;
        if (++qs == QS) { qs = 0; qph ^= 1; }
      }
      AttnTile tl;
      AttnSeg sg;
      int g, i0_, nqt_;
      item_of(item, tl, sg, g, i0_, nqt_);
      const int key = tl.first + row;
      const bool kok = row < tl.count && key < sg.prefix + sg.len;
      mbar_wait(dkv_done, n & 1);
      tc_fence_after();
      // read-out in two 16-column halves (register budget); dkv_free after
      // the last TMEM load, the global stores overlap the next item's MMAs
      if (a.dkv_out) {
        // parts 0, 1: dK chunks (part, part + 2), rotated back; parts 2, 3: dV
        const bool is_k = part < 2;
        const int c0 = part & 1;
        const uint32_t src = (is_k ? tdK : tdV) + lane_off;
        const int64_t r = sg.kv_row0 + key;
        const float sc = is_k ? a.scale : 1.f;
        __nv_bfloat16* dst = a.dkv_out + r * a.dkv_out_ld + (is_k ? a.col_k : a.col_v) + g * DH;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t ra[16], rb[16];
          tmem_ld16(src + c0 * 32 + hh * 16, ra);
          tmem_ld16(src + (c0 + 2) * 32 + hh * 16, rb);
          tmem_ld_wait();
          if (hh == 1) {
            tc_fence_before();
            warp_arrive(dkv_free);
          }
          if (kok) {
            float fa[16], fb[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              fa[e] = __uint_as_float(ra[e]) * sc;
              fb[e] = __uint_as_float(rb[e]) * sc;
            }
            if (is_k && a.rope_tab) rope_inverse16(a.rope_tab + r * (DH / 2) + c0 * 32 + hh * 16, fa, fb);
            store_bf16x16(dst + c0 * 32 + hh * 16, fa);
            store_bf16x16(dst + (c0 + 2) * 32 + hh * 16, fb);
          }
        }
      } else {
        const int c = part;
        float* dkr = a.dk_acc + static_cast<int64_t>(sg.kv_row0 + key) * a.acc_stride + g * DH + c * 32;
        float* dvr = a.dv_acc + static_cast<int64_t>(sg.kv_row0 + key) * a.acc_stride + g * DH + c * 32;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t rk[16], rv[16];
          tmem_ld16(tdK + lane_off + c * 32 + hh * 16, rk);
          tmem_ld16(tdV + lane_off + c * 32 + hh * 16, rv);
          tmem_ld_wait();
          if (hh == 1) {
            tc_fence_before();
            warp_arrive(dkv_free);
          }
          if (kok) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float4 k4 = reinterpret_cast<float4*>(dkr + hh * 16)[q];
              k4.x += __uint_as_float(rk[4 * q]) * a.scale;
              k4.y += __uint_as_float(rk[4 * q + 1]) * a.scale;
              k4.z += __uint_as_float(rk[4 * q + 2]) * a.scale;
              k4.w += __uint_as_float(rk[4 * q + 3]) * a.scale;
              reinterpret_cast<float4*>(dkr + hh * 16)[q] = k4;
              float4 v4 = reinterpret_cast<float4*>(dvr + hh * 16)[q];
              v4.x += __uint_as_float(rv[4 * q]);
              v4.y += __uint_as_float(rv[4 * q + 1]);
              v4.z += __uint_as_float(rv[4 * q + 2]);
              v4.w += __uint_as_float(rv[4 * q + 3]);
              reinterpret_cast<float4*>(dvr + hh * 16)[q] = v4;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool map_rows(CUtensorMap* m, const void* ptr, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  static EncodeFn enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<EncodeFn>(p);
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// dQ kernel choice: the 128-key-tile kernel (N = 128 S / dP MMAs) wins on
// long-context launches (T = 16384 causal: -11 % dQ time) and loses a little
// on short ones, where 64-key sub-tiles cut less into the causal diagonal
// (T = 2048: +3 %).  CF_DQ_WIDE=1 / 0 forces it on / off (A/B, tests).
bool dq_wide(const AttnParams& p) {
  static const int v = [] {
    const char* e = std::getenv("CF_DQ_WIDE");
    return e ? std::atoi(e) : -1;
  }();
  return v >= 0 ? v == 1 : p.keys_per_query >= 3072.0;
}

// 64-key dQ kernel choice (CF_DQ_PERSIST): 2 (default) the TMA-fed
// persistent kernel with D from dsum_rows_kernel (packed short chunks: in-step
// attention backward +2 %, profiles/round2_ab_dq_tma.txt), 1 the persistent
// kernel staging Q / dO / O itself, 0 one CTA per (tile, head)
int dq_persist() {
  static const int v = [] {
    const char* e = std::getenv("CF_DQ_PERSIST");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}
// dK/dV kernel choice: the persistent kernel for short-context launches
// (packed short chunks: in-step attention backward 135 -> 143 TFLOP/s), the
// one-CTA-per-(key tile, kv head) grid for long-context ones (>= 3072 keys per
// query, the wide-dQ criterion), where hardware scheduling of the causal work
// does as well (profiles/round2_ab_dkv_persist.txt).  CF_DKV_PERSIST=1 / 0
// forces it on / off (A/B, tests).
bool dkv_persist(const AttnParams& p) {
  static const int v = [] {
    const char* e = std::getenv("CF_DKV_PERSIST");
    return e ? std::atoi(e) : -1;
  }();
  return v >= 0 ? v == 1 : p.keys_per_query < 3072.0;
}
int attn_num_sms() {
  static const int n = [] {
    int dev = 0, c = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
    return c > 0 ? c : 148;
  }();
  return n;
}

int g_attn_stress = 0;
void set_attn_stress(int on) { g_attn_stress = on ? 1 : 0; }

cudaError_t attn_backward_tc(const AttnParams& p, const AttnTile* qtiles128, int32_t nq, const AttnTile* ktiles128,
                             int32_t nk, int64_t kv_rows, cudaStream_t st) {
  if (nq == 0) return cudaSuccess;
  const uint64_t qc = static_cast<uint64_t>(p.H) * DH, kc = static_cast<uint64_t>(p.KVH) * DH;
  CUtensorMap q128, o128, k64, v64, q64, o64;
  if (!map_rows(&q128, p.q, qc, p.T, p.q_stride, 128) || !map_rows(&o128, p.dout, qc, p.T, p.dout_stride, 128) ||
      !map_rows(&k64, p.k, kc, kv_rows, p.kv_stride, 64) || !map_rows(&v64, p.v, kc, kv_rows, p.kv_stride, 64) ||
      !map_rows(&q64, p.q, qc, p.T, p.q_stride, 64) || !map_rows(&o64, p.dout, qc, p.T, p.dout_stride, 64))
    return cudaErrorInvalidValue;
  Args a{p.segs, qtiles128, p.q, p.q_stride, p.dout, p.dout_stride, p.k, p.v, p.kv_stride, p.lse, p.dsum, p.o,
         p.o_stride, p.dq, p.dq_stride, p.dk_acc, p.dv_acc, p.acc_stride, p.T, p.H, p.KVH, p.scale * kLog2e,
         p.scale, p.rope_tab, p.dkv_out, p.dkv_out_ld, p.col_k, p.col_v, g_attn_stress};
  const size_t smem_dq = 1024 + (KS + VS) * 2 * kBox64 + 2 * kBox128 + 256 * 4 + 256;
  const size_t smem_dkv = 1024 + QS * 2 * 2 * kBox64 + 4 * kBox128 + QS * 512 + 256;
  // per (kernel, device), thread-safe
  cudaError_t attr = cudaSuccess;
  if (attr == cudaSuccess) attr = smem_optin(reinterpret_cast<const void*>(dq_kernel), static_cast<int>(smem_dq));
  if (attr == cudaSuccess) attr = smem_optin(reinterpret_cast<const void*>(dkv_kernel), static_cast<int>(smem_dkv));
  if (attr != cudaSuccess) return attr;
  // D = rowsum(dO * O) is produced by the dQ kernel (no separate dsum pass)
  if (dq_wide(p)) {
    CUtensorMap k128, v128;
    if (!map_rows(&k128, p.k, kc, kv_rows, p.kv_stride, 128) || !map_rows(&v128, p.v, kc, kv_rows, p.kv_stride, 128))
      return cudaErrorInvalidValue;
    const size_t smem_w = 1024 + (kWKS + kWVS) * 2 * kBox128 + 4 * kBox128 + 256;
    attr = smem_optin(reinterpret_cast<const void*>(dq_wide_kernel), static_cast<int>(smem_w));
    if (attr != cudaSuccess) return attr;
    dq_wide_kernel<<<dim3(nq, p.H), kDqWideThreads, smem_w, st>>>(k128, v128, a);
  } else if (dq_persist() == 2) {
    // D first (HBM-bound pass), then the TMA-fed persistent dQ kernel
    const size_t smem_t = 1024 + (KS + VS) * 2 * kBox64 + 6 * kBox128 + 256;
    attr = smem_optin(reinterpret_cast<const void*>(dq_persist_tma_kernel), static_cast<int>(smem_t));
    if (attr != cudaSuccess) return attr;
    dsum_rows_kernel<<<p.T, 256, 0, st>>>(a);
    const int items = nq * p.H;
    dq_persist_tma_kernel<<<std::min(items, attn_num_sms()), kThreads, smem_t, st>>>(k64, v64, q128, o128, a, nq);
  } else if (dq_persist()) {
    const int items = nq * p.H;
    const int grid = std::min(items, attn_num_sms());
    attr = smem_optin(reinterpret_cast<const void*>(dq_persist_kernel), static_cast<int>(smem_dq));
    if (attr != cudaSuccess) return attr;
    dq_persist_kernel<<<grid, kThreads, smem_dq, st>>>(k64, v64, a, nq);
  } else {
    dq_kernel<<<dim3(nq, p.H), kThreads, smem_dq, st>>>(q128, o128, k64, v64, a);
  }
#if CF_ATTN_TRACE
  {
    cudaStreamSynchronize(st);
    static unsigned long long h[3][8192];
    int n[3] = {0, 0, 0};
    cudaMemcpyFromSymbol(h, g_trace, sizeof(h));
    cudaMemcpyFromSymbol(n, g_trace_n, sizeof(n));
    if (const char* path = std::getenv("CF_TRACE_OUT")) {
      if (FILE* f = std::fopen(path, "a")) {
        std::fprintf(f, "# launch nq=%d H=%d\n", nq, p.H);
        for (int r = 0; r < 3; ++r)
          for (int i = 0; i < std::min(n[r], 8192); ++i)
            std::fprintf(f, "%d %llu %llu %llu\n", r, h[r][i] >> 20, (h[r][i] >> 16) & 15, h[r][i] & 0xffff);
        std::fclose(f);
      }
    }
    const int z[3] = {0, 0, 0};
    cudaMemcpyToSymbol(g_trace_n, z, sizeof(z));
  }
#endif
  a.tiles = ktiles128;
  if (nk > 0 && dkv_persist(p)) {
    CUtensorMap k128, v128;
    if (!map_rows(&k128, p.k, kc, kv_rows, p.kv_stride, 128) || !map_rows(&v128, p.v, kc, kv_rows, p.kv_stride, 128))
      return cudaErrorInvalidValue;
    const size_t smem_p = smem_dkv + 4 * kBox128;
    attr = smem_optin(reinterpret_cast<const void*>(dkv_persist_kernel), static_cast<int>(smem_p));
    if (attr != cudaSuccess) return attr;
    const int items = nk * p.KVH;
    dkv_persist_kernel<<<std::min(items, attn_num_sms()), kDkvThreads, smem_p, st>>>(q64, o64, k128, v128, a, nk);
  } else if (nk > 0) {
    dkv_kernel<<<dim3(nk, p.KVH), kDkvThreads, smem_dkv, st>>>(q64, o64, a);
  }
  return cudaGetLastError();
}

}  // namespace cfk
