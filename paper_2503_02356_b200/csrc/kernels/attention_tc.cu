// tcgen05 chunked causal attention forward for head_dim 128 (sm_100a).
//
// One CTA = 128 queries of one q head of one packed segment; loops over
// 128-key tiles of the segment's keys [0, prefix + last query] (bottom-right
// causal mask, KV prefix read straight from the per-sequence cache).
//
//   warps 0-7  softmax: thread = (query row, 64-column half of the tile);
//              tcgen05.ld of its half-row of S from TMEM, row max exchanged
//              with the partner warp through smem, online softmax (exp2, lazy
//              O rescale when the running max grows by > 2^8), P -> bf16 ->
//              128B-swizzled smem (UMMA A operand).  Two softmax warps per SM
//              sub-partition hide each other's MUFU / TMEM-load latency.
//   warp  8    TMA producer: Q once, K/V tiles into a 2-stage ring
//   warp  9    MMA issuer (one lane): S = Q K^T (M128 N128 K128, K-major x2),
//              O += P V (A = P K-major in smem, B = V N-major view of the same
//              TMA tile), accumulators in TMEM: S0 | S1 | O (384 of 512 cols)
// Reference semantics: toy_model.hpp:263-302 (scale 1/sqrt(dh), max-
// subtracted softmax, PV, GQA head map hq / per_kv).
#include <cfloat>

#include "attention.h"
#include "attention_tc.h"
#include "common.cuh"

namespace cfk {
namespace {

constexpr int TQ = 128, TK = 128, DH = 128;
constexpr uint32_t kBox = 128 * 64 * 2;  // [128 rows][64 cols] bf16 = 16 KiB
constexpr uint32_t kTile = 2 * kBox;     // 128 rows x 128 cols
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescale = 8.0f;  // log2 threshold for lazy O rescaling

constexpr int KVS = 3;  // forward K/V ring depth

struct TcArgs {
  const AttnSeg* segs;
  const AttnTile* tiles;  // 128-row query tiles
  const __nv_bfloat16* q;
  int64_t q_stride;
  __nv_bfloat16* o;
  int64_t o_stride;
  float* lse;
  int32_t T, H, KVH;
  float sl2;  // scale * log2(e)
};

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 16-byte chunk c (0..15 over 128 columns) of row r in a K-major SW128 tile
// made of two [128 rows][64 cols] boxes.
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
  return static_cast<uint32_t>((c >> 3) * kBox + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// K-major operand descriptor at k-step ks (16 elements) of a 2-box tile.
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int ks) {
  return umma_desc_sw128(base + (ks >> 2) * kBox + (ks & 3) * 32, 16, 1024);
}
// MN-major view (N = the 128 tile columns, K = the 128 tile rows) at k-step ks.
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int ks) {
  return umma_desc_sw128(base + ks * 2048, kBox, 1024);
}

constexpr int kFwdThreads = 320;

__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // Q and P live in TMEM (A operands of S = QK^T and O += PV): shared memory
  // only streams K and V (3-stage rings), halving smem operand traffic.
  uint8_t* sK = sm;                      // KV stages
  uint8_t* sV = sK + KVS * kTile;        // KV stages
  float* sRed = reinterpret_cast<float*>(sV + KVS * kTile);  // [2 parity][2 half][128 rows] row-max / row-sum
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRed + 512);
  uint64_t* q_ready = bar;
  uint64_t* k_full = bar + 1;           // [KVS]
  uint64_t* k_empty = k_full + KVS;     // [KVS]
  uint64_t* v_full = k_empty + KVS;     // [KVS]
  uint64_t* v_empty = v_full + KVS;     // [KVS]
  uint64_t* s_full = v_empty + KVS;     // [2]
  uint64_t* s_free = s_full + 2;        // [2]
  uint64_t* p_full = s_free + 2;
  uint64_t* p_free = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + 1);

  const AttnTile tl = a.tiles[blockIdx.x];
  const AttnSeg sg = a.segs[tl.seg];
  const int h = blockIdx.y, g = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_row0 = sg.q_start + tl.first;
  const int kv_len = sg.prefix + tl.first + tl.count;  // keys needed by this tile
  const int nkt = (kv_len + TK - 1) / TK;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_ready, 8);  // arrivals count softmax warps
    for (int i = 0; i < KVS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
    }
    mbar_init(p_full, 8);
    mbar_init(p_free, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO = tmem + 256;
  const uint32_t tQ = tmem + 384;  // Q: 128 rows x 128 bf16 = 64 columns
  const uint32_t tP = tmem + 448;  // P: 128 rows x 128 bf16 = 64 columns

  if (warp == 8) {
    if (lane == 0) {
      for (int j = 0; j < nkt; ++j) {
        const int st = j % KVS;
        const uint32_t ph = (j / KVS) & 1;
        const int krow = sg.kv_row0 + j * TK;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], kTile);
        tma_load_2d(sK + st * kTile, &tmK, &k_full[st], g * DH, krow);
        tma_load_2d(sK + st * kTile + kBox, &tmK, &k_full[st], g * DH + 64, krow);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], kTile);
        tma_load_2d(sV + st * kTile, &tmV, &v_full[st], g * DH, krow);
        tma_load_2d(sV + st * kTile + kBox, &tmV, &v_full[st], g * DH + 64, krow);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {
      constexpr uint32_t idS = umma_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idO = umma_idesc_bf16(128, 128, 0, 1);
      auto issue_s = [&](int j) {
        const int st = j % KVS, b = j & 1;
        mbar_wait(&k_full[st], (j / KVS) & 1);
        mbar_wait(&s_free[b], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k0 = smem_u32(sK + st * kTile);
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks)
          umma_bf16_ts(tS[b], tQ + ks * 8, kdesc(k0, ks), idS, ks > 0 ? 1u : 0u);
        umma_commit(&k_empty[st]);
        umma_commit(&s_full[b]);
      };
      mbar_wait(q_ready, 0);
      tc_fence_after();
      issue_s(0);
      for (int j = 0; j < nkt; ++j) {
        if (j + 1 < nkt) issue_s(j + 1);
        const int st = j % KVS;
        mbar_wait(p_full, j & 1);
        mbar_wait(&v_full[st], (j / KVS) & 1);
        tc_fence_after();
        const uint32_t v0 = smem_u32(sV + st * kTile);
#pragma unroll
        for (int ks = 0; ks < TK / 16; ++ks)
          umma_bf16_ts(tO, tP + ks * 8, mndesc(v0, ks), idO, (j > 0 || ks > 0) ? 1u : 0u);
        umma_commit(&v_empty[st]);
        umma_commit(p_free);
      }
    }
  } else {
    // softmax warps 0..7: TMEM lane quarter = warp & 3, half = warp >> 2
    const int quarter = warp & 3, half = warp >> 2;
    const int row = quarter * 32 + lane;
    const int qi = tl.first + row;                      // query index in segment
    const int lim = sg.prefix + min(qi, sg.len - 1);    // last visible key
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t col0 = static_cast<uint32_t>(half * 64);
    {
      // stage this row's Q (this half's 64 dims) into TMEM as the A operand
      uint32_t qw[32];
      const bool qok = row < tl.count;
      const uint4* src = reinterpret_cast<const uint4*>(a.q + static_cast<int64_t>(q_row0 + row) * a.q_stride +
                                                        static_cast<int64_t>(h) * DH + half * 64);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = qok ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
        qw[4 * c] = v.x;
        qw[4 * c + 1] = v.y;
        qw[4 * c + 2] = v.z;
        qw[4 * c + 3] = v.w;
      }
      tmem_st32(tQ + lane_off + half * 32, qw);
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(q_ready);
    }
    float m = -FLT_MAX, l = 0.f;
    for (int j = 0; j < nkt; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[64];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
        tmem_ld32(tS[st] + lane_off + col0 + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(r[e]);
      }
      tc_fence_before();
      warp_arrive(&s_free[st]);
      const int key0 = j * TK + half * 64;
      // tiles entirely below the diagonal of every row of the CTA need no mask
      const bool full = j * TK + TK - 1 <= sg.prefix + tl.first;
      float tmax = -FLT_MAX;
      if (full) {
#pragma unroll
        for (int e = 0; e < 64; ++e) tmax = fmaxf(tmax, s[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          s[e] = (key0 + e <= lim) ? s[e] : -FLT_MAX;  // exp2 of the masked scores underflows to 0
          tmax = fmaxf(tmax, s[e]);
        }
      }
      // exchange the half-row maxima with the partner warp (same rows)
      const uint32_t red = smem_u32(sRed) + (j & 1) * 1024;
      sts_f32(red + (half * 128 + row) * 4, tmax);
      asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory");
      tmax = fmaxf(tmax, lds_f32(red + ((half ^ 1) * 128 + row) * 4)) * a.sl2;  // scaled log2 domain (sl2 > 0)
      bool rescale = false;
      float alpha = 1.f;
      if (tmax > m + kRescale || j == 0) {
        const float mn = fmaxf(m, tmax);
        alpha = ex2(m - mn);
        rescale = j > 0;
        m = mn;
      }
      l *= alpha;
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float p0 = ex2(fmaf(s[2 * e], a.sl2, -m));
        const float p1 = ex2(fmaf(s[2 * e + 1], a.sl2, -m));
        l += p0 + p1;
        pk[e] = pack_bf16(p0, p1);
      }
      if (j > 0) {
        mbar_wait(p_free, (j - 1) & 1);  // PV_{j-1} done: O stable, P buffer free
        tc_fence_after();
      }
      if (rescale) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld32(tO + lane_off + col0 + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
          tmem_st32(tO + lane_off + col0 + c * 32, r);
        }
        tmem_st_wait();
      }
      // P row -> TMEM (A operand of O += P V): this half's 64 keys = 32 columns
      tmem_st32(tP + lane_off + half * 32, pk);
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(p_full);
    }
    // combine the two half-row sums
    const uint32_t red = smem_u32(sRed) + (nkt & 1) * 1024;
    sts_f32(red + (half * 128 + row) * 4, l);
    asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory");
    l += lds_f32(red + ((half ^ 1) * 128 + row) * 4);
    mbar_wait(p_free, (nkt - 1) & 1);
    tc_fence_after();
    const bool ok = qi < sg.len && row < tl.count;
    const float inv = 1.f / l;
    __nv_bfloat16* orow = a.o + static_cast<int64_t>(q_row0 + row) * a.o_stride + h * DH + half * 64;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t r[32];
      tmem_ld32(tO + lane_off + col0 + c * 32, r);
      tmem_ld_wait();
      if (ok) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_uint4(pack_bf16(__uint_as_float(r[8 * q]) * inv, __uint_as_float(r[8 * q + 1]) * inv),
                              pack_bf16(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv),
                              pack_bf16(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv),
                              pack_bf16(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv));
      }
    }
    if (ok && half == 0) a.lse[static_cast<int64_t>(h) * a.T + q_row0 + row] = (m + log2f(l)) * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// ------------------------------------------------------------------ backward
struct TcBwdArgs {
  const AttnSeg* segs;
  const AttnTile* tiles;  // 128-row tiles (queries for dQ, keys for dK/dV)
  const float* lse;       // [H, T] natural log
  const float* dsum;      // [H, T]
  __nv_bfloat16* dq;
  int64_t dq_stride;
  float* dk_acc;
  float* dv_acc;
  int64_t acc_stride;
  int32_t T, H, KVH;
  float sl2, scale;
};

__device__ __forceinline__ void named_sync_128() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// dQ: CTA = 128 queries of one q head; per 128-key tile
//   S = Q K^T, dP = dO V^T (TMEM) -> dS = P (dP - D) (bf16, smem) -> dQ += dS K.
__global__ void __launch_bounds__(192, 1)
    attn_dq_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO,
                      const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, TcBwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sdO = sQ + kTile;
  uint8_t* sK = sdO + kTile;     // 2 stages
  uint8_t* sV = sK + 2 * kTile;  // 2 stages
  uint8_t* sS = sV + 2 * kTile;  // dS
  uint64_t* bar = reinterpret_cast<uint64_t*>(sS + kTile);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;
  uint64_t* k_empty = bar + 3;
  uint64_t* v_full = bar + 5;
  uint64_t* v_empty = bar + 7;
  uint64_t* s_full = bar + 9;
  uint64_t* s_free = bar + 10;
  uint64_t* ds_full = bar + 11;
  uint64_t* ds_free = bar + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);

  const AttnTile tl = a.tiles[blockIdx.x];
  const AttnSeg sg = a.segs[tl.seg];
  const int h = blockIdx.y, g = h / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_row0 = sg.q_start + tl.first;
  const int kv_len = sg.prefix + tl.first + tl.count;
  const int nkt = (kv_len + TK - 1) / TK;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmO);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);  // arrivals count softmax warps
    mbar_init(ds_full, 4);
    mbar_init(ds_free, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256;

  if (warp == 4) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * kTile);
      tma_load_2d(sQ, &tmQ, q_full, h * DH, q_row0);
      tma_load_2d(sQ + kBox, &tmQ, q_full, h * DH + 64, q_row0);
      tma_load_2d(sdO, &tmO, q_full, h * DH, q_row0);
      tma_load_2d(sdO + kBox, &tmO, q_full, h * DH + 64, q_row0);
      for (int j = 0; j < nkt; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        const int krow = sg.kv_row0 + j * TK;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], kTile);
        tma_load_2d(sK + st * kTile, &tmK, &k_full[st], g * DH, krow);
        tma_load_2d(sK + st * kTile + kBox, &tmK, &k_full[st], g * DH + 64, krow);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], kTile);
        tma_load_2d(sV + st * kTile, &tmV, &v_full[st], g * DH, krow);
        tma_load_2d(sV + st * kTile + kBox, &tmV, &v_full[st], g * DH + 64, krow);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idKK = umma_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idKN = umma_idesc_bf16(128, 128, 0, 1);
      const uint32_t q0 = smem_u32(sQ), o0 = smem_u32(sdO), s0 = smem_u32(sS);
      mbar_wait(q_full, 0);
      for (int j = 0; j < nkt; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_full[st], ph);
        mbar_wait(&v_full[st], ph);
        mbar_wait(s_free, (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t k0 = smem_u32(sK + st * kTile), v0 = smem_u32(sV + st * kTile);
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) umma_bf16(tS, kdesc(q0, ks), kdesc(k0, ks), idKK, ks > 0 ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) umma_bf16(tP, kdesc(o0, ks), kdesc(v0, ks), idKK, ks > 0 ? 1u : 0u);
        umma_commit(&v_empty[st]);
        umma_commit(s_full);
        mbar_wait(ds_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < TK / 16; ++ks)
          umma_bf16(tQ, kdesc(s0, ks), mndesc(k0, ks), idKN, (j > 0 || ks > 0) ? 1u : 0u);
        umma_commit(&k_empty[st]);
        umma_commit(ds_free);
      }
    }
  } else {
    const int row = warp * 32 + lane;
    const int qi = tl.first + row;
    const bool ok = qi < sg.len && row < tl.count;
    const int lim = sg.prefix + min(qi, sg.len - 1);
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float lse2 = ok ? a.lse[static_cast<int64_t>(h) * a.T + q_row0 + row] * kLog2e : 0.f;
    const float D = ok ? a.dsum[static_cast<int64_t>(h) * a.T + q_row0 + row] : 0.f;
    for (int j = 0; j < nkt; ++j) {
      // s_full(j) is committed after dQ_{j-1}: the dS buffer is free too.
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      const int key0 = j * TK;
      const bool full = ok && key0 + TK - 1 <= sg.prefix + tl.first;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rs[32], rp[32];
        tmem_ld32(tS + lane_off + c * 32, rs);
        tmem_ld32(tP + lane_off + c * 32, rp);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int k0 = key0 + c * 32 + 2 * e;
          float p0 = exp2f(fmaf(__uint_as_float(rs[2 * e]), a.sl2, -lse2));
          float p1 = exp2f(fmaf(__uint_as_float(rs[2 * e + 1]), a.sl2, -lse2));
          if (!full) {
            p0 = (ok && k0 <= lim) ? p0 : 0.f;
            p1 = (ok && k0 + 1 <= lim) ? p1 : 0.f;
          }
          pk[e] = pack_bf16(p0 * (__uint_as_float(rp[2 * e]) - D), p1 * (__uint_as_float(rp[2 * e + 1]) - D));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(sS + sw128_off(row, 4 * c + q)) =
              make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
      tc_fence_before();
      warp_arrive(s_free);
      fence_async_smem();
      warp_arrive(ds_full);
    }
    mbar_wait(ds_free, (nkt - 1) & 1);
    tc_fence_after();
    __nv_bfloat16* out = a.dq + static_cast<int64_t>(q_row0 + row) * a.dq_stride + h * DH;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(tQ + lane_off + c * 32, r);
      tmem_ld_wait();
      if (ok) {
        uint4* dst = reinterpret_cast<uint4*>(out + c * 32);
        const float sc = a.scale;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_uint4(pack_bf16(__uint_as_float(r[8 * q]) * sc, __uint_as_float(r[8 * q + 1]) * sc),
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

// dK/dV: CTA = 128 keys of one kv head (owner of those rows -> deterministic);
// loops over every q head of the GQA group and every 128-query tile that
// sees the keys: S^T = K Q^T, dP^T = V dO^T -> P^T, dS^T (bf16, smem) ->
// dV += P^T dO, dK += dS^T Q.  Q / dO tiles are used both K-major (first two
// MMAs) and as N-major views (last two) of the same TMA tile.
__global__ void __launch_bounds__(192, 1)
    attn_dkv_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO,
                       const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       TcBwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;
  uint8_t* sV = sK + kTile;
  uint8_t* sQ = sV + kTile;
  uint8_t* sdO = sQ + kTile;
  uint8_t* sP = sdO + kTile;  // P^T
  uint8_t* sS = sP + kTile;   // dS^T
  float* sL = reinterpret_cast<float*>(sS + kTile);  // [2][128] lse*log2e (INF = invalid query)
  float* sD = sL + 256;                              // [2][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + 256);
  uint64_t* kv_full = bar;
  uint64_t* q_full = bar + 1;
  uint64_t* q_empty = bar + 2;
  uint64_t* s_full = bar + 3;
  uint64_t* s_free = bar + 4;
  uint64_t* pds_full = bar + 5;
  uint64_t* pds_free = bar + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);

  const AttnTile tl = a.tiles[blockIdx.x];
  const AttnSeg sg = a.segs[tl.seg];
  const int g = blockIdx.y, per = a.H / a.KVH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int key_first = tl.first;
  const int kv_len = sg.prefix + sg.len;
  const int i0 = max(0, key_first - sg.prefix);
  const int nqt = (sg.len - i0 + TQ - 1) / TQ;
  const int iters = per * nqt;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmO);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(kv_full, 1);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(pds_full, 4);
    mbar_init(pds_free, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tdV = tmem + 256, tdK = tmem + 384;

  if (warp == 4) {
    if (lane == 0) {
      const int krow = sg.kv_row0 + key_first;
      mbar_expect_tx(kv_full, 2 * kTile);
      tma_load_2d(sK, &tmK, kv_full, g * DH, krow);
      tma_load_2d(sK + kBox, &tmK, kv_full, g * DH + 64, krow);
      tma_load_2d(sV, &tmV, kv_full, g * DH, krow);
      tma_load_2d(sV + kBox, &tmV, kv_full, g * DH + 64, krow);
      for (int it = 0; it < iters; ++it) {
        const int hq = g * per + it / nqt;
        const int qrow = sg.q_start + i0 + (it % nqt) * TQ;
        mbar_wait(q_empty, (it & 1) ^ 1);
        mbar_expect_tx(q_full, 2 * kTile);
        tma_load_2d(sQ, &tmQ, q_full, hq * DH, qrow);
        tma_load_2d(sQ + kBox, &tmQ, q_full, hq * DH + 64, qrow);
        tma_load_2d(sdO, &tmO, q_full, hq * DH, qrow);
        tma_load_2d(sdO + kBox, &tmO, q_full, hq * DH + 64, qrow);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idKK = umma_idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idKN = umma_idesc_bf16(128, 128, 0, 1);
      const uint32_t k0 = smem_u32(sK), v0 = smem_u32(sV), q0 = smem_u32(sQ), o0 = smem_u32(sdO);
      const uint32_t p0 = smem_u32(sP), s0 = smem_u32(sS);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < iters; ++it) {
        mbar_wait(q_full, it & 1);
        mbar_wait(s_free, (it & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) umma_bf16(tS, kdesc(k0, ks), kdesc(q0, ks), idKK, ks > 0 ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < DH / 16; ++ks) umma_bf16(tP, kdesc(v0, ks), kdesc(o0, ks), idKK, ks > 0 ? 1u : 0u);
        umma_commit(s_full);
        mbar_wait(pds_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < TQ / 16; ++ks)
          umma_bf16(tdV, kdesc(p0, ks), mndesc(o0, ks), idKN, (it > 0 || ks > 0) ? 1u : 0u);
#pragma unroll
        for (int ks = 0; ks < TQ / 16; ++ks)
          umma_bf16(tdK, kdesc(s0, ks), mndesc(q0, ks), idKN, (it > 0 || ks > 0) ? 1u : 0u);
        umma_commit(q_empty);
        umma_commit(pds_free);
      }
    }
  } else {
    const int row = warp * 32 + lane;  // key row within the tile
    const int key = key_first + row;
    const bool kok = row < tl.count && key < kv_len;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    for (int it = 0; it < iters; ++it) {
      const int hq = g * per + it / nqt;
      const int qt0 = i0 + (it % nqt) * TQ;  // first query of the tile (segment index)
      float* L_ = sL + (it & 1) * 128;
      float* D_ = sD + (it & 1) * 128;
      {
        const int qi = qt0 + row;
        const bool qok = qi < sg.len;
        const int64_t idx = static_cast<int64_t>(hq) * a.T + sg.q_start + qi;
        L_[row] = qok ? a.lse[idx] * kLog2e : INFINITY;
        D_[row] = qok ? a.dsum[idx] : 0.f;
      }
      named_sync_128();
      // s_full(it) is committed after dV/dK of it-1: P^T / dS^T buffers free.
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      // every (key, query) pair of the tile visible and valid -> no masking
      const bool full = key_first + TQ - 1 < kv_len && key_first + TQ - 1 <= sg.prefix + qt0 && qt0 + TQ <= sg.len;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rs[32], rp[32];
        tmem_ld32(tS + lane_off + c * 32, rs);
        tmem_ld32(tP + lane_off + c * 32, rp);
        tmem_ld_wait();
        uint32_t pp[16], pd[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int ql = c * 32 + 2 * e;
          const int qi = qt0 + ql;
          float p0 = exp2f(fmaf(__uint_as_float(rs[2 * e]), a.sl2, -L_[ql]));
          float p1 = exp2f(fmaf(__uint_as_float(rs[2 * e + 1]), a.sl2, -L_[ql + 1]));
          if (!full) {
            p0 = (kok && key <= sg.prefix + qi) ? p0 : 0.f;
            p1 = (kok && key <= sg.prefix + qi + 1) ? p1 : 0.f;
          }
          pp[e] = pack_bf16(p0, p1);
          pd[e] = pack_bf16(p0 * (__uint_as_float(rp[2 * e]) - D_[ql]),
                            p1 * (__uint_as_float(rp[2 * e + 1]) - D_[ql + 1]));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          *reinterpret_cast<uint4*>(sP + sw128_off(row, 4 * c + q)) =
              make_uint4(pp[4 * q], pp[4 * q + 1], pp[4 * q + 2], pp[4 * q + 3]);
          *reinterpret_cast<uint4*>(sS + sw128_off(row, 4 * c + q)) =
              make_uint4(pd[4 * q], pd[4 * q + 1], pd[4 * q + 2], pd[4 * q + 3]);
        }
      }
      tc_fence_before();
      warp_arrive(s_free);
      fence_async_smem();
      warp_arrive(pds_full);
    }
    mbar_wait(pds_free, (iters - 1) & 1);
    tc_fence_after();
    float* dkr = a.dk_acc + static_cast<int64_t>(sg.kv_row0 + key) * a.acc_stride + g * DH;
    float* dvr = a.dv_acc + static_cast<int64_t>(sg.kv_row0 + key) * a.acc_stride + g * DH;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t rk[32], rv[32];
      tmem_ld32(tdK + lane_off + c * 32, rk);
      tmem_ld32(tdV + lane_off + c * 32, rv);
      tmem_ld_wait();
      if (kok) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 ok4 = reinterpret_cast<float4*>(dkr + c * 32)[q];
          ok4.x += __uint_as_float(rk[4 * q]) * a.scale;
          ok4.y += __uint_as_float(rk[4 * q + 1]) * a.scale;
          ok4.z += __uint_as_float(rk[4 * q + 2]) * a.scale;
          ok4.w += __uint_as_float(rk[4 * q + 3]) * a.scale;
          reinterpret_cast<float4*>(dkr + c * 32)[q] = ok4;
          float4 ov = reinterpret_cast<float4*>(dvr + c * 32)[q];
          ov.x += __uint_as_float(rv[4 * q]);
          ov.y += __uint_as_float(rv[4 * q + 1]);
          ov.z += __uint_as_float(rv[4 * q + 2]);
          ov.w += __uint_as_float(rv[4 * q + 3]);
          reinterpret_cast<float4*>(dvr + c * 32)[q] = ov;
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

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

bool map_rows(CUtensorMap* m, const void* ptr, uint64_t cols, uint64_t rows, uint64_t ld) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool attn_tc_supported(const AttnParams& p) {
  return p.dh == 128 && (p.q_stride % 8) == 0 && (p.kv_stride % 8) == 0 &&
         (reinterpret_cast<uintptr_t>(p.q) & 15) == 0 && (reinterpret_cast<uintptr_t>(p.k) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.v) & 15) == 0;
}

cudaError_t attn_forward_tc(const AttnParams& p, const AttnTile* tiles128, int32_t ntiles, int64_t kv_rows,
                            cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  CUtensorMap mq, mk, mv;
  if (!map_rows(&mq, p.q, static_cast<uint64_t>(p.H) * DH, static_cast<uint64_t>(p.T), p.q_stride) ||
      !map_rows(&mk, p.k, static_cast<uint64_t>(p.KVH) * DH, static_cast<uint64_t>(kv_rows), p.kv_stride) ||
      !map_rows(&mv, p.v, static_cast<uint64_t>(p.KVH) * DH, static_cast<uint64_t>(kv_rows), p.kv_stride))
    return cudaErrorInvalidValue;
  TcArgs a{p.segs, tiles128, p.q, p.q_stride, p.o, p.o_stride, p.lse, p.T, p.H, p.KVH, p.scale * kLog2e};
  const size_t smem = 1024 + 2 * KVS * kTile + 512 * 4 + 256;
  // per (kernel, device), thread-safe
  const cudaError_t attr = smem_optin(reinterpret_cast<const void*>(attn_fwd_tc_kernel), static_cast<int>(smem));
  if (attr != cudaSuccess) return attr;
  attn_fwd_tc_kernel<<<dim3(ntiles, p.H), kFwdThreads, smem, st>>>(mq, mk, mv, a);
  return cudaGetLastError();
}

cudaError_t attn_backward_tc_v1(const AttnParams& p, const AttnTile* qtiles128, int32_t nq, const AttnTile* ktiles128,
                             int32_t nk, int64_t kv_rows, cudaStream_t st) {
  if (nq == 0) return cudaSuccess;
  CUtensorMap mq, mo, mk, mv;
  if (!map_rows(&mq, p.q, static_cast<uint64_t>(p.H) * DH, static_cast<uint64_t>(p.T), p.q_stride) ||
      !map_rows(&mo, p.dout, static_cast<uint64_t>(p.H) * DH, static_cast<uint64_t>(p.T), p.dout_stride) ||
      !map_rows(&mk, p.k, static_cast<uint64_t>(p.KVH) * DH, static_cast<uint64_t>(kv_rows), p.kv_stride) ||
      !map_rows(&mv, p.v, static_cast<uint64_t>(p.KVH) * DH, static_cast<uint64_t>(kv_rows), p.kv_stride))
    return cudaErrorInvalidValue;
  TcBwdArgs a{p.segs, qtiles128, p.lse, p.dsum, p.dq, p.dq_stride, p.dk_acc, p.dv_acc, p.acc_stride,
              p.T, p.H, p.KVH, p.scale * kLog2e, p.scale};
  const size_t smem_dq = 1024 + 7 * kTile + 256;
  const size_t smem_dkv = 1024 + 6 * kTile + 4 * 256 * 4 + 128;
  // per (kernel, device), thread-safe
  cudaError_t attr = cudaSuccess;
  if (attr == cudaSuccess) attr = smem_optin(reinterpret_cast<const void*>(attn_dq_tc_kernel), static_cast<int>(smem_dq));
  if (attr == cudaSuccess) attr = smem_optin(reinterpret_cast<const void*>(attn_dkv_tc_kernel), static_cast<int>(smem_dkv));
  if (attr != cudaSuccess) return attr;
  attn_dsum(p, st);
  attn_dq_tc_kernel<<<dim3(nq, p.H), 192, smem_dq, st>>>(mq, mo, mk, mv, a);
  a.tiles = ktiles128;
  if (nk > 0) attn_dkv_tc_kernel<<<dim3(nk, p.KVH), 192, smem_dkv, st>>>(mq, mo, mk, mv, a);
  return cudaGetLastError();
}

}  // namespace cfk
