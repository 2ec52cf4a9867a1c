// tcgen05 attention forward, two q heads per CTA in ping-pong (sm_100a,
// head_dim 128).  Same math as attn_fwd_tc_kernel (attention_tc.cu;
// reference toy_model.hpp:263-302), restructured so the tensor core always
// has the other head's MMAs to run while one head's softmax executes:
//
//   CTA = 128 queries x q heads (h0, h0+1) of one GQA group: both heads
//   stream the SAME K/V tiles (loaded once into a 2-stage smem ring).
//   TMEM (512 cols): head w owns S_w (128 fp32 cols; P_w bf16 is written
//   over its first 64 cols) and O_w (128 cols).  Q_w lives in smem.
//   MMA issue order per key tile j (one thread):
//       [P_0(j)] O_0 += P_0 V_j ; S_0(j+1) = Q_0 K_{j+1}^T ;
//       [P_1(j)] O_1 += P_1 V_j ; S_1(j+1) = Q_1 K_{j+1}^T
//   so softmax_0(j+1) overlaps PV_1(j) + S_1(j+1), and vice versa.  A later
//   MMA into S_w is issued after the PV that read P_w, and tcgen05 MMAs of
//   one thread complete in order, so s_full_w(j) also certifies PV_w(j-1)
//   (O_w stable for the lazy rescale, P_w region free).
//   warps 0-7: softmax of head 0 (two warps per query row, 64 keys each,
//   S read from TMEM once, half-row maxima exchanged through smem); warps
//   8-15: head 1; warp 16: TMA producer; warp 17: MMA issuer.  576 threads
//   cap registers at 96 per thread.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "attention.h"
#include "attention_tc.h"
#include "common.cuh"

namespace cfk {
namespace {

constexpr int TK = 128, DH = 128;
constexpr uint32_t kBox = 128 * 64 * 2;  // [128 rows][64 cols] bf16
constexpr uint32_t kTile = 2 * kBox;     // 128 x 128
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescale = 8.0f;
constexpr int KS = 2, VS = 2;  // K / V ring depths
#ifndef CF_FWD_DIAG
#define CF_FWD_DIAG 0
#endif
constexpr int kThreads = 576;  // 16 softmax warps + TMA + MMA

struct Args {
  const AttnSeg* segs;
  const AttnTile* tiles;
  __nv_bfloat16* o;
  int64_t o_stride;
  float* lse;
  int32_t T, H, KVH;
  float sl2;
};

__device__ __forceinline__ uint64_t kdesc(uint32_t base, int ks) {
  return umma_desc_sw128(base + (ks >> 2) * kBox + (ks & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int ks) {
  return umma_desc_sw128(base + ks * 2048, kBox, 1024);
}
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
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                       // 2 heads
  uint8_t* sK = sQ + 2 * kTile;           // KS stages
  uint8_t* sV = sK + KS * kTile;          // VS stages
  float* sRed = reinterpret_cast<float*>(sV + VS * kTile);  // [2 heads][2 parity][2 half][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRed + 1024);
  uint64_t* q_full = bar;
  uint64_t* k_full = bar + 1;                 // [KS]
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;            // [VS]
  uint64_t* v_empty = v_full + VS;
  uint64_t* s_full = v_empty + VS;            // [2 heads]
  uint64_t* p_full = s_full + 2;              // [2 heads]
  uint64_t* o_done = p_full + 2;              // [2 heads]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const AttnTile tl = a.tiles[blockIdx.x];
  const AttnSeg sg = a.segs[tl.seg];
  const int h0 = 2 * blockIdx.y, g = h0 / (a.H / a.KVH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_row0 = sg.q_start + tl.first;
  const int kv_len = sg.prefix + tl.first + tl.count;
  const int nkt = (kv_len + TK - 1) / TK;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], 8);  // one arrive per softmax warp of the head
      mbar_init(&o_done[w], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 16) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * kTile);
      for (int w = 0; w < 2; ++w) {
        tma_load_2d(sQ + w * kTile, &tmQ, q_full, (h0 + w) * DH, q_row0);
        tma_load_2d(sQ + w * kTile + kBox, &tmQ, q_full, (h0 + w) * DH + 64, q_row0);
      }
      // K runs one tile ahead of V: K_j is needed by S(j) one MMA step
      // before V_j is needed by PV(j)
      auto load_k = [&](int j) {
        const int st = j % KS;
        mbar_wait(&k_empty[st], ((j / KS) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], kTile);
        tma_load_2d(sK + st * kTile, &tmK, &k_full[st], g * DH, sg.kv_row0 + j * TK);
        tma_load_2d(sK + st * kTile + kBox, &tmK, &k_full[st], g * DH + 64, sg.kv_row0 + j * TK);
      };
      load_k(0);
      for (int j = 0; j < nkt; ++j) {
        if (j + 1 < nkt) load_k(j + 1);
        const int st = j % VS;
        mbar_wait(&v_empty[st], ((j / VS) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], kTile);
        tma_load_2d(sV + st * kTile, &tmV, &v_full[st], g * DH, sg.kv_row0 + j * TK);
        tma_load_2d(sV + st * kTile + kBox, &tmV, &v_full[st], g * DH + 64, sg.kv_row0 + j * TK);
      }
    }
  } else if (warp == 17) {
    // whole warp, convergent (elect.sync inside the issue helpers)
    constexpr uint32_t idS = umma_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idO = umma_idesc_bf16(128, 128, 0, 1);
    const uint32_t q0 = smem_u32(sQ);
    const uint32_t bSf = smem_u32(s_full), bPf = smem_u32(p_full), bKf = smem_u32(k_full), bKe = smem_u32(k_empty),
                   bVf = smem_u32(v_full), bVe = smem_u32(v_empty), bOd = smem_u32(o_done);
    // S_w = Q_w K_j^T: K = dh in two 4-MMA chains (one 64-column box each)
    auto issue_s = [&](int w, int j) {
      const uint32_t k0 = smem_u32(sK + (j % KS) * kTile);
      const uint32_t qw = q0 + w * kTile;
      umma4_ss_w<2, 2>(tmem + 256 * w, kdesc(qw, 0), kdesc(k0, 0), idS, 0u);
      umma4_ss_w<2, 2>(tmem + 256 * w, kdesc(qw, 4), kdesc(k0, 4), idS, 1u);
      umma_commit_w(bSf + w * 8);
    };
    mbar_wait(q_full, 0);
    mbar_wait_s(bKf, 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    umma_commit_w(bKe);
    for (int j = 0; j < nkt; ++j) {
      const int sv = j % VS;
      const bool more = j + 1 < nkt;
      const int sk = (j + 1) % KS;
      const uint32_t v0 = smem_u32(sV + sv * kTile);
      for (int w = 0; w < 2; ++w) {
        mbar_wait_s(bPf + w * 8, j & 1);
        if (w == 0) mbar_wait_s(bVf + sv * 8, (j / VS) & 1);
        tc_fence_after();
        const uint32_t tS = tmem + 256 * w, tO = tS + 128;
        // O_w += P_w V_j (P in TMEM over S_w), K = 128 keys in two chains
        umma4_ts_w<8, 128>(tO, tS, mndesc(v0, 0), idO, j > 0 ? 1u : 0u);
        umma4_ts_w<8, 128>(tO, tS + 32, mndesc(v0, 4), idO, 1u);
        if (w == 1) umma_commit_w(bVe + sv * 8);
        if (more) {
          if (w == 0) {
            mbar_wait_s(bKf + sk * 8, ((j + 1) / KS) & 1);
            tc_fence_after();
          }
          issue_s(w, j + 1);
          if (w == 1) umma_commit_w(bKe + sk * 8);
        } else {
          umma_commit_w(bOd + w * 8);
        }
      }
    }
  } else {
    // softmax: warps 0-7 head h0, warps 8-15 head h0+1; two warps per query
    // row (warp w and w+4 of a head share TMEM lanes), 64 keys each
    const int w = warp >> 3, quarter = warp & 3, half = (warp >> 2) & 1;
    const int row = quarter * 32 + lane;
    const int qi = tl.first + row;
    const int lim = sg.prefix + min(qi, sg.len - 1);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + 256 * w + lane_off, tO = tS + 128;
    const uint32_t red = smem_u32(sRed) + w * 2048;  // [2 parity][2 half][128 rows] per head
    const float sl2 = a.sl2;
    float m = -FLT_MAX, l = 0.f;
    for (int j = 0; j < nkt; ++j) {
      mbar_wait(&s_full[w], j & 1);
      tc_fence_after();
#if CF_FWD_DIAG  // diagnostics: softmax side skipped (MMA + TMA pipeline only)
      tc_fence_before();
      warp_arrive(&p_full[w]);
      continue;
#endif
      const int key0 = j * TK + half * 64;
      const bool full = j * TK + TK - 1 <= sg.prefix + tl.first;
      // this half-row of S, read from TMEM once (kept as raw bits)
      uint32_t r[2][32];
      tmem_ld32(tS + half * 64, r[0]);
      tmem_ld32(tS + half * 64 + 32, r[1]);
      tmem_ld_wait();
      if (!full) {
#pragma unroll
        for (int e = 0; e < 64; ++e)
          if (key0 + e > lim) r[e >> 5][e & 31] = 0xff7fffffu;  // -FLT_MAX: ex2 underflows to 0
      }
      float pm[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
#pragma unroll
      for (int e = 0; e < 64; ++e) pm[e & 3] = fmaxf(pm[e & 3], __uint_as_float(r[e >> 5][e & 31]));
      float tmax = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3]));
      // exchange half-row maxima with the partner warp; after this barrier
      // both halves hold their S values, so P may overwrite any S column
      sts_f32(red + (j & 1) * 1024 + (half * 128 + row) * 4, tmax);
      asm volatile("bar.sync %0, 64;" ::"r"(1 + w * 4 + quarter) : "memory");
      tmax = fmaxf(tmax, lds_f32(red + (j & 1) * 1024 + ((half ^ 1) * 128 + row) * 4)) * sl2;  // sl2 > 0
      float alpha = 1.f;
      bool rescale = false;
      if (tmax > m + kRescale || j == 0) {
        const float mn = fmaxf(m, tmax);
        alpha = ex2(m - mn);
        rescale = j > 0;
        m = mn;
      }
      // pairs of scores in FFMA2 (x = s * sl2 - m); the row sum keeps the
      // scalar order (ps[e & 3] += p0 + p1) so l stays bitwise what the
      // operator-level segment path reproduces
      float ps[4] = {0.f, 0.f, 0.f, 0.f};
      const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m, -m);
      // P (bf16 pairs) over S columns [0, 64), stored per 32-key half as soon
      // as it is packed, so a half's S registers die early (no spills)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float2 x = ffma2(make_float2(__uint_as_float(r[hh][2 * e]), __uint_as_float(r[hh][2 * e + 1])),
                                 sl2v, nm);
          const float2 p = make_float2(ex2(x.x), ex2(x.y));
          ps[e & 3] += p.x + p.y;
          pk[e] = pack_bf16(p.x, p.y);
        }
        tmem_st16(tS + half * 32 + hh * 16, pk);
      }
      l = fmaf(l, alpha, (ps[0] + ps[1]) + (ps[2] + ps[3]));
      if (rescale) {  // after P (S registers dead); PV_w(j-1) is complete (s_full_w(j) followed it)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld32(tO + half * 64 + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 v = fmul2(make_float2(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])),
                                   make_float2(alpha, alpha));
            r[2 * e] = __float_as_uint(v.x);
            r[2 * e + 1] = __float_as_uint(v.y);
          }
          tmem_st32(tO + half * 64 + c * 32, r);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      warp_arrive(&p_full[w]);
    }
    // combine the half-row sums (the pair re-syncs before the buffer is reused)
    sts_f32(red + (nkt & 1) * 1024 + (half * 128 + row) * 4, l);
    asm volatile("bar.sync %0, 64;" ::"r"(1 + w * 4 + quarter) : "memory");
    l += lds_f32(red + (nkt & 1) * 1024 + ((half ^ 1) * 128 + row) * 4);
    mbar_wait(&o_done[w], 0);
    tc_fence_after();
    const int h = h0 + w;
    const bool ok = qi < sg.len && row < tl.count;
    const float inv = 1.f / l;
    __nv_bfloat16* orow =
        a.o + static_cast<int64_t>(q_row0 + row) * a.o_stride + static_cast<int64_t>(h) * DH + half * 64;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t r[32];
      tmem_ld32(tO + half * 64 + c * 32, r);
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

// ---------------------------------------------------------------- persistent
// attn_fwd_pp_kernel's math with one CTA per SM looping over items.  Built
// for packed short-sequence chunks, where an item (128-query tile x head
// pair) sees only a few key tiles and a one-CTA-per-item grid spends most of
// each CTA in its prologue (TMEM / barrier set-up, the Q fetch from HBM) and
// epilogue; it also wins on long-context launches (hidden Q fetches).  One CTA per SM loops over items
// (snake_item order over tile-major items, the heaviest tiles of every head
// pair first); ring positions and barrier phases run on
// counters that continue across items:
//   * Q(n+1) is fetched as soon as item n's last S MMAs have read Q(n)
//     (q_empty), i.e. during item n's last softmax, PV and epilogue;
//   * S_w(n+1, 0) is issued straight after PV_w(n, last) (tcgen05 MMAs of one
//     thread complete in order, so P_w(n, last) has been consumed);
//   * PV_w(n+1, 0) overwrites O_w, so it waits for o_free_w: the softmax
//     warps' read-out of O_w(n).
// Per item, every value is computed in the same order as attn_fwd_pp_kernel,
// so the two kernels' outputs are bitwise equal.
// The item a persistent CTA takes in round r: boustrophedon order over the
// grid (even rounds ascending, odd rounds descending), so with items sorted
// by decreasing work each CTA's total stays close to the mean (plain
// round-robin hands CTA 0 the heaviest item of every round).
__device__ __forceinline__ int snake_item(int r) {
  const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
  return r * G + ((r & 1) ? G - 1 - b : b);
}
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_pp_persist_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                               const __grid_constant__ CUtensorMap tmV, Args a, int ntiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + 2 * kTile;
  uint8_t* sV = sK + KS * kTile;
  float* sRed = reinterpret_cast<float*>(sV + VS * kTile);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRed + 1024);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;                 // [KS]
  uint64_t* k_empty = k_full + KS;
  uint64_t* v_full = k_empty + KS;            // [VS]
  uint64_t* v_empty = v_full + VS;
  uint64_t* s_full = v_empty + VS;            // [2 heads]
  uint64_t* p_full = s_full + 2;              // [2 heads]
  uint64_t* o_done = p_full + 2;              // [2 heads]
  uint64_t* o_free = o_done + 2;              // [2 heads]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 2);

  const int hp = a.H / 2;  // head pairs
  const int items = ntiles * hp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto item_of = [&](int it, AttnTile& tl, AttnSeg& sg, int& h0) {
    const int t = it / hp;
    h0 = 2 * (it - t * hp);
    tl = a.tiles[t];
    sg = a.segs[tl.seg];
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], 8);
      mbar_init(&o_done[w], 1);
      mbar_init(&o_free[w], 8);  // one arrive per softmax warp of the head
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 16) {
    if (lane == 0) {
      int jk = 0, jv = 0, n = 0;  // K / V ring positions, item count
      for (int it = snake_item(0); it < items; it = snake_item(++n)) {
        AttnTile tl;
        AttnSeg sg;
        int h0;
        item_of(it, tl, sg, h0);
        const int g = h0 / (a.H / a.KVH);
        const int nkt = (sg.prefix + tl.first + tl.count + TK - 1) / TK;
        const int q_row0 = sg.q_start + tl.first;
        mbar_wait(q_empty, (n & 1) ^ 1);
        mbar_expect_tx(q_full, 2 * kTile);
        for (int w = 0; w < 2; ++w) {
          tma_load_2d(sQ + w * kTile, &tmQ, q_full, (h0 + w) * DH, q_row0);
          tma_load_2d(sQ + w * kTile + kBox, &tmQ, q_full, (h0 + w) * DH + 64, q_row0);
        }
        auto load_k = [&](int j) {
          const int st = jk % KS;
          mbar_wait(&k_empty[st], ((jk / KS) & 1) ^ 1);
          mbar_expect_tx(&k_full[st], kTile);
          tma_load_2d(sK + st * kTile, &tmK, &k_full[st], g * DH, sg.kv_row0 + j * TK);
          tma_load_2d(sK + st * kTile + kBox, &tmK, &k_full[st], g * DH + 64, sg.kv_row0 + j * TK);
          ++jk;
        };
        load_k(0);
        for (int j = 0; j < nkt; ++j) {
          if (j + 1 < nkt) load_k(j + 1);
          const int st = jv % VS;
          mbar_wait(&v_empty[st], ((jv / VS) & 1) ^ 1);
          mbar_expect_tx(&v_full[st], kTile);
          tma_load_2d(sV + st * kTile, &tmV, &v_full[st], g * DH, sg.kv_row0 + j * TK);
          tma_load_2d(sV + st * kTile + kBox, &tmV, &v_full[st], g * DH + 64, sg.kv_row0 + j * TK);
          ++jv;
        }
      }
    }
  } else if (warp == 17) {
    constexpr uint32_t idS = umma_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t idO = umma_idesc_bf16(128, 128, 0, 1);
    const uint32_t q0 = smem_u32(sQ);
    const uint32_t bSf = smem_u32(s_full), bPf = smem_u32(p_full), bKf = smem_u32(k_full), bKe = smem_u32(k_empty),
                   bVf = smem_u32(v_full), bVe = smem_u32(v_empty), bOd = smem_u32(o_done),
                   bOr = smem_u32(o_free), bQf = smem_u32(q_full), bQe = smem_u32(q_empty);
    int jk = 0, jv = 0, J = 0, n = 0;  // K / V ring positions, key tiles so far, items so far
    auto issue_s = [&](int w) {
      const uint32_t k0 = smem_u32(sK + (jk % KS) * kTile);
      const uint32_t qw = q0 + w * kTile;
      umma4_ss_w<2, 2>(tmem + 256 * w, kdesc(qw, 0), kdesc(k0, 0), idS, 0u);
      umma4_ss_w<2, 2>(tmem + 256 * w, kdesc(qw, 4), kdesc(k0, 4), idS, 1u);
      umma_commit_w(bSf + w * 8);
    };
    for (int it = snake_item(0); it < items; it = snake_item(++n)) {
      AttnTile tl;
      AttnSeg sg;
      int h0;
      item_of(it, tl, sg, h0);
      const int nkt = (sg.prefix + tl.first + tl.count + TK - 1) / TK;
      mbar_wait_s(bQf, n & 1);
      mbar_wait_s(bKf + (jk % KS) * 8, (jk / KS) & 1);
      tc_fence_after();
      issue_s(0);
      issue_s(1);
      umma_commit_w(bKe + (jk % KS) * 8);
      ++jk;
      if (nkt == 1) umma_commit_w(bQe);
      for (int j = 0; j < nkt; ++j, ++J) {
        const int sv = jv % VS;
        const bool more = j + 1 < nkt;
        const uint32_t v0 = smem_u32(sV + sv * kTile);
        for (int w = 0; w < 2; ++w) {
          mbar_wait_s(bPf + w * 8, J & 1);
          if (w == 0) mbar_wait_s(bVf + sv * 8, (jv / VS) & 1);
          if (j == 0 && n > 0) mbar_wait_s(bOr + w * 8, (n - 1) & 1);  // O_w of the previous item read out
          tc_fence_after();
          const uint32_t tS = tmem + 256 * w, tO = tS + 128;
          umma4_ts_w<8, 128>(tO, tS, mndesc(v0, 0), idO, j > 0 ? 1u : 0u);
          umma4_ts_w<8, 128>(tO, tS + 32, mndesc(v0, 4), idO, 1u);
          if (w == 1) umma_commit_w(bVe + sv * 8);
          if (more) {
            if (w == 0) {
              mbar_wait_s(bKf + (jk % KS) * 8, (jk / KS) & 1);
              tc_fence_after();
            }
            issue_s(w);
            if (w == 1) {
              umma_commit_w(bKe + (jk % KS) * 8);
              ++jk;
              if (j + 2 == nkt) umma_commit_w(bQe);  // the item's last S MMAs: Q may be refilled
            }
          } else {
            umma_commit_w(bOd + w * 8);
          }
        }
        ++jv;
      }
    }
  } else {
    const int w = warp >> 3, quarter = warp & 3, half = (warp >> 2) & 1;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tmem + 256 * w + lane_off, tO = tS + 128;
    const uint32_t red = smem_u32(sRed) + w * 2048;  // [2 parity][2 half][128 rows] per head
    const float sl2 = a.sl2;
    // key tiles so far, items so far; half-row exchanges so far = J + n (one
    // per key tile and one per item), their parity picks the smem buffer
    int J = 0, n = 0;
    for (int it = snake_item(0); it < items; it = snake_item(++n)) {
      int nkt, lim, tile_lo;
      {
        AttnTile tl;
        AttnSeg sg;
        int h0;
        item_of(it, tl, sg, h0);
        nkt = (sg.prefix + tl.first + tl.count + TK - 1) / TK;
        lim = sg.prefix + min(tl.first + row, sg.len - 1);
        tile_lo = sg.prefix + tl.first;
      }
      float m = -FLT_MAX, l = 0.f;
      for (int j = 0; j < nkt; ++j, ++J) {
        mbar_wait(&s_full[w], J & 1);
        tc_fence_after();
        const int key0 = j * TK + half * 64;
        const bool full = j * TK + TK - 1 <= tile_lo;
        uint32_t r[2][32];
        tmem_ld32(tS + half * 64, r[0]);
        tmem_ld32(tS + half * 64 + 32, r[1]);
        tmem_ld_wait();
        if (!full) {
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (key0 + e > lim) r[e >> 5][e & 31] = 0xff7fffffu;
        }
        float pm[4] = {-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX};
#pragma unroll
        for (int e = 0; e < 64; ++e) pm[e & 3] = fmaxf(pm[e & 3], __uint_as_float(r[e >> 5][e & 31]));
        float tmax = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3]));
        const uint32_t xb = red + ((J + n) & 1) * 1024;
        sts_f32(xb + (half * 128 + row) * 4, tmax);
        asm volatile("bar.sync %0, 64;" ::"r"(1 + w * 4 + quarter) : "memory");
        tmax = fmaxf(tmax, lds_f32(xb + ((half ^ 1) * 128 + row) * 4)) * sl2;
        float alpha = 1.f;
        bool rescale = false;
        if (tmax > m + kRescale || j == 0) {
          const float mn = fmaxf(m, tmax);
          alpha = ex2(m - mn);
          rescale = j > 0;
          m = mn;
        }
        float ps[4] = {0.f, 0.f, 0.f, 0.f};
        const float2 sl2v = make_float2(sl2, sl2), nm = make_float2(-m, -m);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 xx = ffma2(make_float2(__uint_as_float(r[hh][2 * e]), __uint_as_float(r[hh][2 * e + 1])),
                                    sl2v, nm);
            const float2 p = make_float2(ex2(xx.x), ex2(xx.y));
            ps[e & 3] += p.x + p.y;
            pk[e] = pack_bf16(p.x, p.y);
          }
          tmem_st16(tS + half * 32 + hh * 16, pk);
        }
        l = fmaf(l, alpha, (ps[0] + ps[1]) + (ps[2] + ps[3]));
        if (rescale) {
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t rr[32];
            tmem_ld32(tO + half * 64 + c * 32, rr);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float2 v = fmul2(make_float2(__uint_as_float(rr[2 * e]), __uint_as_float(rr[2 * e + 1])),
                                     make_float2(alpha, alpha));
              rr[2 * e] = __float_as_uint(v.x);
              rr[2 * e + 1] = __float_as_uint(v.y);
            }
            tmem_st32(tO + half * 64 + c * 32, rr);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        warp_arrive(&p_full[w]);
      }
      const uint32_t xb = red + ((J + n) & 1) * 1024;
      sts_f32(xb + (half * 128 + row) * 4, l);
      asm volatile("bar.sync %0, 64;" ::"r"(1 + w * 4 + quarter) : "memory");
      l += lds_f32(xb + ((half ^ 1) * 128 + row) * 4);
      mbar_wait(&o_done[w], n & 1);
      tc_fence_after();
      // the item's rows / head, re-read here so they are not live across the
      // key loop (register budget: 96 per thread at 576 threads)
      AttnTile tl;
      AttnSeg sg;
      int h0;
      item_of(it, tl, sg, h0);
      const int q_row0 = sg.q_start + tl.first;
      const int h = h0 + w;
      const bool ok = tl.first + row < sg.len && row < tl.count;
      const float inv = 1.f / l;
      __nv_bfloat16* orow =
          a.o + static_cast<int64_t>(q_row0 + row) * a.o_stride + static_cast<int64_t>(h) * DH + half * 64;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t ro[32];
        tmem_ld32(tO + half * 64 + c * 32, ro);
        tmem_ld_wait();
        if (c == 1) {
          tc_fence_before();
          warp_arrive(&o_free[w]);  // O_w may be overwritten by the next item's first PV
        }
        if (ok) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[q] = make_uint4(pack_bf16(__uint_as_float(ro[8 * q]) * inv, __uint_as_float(ro[8 * q + 1]) * inv),
                                pack_bf16(__uint_as_float(ro[8 * q + 2]) * inv, __uint_as_float(ro[8 * q + 3]) * inv),
                                pack_bf16(__uint_as_float(ro[8 * q + 4]) * inv, __uint_as_float(ro[8 * q + 5]) * inv),
                                pack_bf16(__uint_as_float(ro[8 * q + 6]) * inv, __uint_as_float(ro[8 * q + 7]) * inv));
        }
      }
      if (ok) {
        if (half == 0) a.lse[static_cast<int64_t>(h) * a.T + q_row0 + row] = (m + log2f(l)) * kLn2;
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

bool map_rows(CUtensorMap* m, const void* ptr, uint64_t cols, uint64_t rows, uint64_t ld) {
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
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int attn_num_sms();  // attention_tc_bwd.cu

// The persistent forward serves every launch: packed short chunks -11..-25 %,
// causal T = 16K -4 % (1.88 -> 1.80 ms), the C2 long group's chunks +1.8 %
// TFLOP/s in-step (profiles/round2_ab_short_attention.txt,
// profiles/round2_ab_fwd_persist_long.txt).  CF_FWD_PERSIST=0 selects the
// one-CTA-per-item kernel (A/B, tests).
bool fwd_persist(const AttnParams&) {
  static const int v = [] {
    const char* e = std::getenv("CF_FWD_PERSIST");
    return e ? std::atoi(e) : -1;
  }();
  return v != 0;
}

bool attn_fwd_pp_supported(const AttnParams& p) {
  return attn_tc_supported(p) && (p.H / p.KVH) % 2 == 0 && (reinterpret_cast<uintptr_t>(p.q) & 15) == 0;
}

cudaError_t attn_forward_tc_pp(const AttnParams& p, const AttnTile* tiles128, int32_t ntiles, int64_t kv_rows,
                               cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  if (!attn_fwd_pp_supported(p)) return cudaErrorInvalidValue;
  CUtensorMap mq, mk, mv;
  if (!map_rows(&mq, p.q, static_cast<uint64_t>(p.H) * DH, static_cast<uint64_t>(p.T), p.q_stride) ||
      !map_rows(&mk, p.k, static_cast<uint64_t>(p.KVH) * DH, static_cast<uint64_t>(kv_rows), p.kv_stride) ||
      !map_rows(&mv, p.v, static_cast<uint64_t>(p.KVH) * DH, static_cast<uint64_t>(kv_rows), p.kv_stride))
    return cudaErrorInvalidValue;
  Args a{p.segs, tiles128, p.o, p.o_stride, p.lse, p.T, p.H, p.KVH, p.scale * kLog2e};
  const size_t smem = 1024 + (2 + KS + VS) * kTile + 1024 * 4 + 256;
  // per (kernel, device), thread-safe
  if (fwd_persist(p)) {
    const cudaError_t attr =
        smem_optin(reinterpret_cast<const void*>(attn_fwd_pp_persist_kernel), static_cast<int>(smem));
    if (attr != cudaSuccess) return attr;
    const int items = ntiles * (p.H / 2);
    attn_fwd_pp_persist_kernel<<<std::min(items, attn_num_sms()), kThreads, smem, st>>>(mq, mk, mv, a, ntiles);
    return cudaGetLastError();
  }
  const cudaError_t attr = smem_optin(reinterpret_cast<const void*>(attn_fwd_pp_kernel), static_cast<int>(smem));
  if (attr != cudaSuccess) return attr;
  attn_fwd_pp_kernel<<<dim3(ntiles, p.H / 2), kThreads, smem, st>>>(mq, mk, mv, a);
  return cudaGetLastError();
}

}  // namespace cfk
