// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] (op)= sum_k A(m,k) * B(n,k)          bf16 x bf16 -> fp32 in TMEM
//
// A is K-major ([M,K] row-major, activations) or M-major ([K,M] row-major,
// i.e. a transposed view of activations for weight gradients); B is K-major
// ([N,K]) or N-major ([K,N], the reference's [in,out] weight layout).  Both
// majors are fed by TMA with 128B swizzle straight into the UMMA canonical
// layouts, so no transpose kernels exist anywhere on the path.
//
// Roles (256 threads, 1 CTA/SM, grid = min(tiles, #SM)):
//   warp 0      TMA producer  (one lane)   smem ring of kStages A/B stages
//   warp 1      MMA issuer    (one lane)   tcgen05.mma 128xBNx16, fp32 accum
//   warp 2      TMEM allocator             2 accumulator buffers (2*BN cols)
//   warps 4-7   epilogue                   tcgen05.ld -> fused op -> global
// The epilogue of tile i overlaps the main loop of tile i+1 through the two
// TMEM accumulators (tmem_full / tmem_empty mbarriers).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gemm.h"

namespace cfk {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr uint32_t kSlab = 64 * BK * 2;  // one 64-wide MN slab x BK rows = 8 KiB

template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr uint32_t kABytes = BM * BK * 2;
  static constexpr uint32_t kBBytes = BN * BK * 2;
  static constexpr uint32_t kTmemCols = 2 * BN;
  static constexpr size_t kSmem = 1024 + kStages * (kABytes + kBBytes) + 256;
};

struct Args {
  int M, N, K;
  int num_m, num_n, num_k;
  void* C;
  int64_t ldc;
  const void* R;  // fp32 residual (EPI_F32_RES) or bf16 aux (EPI_BF16_TANHGRAD)
  int64_t ldr;
  int group_m;  // raster: tiles walk group_m M-blocks x all N-blocks, M fastest
  int serp;     // CTA-pair kernel: odd waves walk K backwards (see gemm_pair_kernel)
  int split_n;  // EPI_BF16_SWIGLU: F (the up half starts at column F)
  int col_k, col_v;  // EPI_BF16_ROPE
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  int64_t cache_ld;
  // EPI_CE_STATS / EPI_CE_GRAD
  const int32_t* ce_tgt;
  float2* ce_part;
  float* ce_tlogit;
  const float* ce_lse;
  float ce_scale;
  int ce_nparts;
};

// Grouped raster.  Persistent CTAs take consecutive tile indices, so one wave
// is a contiguous index range; walking group_m M-blocks at a time makes that
// range a near-square block of the output (e.g. 8 x 9 for 74 pairs), and the
// operand slabs it streams are shared by ~8 tiles each in L2 instead of the
// M operand being re-read from HBM once per wave.
__device__ __forceinline__ void tile_coords(const Args& g, int tile, int& mb, int& nb) {
  const int per_group = g.group_m * g.num_n;
  const int first_m = (tile / per_group) * g.group_m;
  const int gm = min(g.num_m - first_m, g.group_m);
  const int r = tile - (tile / per_group) * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

template <int EPI>
__device__ __forceinline__ void store_row32(const Args& g, int row, int col0, const uint32_t (&r)[32]) {
  if (row >= g.M) return;
  const bool full = col0 + 32 <= g.N;
  if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_TANH || EPI == EPI_BF16_TANHGRAD) {
    __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(g.C) + static_cast<int64_t>(row) * g.ldc + col0;
    const __nv_bfloat16* aux = nullptr;
    if constexpr (EPI == EPI_BF16_TANHGRAD)
      aux = reinterpret_cast<const __nv_bfloat16*>(g.R) + static_cast<int64_t>(row) * g.ldr + col0;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float x = __uint_as_float(r[j]);
      if constexpr (EPI == EPI_BF16_TANH) x = tanhf(x);
      if constexpr (EPI == EPI_BF16_TANHGRAD) {
        if (full || col0 + j < g.N) {
          const float h = __bfloat162float(aux[j]);
          x = x * (1.0f - h * h);
        }
      }
      v[j] = x;
    }
    if (full) {
      uint4* dst = reinterpret_cast<uint4*>(c);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        dst[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                            pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < g.N) c[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* c = reinterpret_cast<float*>(g.C) + static_cast<int64_t>(row) * g.ldc + col0;
    const float* res = nullptr;
    if constexpr (EPI == EPI_F32_RES) res = reinterpret_cast<const float*>(g.R) + static_cast<int64_t>(row) * g.ldr + col0;
    if (full) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 v = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                               __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
        if constexpr (EPI == EPI_F32_ACC) {
          const float4 o = reinterpret_cast<const float4*>(c)[q];
          v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        }
        if constexpr (EPI == EPI_F32_RES) {
          const float4 o = reinterpret_cast<const float4*>(res)[q];
          v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        }
        reinterpret_cast<float4*>(c)[q] = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col0 + j >= g.N) continue;
        float x = __uint_as_float(r[j]);
        if constexpr (EPI == EPI_F32_ACC) x += c[j];
        if constexpr (EPI == EPI_F32_RES) x += res[j];
        c[j] = x;
      }
    }
  }
}

// EPI_CE_STATS: fold 32 logits of one row into the running (max, sum exp) of
// the tile's 256-column slab; the target column's logit is written once.
__device__ __forceinline__ void ce_stats_row32(const Args& g, int row, int col0, const uint32_t (&r)[32], int tgt,
                                               float& m, float& s) {
  float cm = -INFINITY;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (col0 + j < g.N) cm = fmaxf(cm, __uint_as_float(r[j]));
  if (tgt >= col0 && tgt < col0 + 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j == tgt) g.ce_tlogit[row] = __uint_as_float(r[j]);
  }
  if (cm == -INFINITY) return;
  const float nm = fmaxf(m, cm);
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (col0 + j < g.N) acc += __expf(__uint_as_float(r[j]) - nm);
  s = s * __expf(m - nm) + acc;
  m = nm;
}

// EPI_CE_GRAD: dlogits of 32 columns of one row from the saved LSE.
__device__ __forceinline__ void ce_grad_row32(const Args& g, int row, int col0, const uint32_t (&r)[32], int tgt,
                                              float lse) {
  __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(g.C) + static_cast<int64_t>(row) * g.ldc + col0;
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float p = __expf(__uint_as_float(r[j]) - lse) - (col0 + j == tgt ? 1.f : 0.f);
    v[j] = tgt >= 0 ? p * g.ce_scale : 0.f;
  }
  if (col0 + 32 <= g.N) {
    uint4* dst = reinterpret_cast<uint4*>(c);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      dst[q] = make_uint4(pack_bf16(v[8 * q + 0], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                          pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < g.N) c[j] = __float2bfloat16_rn(v[j]);
  }
}

template <int EPI>
constexpr bool kEpiCe = EPI == EPI_CE_STATS || EPI == EPI_CE_GRAD;

// Epilogues that read a fp32 row segment (residual R or the accumulated C)
// prefetch the next 32-column chunk while the current one is stored: the
// per-row loads otherwise serialise one DRAM latency per chunk.
template <int EPI>
constexpr bool kEpiReads = EPI == EPI_F32_RES || EPI == EPI_F32_ACC;

template <int EPI>
__device__ __forceinline__ void prefetch_row32(const Args& g, int row, int col0, float4 (&v)[8]) {
  if (row >= g.M || col0 >= g.N) return;
  const float* src = EPI == EPI_F32_RES ? reinterpret_cast<const float*>(g.R) + static_cast<int64_t>(row) * g.ldr + col0
                                        : reinterpret_cast<const float*>(g.C) + static_cast<int64_t>(row) * g.ldc + col0;
  if (col0 + 32 <= g.N) {
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = reinterpret_cast<const float4*>(src)[q];
  } else {
    float* f = reinterpret_cast<float*>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) f[j] = col0 + j < g.N ? src[j] : 0.f;
  }
}

// fp32 store of acc + v (v = prefetched residual or previous C)
template <int EPI>
__device__ __forceinline__ void store_row32_pre(const Args& g, int row, int col0, const uint32_t (&r)[32],
                                                const float4 (&v)[8]) {
  if (row >= g.M) return;
  float* c = reinterpret_cast<float*>(g.C) + static_cast<int64_t>(row) * g.ldc + col0;
  if (col0 + 32 <= g.N) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 o = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                             __uint_as_float(r[4 * q + 3]));
      o.x += v[q].x;
      o.y += v[q].y;
      o.z += v[q].z;
      o.w += v[q].w;
      reinterpret_cast<float4*>(c)[q] = o;
    }
  } else {
    const float* f = reinterpret_cast<const float*>(v);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col0 + j < g.N) c[j] = __uint_as_float(r[j]) + f[j];
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Args g) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = g.num_m * g.num_n;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(g, tile, mb, nb);
        for (int kb = 0; kb < g.num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * C::kABytes;
          uint8_t* b = sB + stage * C::kBBytes;
          mbar_expect_tx(&full[stage], C::kABytes + C::kBBytes);
          if constexpr (!A_MN) {
            tma_load_2d(a, &tmA, &full[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(a + j * kSlab, &tmA, &full[stage], mb * BM + j * 64, kb * BK);
          }
          if constexpr (!B_MN) {
            tma_load_2d(b, &tmB, &full[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(b + j * kSlab, &tmB, &full[stage], nb * BN + j * 64, kb * BK);
          }
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < g.num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * C::kABytes);
          const uint32_t b0 = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a0 + k * 2048, kSlab, 1024) : umma_desc_sw128(a0 + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(b0 + k * 2048, kSlab, 1024) : umma_desc_sw128(b0 + k * 32, 16, 1024);
            umma_bf16(d, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      int mb, nb;
      tile_coords(g, tile, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mb * BM + ew * 32 + lane;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * BN);
      if constexpr (kEpiCe<EPI>) {
        static_assert(!kEpiCe<EPI> || BN == 256, "CE epilogues use 256-column slabs");
        const int tgt = row < g.M ? g.ce_tgt[row] : -1;
        const float lse = (EPI == EPI_CE_GRAD && row < g.M) ? g.ce_lse[row] : 0.f;
        float m = -INFINITY, sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          tmem_ld_wait();
          if (c == BN / 32 - 1) {
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
          }
          const int col0 = nb * BN + c * 32;
          if (row < g.M && col0 < g.N) {
            if constexpr (EPI == EPI_CE_STATS)
              ce_stats_row32(g, row, col0, r, tgt, m, sum);
            else
              ce_grad_row32(g, row, col0, r, tgt, lse);
          }
        }
        if constexpr (EPI == EPI_CE_STATS)
          if (row < g.M) g.ce_part[static_cast<int64_t>(row) * g.ce_nparts + nb] = make_float2(m, sum);
      } else {
        float4 pre[8];
        if constexpr (kEpiReads<EPI>) prefetch_row32<EPI>(g, row, nb * BN, pre);
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          tmem_ld_wait();
          if (c == BN / 32 - 1) {
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
          }
          const int col0 = nb * BN + c * 32;
          if constexpr (kEpiReads<EPI>) {
            float4 nxt[8];
            if (c + 1 < BN / 32) prefetch_row32<EPI>(g, row, col0 + 32, nxt);
            if (col0 < g.N) store_row32_pre<EPI>(g, row, col0, r, pre);
#pragma unroll
            for (int q = 0; q < 8; ++q) pre[q] = nxt[q];
          } else {
            if (col0 < g.N) store_row32<EPI>(g, row, col0, r);
          }
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_free<C::kTmemCols>(tmem_base);
  }
}

// ----------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile.  CTA r loads A rows [m0 + 128r, +128) and B rows (N) [n0 +
// 128r, +128); the leader issues tcgen05.mma.cta_group::2 (M256 N256 K16) and
// each CTA's TMEM receives its own 128 rows x 256 columns.  Per SM this halves
// the shared-memory bytes written by TMA and read by the tensor core per FLOP
// (64 + 64 B/clk instead of 96 + 96 B/clk at full MMA rate), which is what
// caps the single-CTA kernel at ~2/3 of the per-clock tensor peak.
// EPI_BF16_SWIGLU store of 32 columns: gate and up (bf16) to C at col0 and
// F + col0, h = silu(g) * u of the rounded values to H (= R) at col0.
__device__ __forceinline__ void swiglu_store_row32(const Args& g, int row, int col0, const uint32_t (&rg)[32],
                                                   const uint32_t (&ru)[32]) {
  __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(g.C) + static_cast<int64_t>(row) * g.ldc + col0;
  __nv_bfloat16* h = const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(g.R)) +
                     static_cast<int64_t>(row) * g.ldr + col0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t pg[4], pu[4], ph[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = 8 * q + 2 * e;
      pg[e] = pack_bf16(__uint_as_float(rg[j]), __uint_as_float(rg[j + 1]));
      pu[e] = pack_bf16(__uint_as_float(ru[j]), __uint_as_float(ru[j + 1]));
      const float g0 = __uint_as_float(pg[e] << 16), g1 = __uint_as_float(pg[e] & 0xFFFF0000u);
      const float u0 = __uint_as_float(pu[e] << 16), u1 = __uint_as_float(pu[e] & 0xFFFF0000u);
      ph[e] = pack_bf16(g0 * sigmoidf_(g0) * u0, g1 * sigmoidf_(g1) * u1);
    }
    reinterpret_cast<uint4*>(c)[q] = make_uint4(pg[0], pg[1], pg[2], pg[3]);
    reinterpret_cast<uint4*>(c + g.split_n)[q] = make_uint4(pu[0], pu[1], pu[2], pu[3]);
    reinterpret_cast<uint4*>(h)[q] = make_uint4(ph[0], ph[1], ph[2], ph[3]);
  }
}

// EPI_BF16_ROPE: columns col0.. and col0+64.. of one head (rotate-half
// partners), 32 each, rounded to bf16 first as rope_qk does, rotated when
// the head is a q or k head, stored, and copied to the KV cache for k / v.
__device__ __forceinline__ void rope_store_pair32(const Args& g, int row, int col0, const uint32_t (&ra)[32],
                                                  const uint32_t (&rb)[32]) {
  uint32_t pa[16], pb[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    pa[e] = pack_bf16(__uint_as_float(ra[2 * e]), __uint_as_float(ra[2 * e + 1]));
    pb[e] = pack_bf16(__uint_as_float(rb[2 * e]), __uint_as_float(rb[2 * e + 1]));
  }
  if (col0 < g.col_v) {
    const float4* tp = reinterpret_cast<const float4*>(reinterpret_cast<const float2*>(g.R) +
                                                       static_cast<int64_t>(row) * g.ldr + (col0 & 63));
#pragma unroll
    for (int e = 0; e < 16; ++e) {  // pairs 2e, 2e+1 of this 32-column half
      const float4 cs = tp[e];
      const float a0 = __uint_as_float(pa[e] << 16), a1 = __uint_as_float(pa[e] & 0xFFFF0000u);
      const float b0 = __uint_as_float(pb[e] << 16), b1 = __uint_as_float(pb[e] & 0xFFFF0000u);
      pa[e] = pack_bf16(a0 * cs.x - b0 * cs.y, a1 * cs.z - b1 * cs.w);
      pb[e] = pack_bf16(b0 * cs.x + a0 * cs.y, b1 * cs.z + a1 * cs.w);
    }
  }
  __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(g.C) + static_cast<int64_t>(row) * g.ldc + col0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    reinterpret_cast<uint4*>(c)[q] = make_uint4(pa[4 * q], pa[4 * q + 1], pa[4 * q + 2], pa[4 * q + 3]);
    reinterpret_cast<uint4*>(c + 64)[q] = make_uint4(pb[4 * q], pb[4 * q + 1], pb[4 * q + 2], pb[4 * q + 3]);
  }
  __nv_bfloat16* cache = nullptr;
  if (col0 >= g.col_v)
    cache = g.vc ? g.vc + static_cast<int64_t>(row) * g.cache_ld + (col0 - g.col_v) : nullptr;
  else if (col0 >= g.col_k)
    cache = g.kc ? g.kc + static_cast<int64_t>(row) * g.cache_ld + (col0 - g.col_k) : nullptr;
  if (cache) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      reinterpret_cast<uint4*>(cache)[q] = make_uint4(pa[4 * q], pa[4 * q + 1], pa[4 * q + 2], pa[4 * q + 3]);
      reinterpret_cast<uint4*>(cache + 64)[q] = make_uint4(pb[4 * q], pb[4 * q + 1], pb[4 * q + 2], pb[4 * q + 3]);
    }
  }
}

namespace pair {

#ifndef CF_PAIR_STAGES
#define CF_PAIR_STAGES 6
#endif
constexpr int kStages = CF_PAIR_STAGES;
constexpr uint32_t kABytes = 128 * BK * 2;  // this CTA's half of A
constexpr uint32_t kBBytes = 128 * BK * 2;  // this CTA's half of B
constexpr size_t kSmem = 1024 + kStages * (kABytes + kBBytes) + 256;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clear the CTA-pair bit -> leader's smem address

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t leader_addr(uint32_t local) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(local));
  return r;
}
// Relaxed remote arrive: no data is published through these barriers (TMA
// bytes are tracked by the transaction count, TMEM reads are ordered by the
// tcgen05 fences), and a release.cluster arrive costs a GPU-scope MEMBAR.
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// Two problems in one persistent launch (`g2`, with its own maps and tile
// raster; tiles [0, g.num_m * g.num_n) belong to `g`, the rest to `g2`): the
// weight-gradient GEMMs of a layer whose tile counts fall just past a wave
// boundary share their last wave (e.g. o 256 + q|k|v 384 tiles = 8.65 waves
// of 74 pairs instead of 4 + 6).  Same epilogue and operand majors.
template <bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Args g1,
                     const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2, Args g2) {
  const Args& g = g1;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int tiles1 = g.num_m * g.num_n;
  const int num_tiles = tiles1 + g2.num_m * g2.num_n;  // g2.num_m = 0: one problem
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (g2.num_m > 0) {
      tma_prefetch(&tmA2);
      tma_prefetch(&tmB2);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 2);  // leader arrive.expect_tx + peer remote arrive
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // one arrive per epilogue warp of both CTAs (leader's copy is used)
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;  // num_m counts 256-row pair tiles

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full_leader0 = leader_addr(smem_u32(&full[0]));
      // Serpentine K: consecutive waves of the grouped raster share their
      // M-operand panels, but with long K a panel's head is evicted from L2
      // before the next wave needs it.  Odd waves stream K from the end, so
      // they start on the panel tail the previous wave just read.  Only the
      // load order changes (the MMA warp consumes stages in order; the fp32
      // summation order of a tile is fixed by its wave, so results stay
      // deterministic).
      int wave = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs, ++wave) {
        const bool second = tile >= tiles1;
        const Args& gp = second ? g2 : g;
        const CUtensorMap* mA = second ? &tmA2 : &tmA;
        const CUtensorMap* mB = second ? &tmB2 : &tmB;
        int mb, nb;
        tile_coords(gp, second ? tile - tiles1 : tile, mb, nb);
        const bool rev = gp.serp && (wave & 1);
        const int m0 = mb * 256 + static_cast<int>(rank) * 128;
        const int n0 = EPI == EPI_BF16_SWIGLU ? (rank == 0 ? nb * 128 : gp.split_n + nb * 128)
                                              : nb * 256 + static_cast<int>(rank) * 128;
        for (int kq = 0; kq < gp.num_k; ++kq) {
          const int kb = rev ? gp.num_k - 1 - kq : kq;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * kABytes;
          uint8_t* b = sB + stage * kBBytes;
          if (leader)
            mbar_expect_tx(&full[stage], 2 * (kABytes + kBBytes));
          else
            arrive_remote(full_leader0 + stage * 8);
          if constexpr (!A_MN) {
            tma_load_2sm(a, mA, &full[stage], kb * BK, m0);
          } else {
            tma_load_2sm(a, mA, &full[stage], m0, kb * BK);
            tma_load_2sm(a + kSlab, mA, &full[stage], m0 + 64, kb * BK);
          }
          if constexpr (!B_MN) {
            tma_load_2sm(b, mB, &full[stage], kb * BK, n0);
          } else {
            tma_load_2sm(b, mB, &full[stage], n0, kb * BK);
            tma_load_2sm(b + kSlab, mB, &full[stage], n0 + 64, kb * BK);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, 256, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = pair; tile < num_tiles; tile += npairs) {
        const int nk = tile >= tiles1 ? g2.num_k : g1.num_k;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * 256);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kABytes);
          const uint32_t b0 = smem_u32(sB + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? umma_desc_sw128(a0 + k * 2048, kSlab, 1024) : umma_desc_sw128(a0 + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? umma_desc_sw128(b0 + k * 2048, kSlab, 1024) : umma_desc_sw128(b0 + k * 32, 16, 1024);
            umma2(d, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          commit2_mc(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        commit2_mc(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t tempty_leader0 = leader_addr(smem_u32(&tempty[0]));
    for (int tile = pair; tile < num_tiles; tile += npairs) {
      const bool second = tile >= tiles1;
      const Args& g = second ? g2 : g1;  // this tile's problem
      int mb, nb;
      tile_coords(g, second ? tile - tiles1 : tile, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = mb * 256 + static_cast<int>(rank) * 128 + ew * 32 + lane;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + static_cast<uint32_t>(acc * 256);
      if constexpr (EPI == EPI_BF16_SWIGLU) {
        // accumulator columns [0,128) = gate, [128,256) = up of the same F columns
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t rg[32], ru[32];
          tmem_ld32(tbase + c * 32, rg);
          tmem_ld32(tbase + 128 + c * 32, ru);
          tmem_ld_wait();
          if (c == 3) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_remote(tempty_leader0 + acc * 8);
          }
          if (row < g.M) swiglu_store_row32(g, row, nb * 128 + c * 32, rg, ru);
        }
      } else if constexpr (EPI == EPI_BF16_ROPE) {
        // rotate-half partners are 64 columns apart inside a 128-column head
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          const int ca = (c >> 1) * 4 + (c & 1);  // chunks 0,1,4,5 pair with 2,3,6,7
          uint32_t ra[32], rb[32];
          tmem_ld32(tbase + ca * 32, ra);
          tmem_ld32(tbase + (ca + 2) * 32, rb);
          tmem_ld_wait();
          if (c == 3) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_remote(tempty_leader0 + acc * 8);
          }
          if (row < g.M) rope_store_pair32(g, row, nb * 256 + ca * 32, ra, rb);
        }
      } else if constexpr (kEpiCe<EPI>) {
        const int tgt = row < g.M ? g.ce_tgt[row] : -1;
        const float lse = (EPI == EPI_CE_GRAD && row < g.M) ? g.ce_lse[row] : 0.f;
        float m = -INFINITY, sum = 0.f;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          tmem_ld_wait();
          if (c == 7) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_remote(tempty_leader0 + acc * 8);
          }
          const int col0 = nb * 256 + c * 32;
          if (row < g.M && col0 < g.N) {
            if constexpr (EPI == EPI_CE_STATS)
              ce_stats_row32(g, row, col0, r, tgt, m, sum);
            else
              ce_grad_row32(g, row, col0, r, tgt, lse);
          }
        }
        if constexpr (EPI == EPI_CE_STATS)
          if (row < g.M) g.ce_part[static_cast<int64_t>(row) * g.ce_nparts + nb] = make_float2(m, sum);
      } else {
        float4 pre[8];
        if constexpr (kEpiReads<EPI>) prefetch_row32<EPI>(g, row, nb * 256, pre);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          tmem_ld_wait();
          if (c == 7) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_remote(tempty_leader0 + acc * 8);
          }
          const int col0 = nb * 256 + c * 32;
          if constexpr (kEpiReads<EPI>) {
            float4 nxt[8];
            if (c + 1 < 8) prefetch_row32<EPI>(g, row, col0 + 32, nxt);
            if (col0 < g.N) store_row32_pre<EPI>(g, row, col0, r, pre);
#pragma unroll
            for (int q = 0; q < 8; ++q) pre[q] = nxt[q];
          } else {
            if (col0 < g.N) store_row32<EPI>(g, row, col0, r);
          }
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

}  // namespace pair

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D bf16 tensor map, dim0 = contiguous.
bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
              uint32_t box_outer) {
  EncodeFn enc = encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int g_num_sms = 0;

// CF_GEMM_SERP=0 turns the serpentine K order off (A/B traffic measurement)
int gemm_serpentine() {
  static const int v = [] {
    const char* e = std::getenv("CF_GEMM_SERP");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

void set_ce(Args& g, const GemmDesc& d) {
  g.ce_tgt = d.ce_tgt;
  g.ce_part = reinterpret_cast<float2*>(d.ce_part);
  g.ce_tlogit = d.ce_tlogit;
  g.ce_lse = d.ce_lse;
  g.ce_scale = d.ce_scale;
  g.ce_nparts = static_cast<int>(ce_nparts(d.N));
}

// M-blocks per raster group (CF_GEMM_GROUP overrides; 0 = M-fastest over the
// whole output, the pre-grouping order).
int raster_group(int num_m, int dflt) {
  static const int env = [] {
    const char* e = std::getenv("CF_GEMM_GROUP");
    return e ? std::atoi(e) : -1;
  }();
  const int gm = env >= 0 ? env : dflt;
  return gm <= 0 || gm > num_m ? num_m : gm;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
cudaError_t launch_t(const GemmDesc& d, cudaStream_t st) {
  using C = Cfg<BN>;
  CUtensorMap ta, tb;
  bool ok = A_MN ? make_map(&ta, d.a, d.M, d.K, d.lda, 64, 64) : make_map(&ta, d.a, d.K, d.M, d.lda, BK, BM);
  ok = ok && (B_MN ? make_map(&tb, d.b, d.N, d.K, d.ldb, 64, 64) : make_map(&tb, d.b, d.K, d.N, d.ldb, BK, BN));
  if (!ok) return cudaErrorInvalidValue;
  Args g{};
  g.M = static_cast<int>(d.M);
  g.N = static_cast<int>(d.N);
  g.K = static_cast<int>(d.K);
  g.num_m = static_cast<int>((d.M + BM - 1) / BM);
  g.num_n = static_cast<int>((d.N + BN - 1) / BN);
  g.num_k = static_cast<int>((d.K + BK - 1) / BK);
  g.group_m = raster_group(g.num_m, 16);
  g.C = d.c;
  g.ldc = d.ldc;
  g.R = d.r;
  g.ldr = d.ldr;
  set_ce(g, d);
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, EPI>;
  // per (kernel, device), thread-safe
  const cudaError_t attr = smem_optin(reinterpret_cast<const void*>(kern), static_cast<int>(C::kSmem));
  if (attr != cudaSuccess) return attr;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = g.num_m * g.num_n;
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  kern<<<grid, 256, C::kSmem, st>>>(ta, tb, g);
  return cudaGetLastError();
}

// Tensor maps and kernel arguments of one CTA-pair problem.
template <bool A_MN, bool B_MN>
bool pair_problem(const GemmDesc& d, CUtensorMap& ta, CUtensorMap& tb, Args& g) {
  bool ok = A_MN ? make_map(&ta, d.a, d.M, d.K, d.lda, 64, 64) : make_map(&ta, d.a, d.K, d.M, d.lda, BK, 128);
  ok = ok && (B_MN ? make_map(&tb, d.b, d.N, d.K, d.ldb, 64, 64) : make_map(&tb, d.b, d.K, d.N, d.ldb, BK, 128));
  if (!ok) return false;
  g = Args{};
  g.M = static_cast<int>(d.M);
  g.N = static_cast<int>(d.N);
  g.K = static_cast<int>(d.K);
  g.num_m = static_cast<int>((d.M + 255) / 256);
  g.num_n = static_cast<int>((d.N + 255) / 256);
  g.num_k = static_cast<int>((d.K + BK - 1) / BK);
  // Short-K, wide-N shapes (qkv / gate|up forward, down dgrad) reuse the A
  // panels best with 16 M-blocks per group (DRAM/algorithmic bytes 1.3-1.6
  // vs 1.6-2.2 at 8, tools/gemm_group_traffic.sh); long-K shapes prefer 8.
  g.group_m = raster_group(g.num_m, g.num_k <= 64 && g.num_n >= 24 ? 16 : 8);
  g.split_n = static_cast<int>(d.N / 2);
  // long-K shapes only (K > 4096: the dgrad / wgrad / down-projection GEMMs
  // whose panels outgrow L2 within a wave); short-K shapes measured neutral
  // to slightly worse, and keeping them in order keeps EPI_BF16 and
  // EPI_BF16_SWIGLU outputs bitwise identical for the same operands
  g.serp = gemm_serpentine() && g.num_k > 64;
  g.col_k = static_cast<int>(d.col_k);
  g.col_v = static_cast<int>(d.col_v);
  g.kc = static_cast<__nv_bfloat16*>(d.kc);
  g.vc = static_cast<__nv_bfloat16*>(d.vc);
  g.cache_ld = d.cache_ld;
  g.C = d.c;
  g.ldc = d.ldc;
  g.R = d.r;
  g.ldr = d.ldr;
  set_ce(g, d);
  return true;
}

// One problem, or two (d2 != nullptr: same epilogue and majors) sharing the
// persistent grid.
template <bool A_MN, bool B_MN, int EPI>
cudaError_t launch_pair(const GemmDesc& d, cudaStream_t st, const GemmDesc* d2 = nullptr) {
  CUtensorMap ta, tb, ta2, tb2;
  Args g{}, g2{};
  if (!pair_problem<A_MN, B_MN>(d, ta, tb, g)) return cudaErrorInvalidValue;
  if (d2 && !pair_problem<A_MN, B_MN>(*d2, ta2, tb2, g2)) return cudaErrorInvalidValue;
  auto kern = pair::gemm_pair_kernel<A_MN, B_MN, EPI>;
  // per (kernel, device), thread-safe
  const cudaError_t attr = smem_optin(reinterpret_cast<const void*>(kern), static_cast<int>(pair::kSmem));
  if (attr != cudaSuccess) return attr;
  const int tiles = g.num_m * g.num_n + (d2 ? g2.num_m * g2.num_n : 0);
  const int pairs = std::min(tiles, gemm_num_sms() / 2);
  if (d2)
    kern<<<2 * pairs, 256, pair::kSmem, st>>>(ta, tb, g, ta2, tb2, g2);
  else
    kern<<<2 * pairs, 256, pair::kSmem, st>>>(ta, tb, g, ta, tb, g2);  // g2.num_m = 0: one problem
  return cudaGetLastError();
}

template <bool A_MN, bool B_MN>
cudaError_t pair_by_epi(const GemmDesc& d, cudaStream_t st) {
  switch (d.epi) {
    case EPI_BF16: return launch_pair<A_MN, B_MN, EPI_BF16>(d, st);
    case EPI_F32: return launch_pair<A_MN, B_MN, EPI_F32>(d, st);
    case EPI_F32_ACC: return launch_pair<A_MN, B_MN, EPI_F32_ACC>(d, st);
    case EPI_F32_RES: return launch_pair<A_MN, B_MN, EPI_F32_RES>(d, st);
    case EPI_BF16_TANH: return launch_pair<A_MN, B_MN, EPI_BF16_TANH>(d, st);
    case EPI_BF16_TANHGRAD: return launch_pair<A_MN, B_MN, EPI_BF16_TANHGRAD>(d, st);
    case EPI_BF16_SWIGLU: return launch_pair<A_MN, B_MN, EPI_BF16_SWIGLU>(d, st);
    case EPI_BF16_ROPE: return launch_pair<A_MN, B_MN, EPI_BF16_ROPE>(d, st);
    case EPI_CE_STATS: return launch_pair<A_MN, B_MN, EPI_CE_STATS>(d, st);
    case EPI_CE_GRAD: return launch_pair<A_MN, B_MN, EPI_CE_GRAD>(d, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t pair_by_major(const GemmDesc& d, cudaStream_t st) {
  if (d.a_kmajor && d.b_kmajor) return pair_by_epi<false, false>(d, st);
  if (d.a_kmajor && !d.b_kmajor) return pair_by_epi<false, true>(d, st);
  if (!d.a_kmajor && !d.b_kmajor) return pair_by_epi<true, true>(d, st);
  return pair_by_epi<true, false>(d, st);
}

template <int BN, bool A_MN, bool B_MN>
cudaError_t by_epi(const GemmDesc& d, cudaStream_t st) {
  switch (d.epi) {
    case EPI_BF16: return launch_t<BN, A_MN, B_MN, EPI_BF16>(d, st);
    case EPI_F32: return launch_t<BN, A_MN, B_MN, EPI_F32>(d, st);
    case EPI_F32_ACC: return launch_t<BN, A_MN, B_MN, EPI_F32_ACC>(d, st);
    case EPI_F32_RES: return launch_t<BN, A_MN, B_MN, EPI_F32_RES>(d, st);
    case EPI_BF16_TANH: return launch_t<BN, A_MN, B_MN, EPI_BF16_TANH>(d, st);
    case EPI_BF16_TANHGRAD: return launch_t<BN, A_MN, B_MN, EPI_BF16_TANHGRAD>(d, st);
    case EPI_CE_STATS:
      if constexpr (BN == 256) return launch_t<BN, A_MN, B_MN, EPI_CE_STATS>(d, st);
      break;
    case EPI_CE_GRAD:
      if constexpr (BN == 256) return launch_t<BN, A_MN, B_MN, EPI_CE_GRAD>(d, st);
      break;
  }
  return cudaErrorInvalidValue;
}

template <int BN>
cudaError_t by_major(const GemmDesc& d, cudaStream_t st) {
  if (d.a_kmajor && d.b_kmajor) return by_epi<BN, false, false>(d, st);
  if (d.a_kmajor && !d.b_kmajor) return by_epi<BN, false, true>(d, st);
  if (!d.a_kmajor && !d.b_kmajor) return by_epi<BN, true, true>(d, st);
  return by_epi<BN, true, false>(d, st);
}

}  // namespace

int gemm_num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

cudaError_t gemm(const GemmDesc& d, cudaStream_t st) {
  if (d.M <= 0 || d.N <= 0 || d.K <= 0) return cudaSuccess;
  // TMA: 16-byte aligned bases and row pitches (EPI_CE_STATS stores no C).
  const bool stores_c = d.epi != EPI_CE_STATS;
  if ((reinterpret_cast<uintptr_t>(d.a) & 15) || (reinterpret_cast<uintptr_t>(d.b) & 15) || (d.lda % 8) ||
      (d.ldb % 8) || (stores_c && ((reinterpret_cast<uintptr_t>(d.c) & 15) || (d.ldc % 8))))
    return cudaErrorMisalignedAddress;
  const int64_t sms = gemm_num_sms();
  const int mode = gemm_mode();
  if (d.epi == EPI_CE_STATS || d.epi == EPI_CE_GRAD) {
    if (!d.ce_tgt || (d.epi == EPI_CE_STATS ? (!d.ce_part || !d.ce_tlogit) : !d.ce_lse)) return cudaErrorInvalidValue;
    // 256-column slabs in both kernels: the partial index is the slab
    const int64_t pair_tiles = ((d.M + 255) / 256) * ((d.N + 255) / 256);
    if (mode != 1 && d.M > 128 && d.N > 128 && (pair_tiles >= sms / 4 || mode == 2)) return pair_by_major(d, st);
    return by_major<256>(d, st);
  }
  if (d.epi == EPI_BF16_ROPE) {
    if (!gemm_rope_ok(d.M, d.N, d.K, 128, d.col_k, d.col_v) || (reinterpret_cast<uintptr_t>(d.r) & 15) ||
        d.ldr != 64 || ((d.kc || d.vc) && (d.cache_ld % 8)))
      return cudaErrorInvalidValue;
    return pair_by_major(d, st);
  }
  if (d.epi == EPI_BF16_SWIGLU) {
    if (!gemm_swiglu_ok(d.M, d.N, d.K) || (reinterpret_cast<uintptr_t>(d.r) & 15) || (d.ldr % 8))
      return cudaErrorInvalidValue;
    return pair_by_major(d, st);
  }
  // CTA pairs for the large GEMMs (the step's hot path); single-CTA tiles for
  // narrow / short problems where a 256 x 256 pair tile would idle.
  const int64_t pair_tiles = ((d.M + 255) / 256) * ((d.N + 255) / 256);
  if (mode != 1 && d.M > 128 && d.N > 128 && (pair_tiles >= sms / 4 || mode == 2)) return pair_by_major(d, st);
  const int64_t tiles256 = ((d.M + BM - 1) / BM) * ((d.N + 255) / 256);
  const bool wide = d.N > 128 && tiles256 >= sms;
  return wide ? by_major<256>(d, st) : by_major<128>(d, st);
}

// Two weight-gradient GEMMs (EPI_F32_ACC, same operand majors) in one
// CTA-pair launch when both would take the pair kernel; otherwise one after
// the other.  Each output tile is computed exactly as in its own launch
// (serpentine K aside, whose direction follows the shared wave index).
cudaError_t gemm2(const GemmDesc& d0, const GemmDesc& d1, cudaStream_t st) {
  auto pair_ok = [](const GemmDesc& d) {
    const int64_t pair_tiles = ((d.M + 255) / 256) * ((d.N + 255) / 256);
    const int mode = gemm_mode();
    return mode != 1 && d.M > 128 && d.N > 128 && (pair_tiles >= gemm_num_sms() / 4 || mode >= 2) &&
           !(reinterpret_cast<uintptr_t>(d.a) & 15) && !(reinterpret_cast<uintptr_t>(d.b) & 15) && d.lda % 8 == 0 &&
           d.ldb % 8 == 0 && !(reinterpret_cast<uintptr_t>(d.c) & 15) && d.ldc % 8 == 0 && d.K > 0;
  };
  if (d0.epi != EPI_F32_ACC || d1.epi != EPI_F32_ACC || d0.a_kmajor != d1.a_kmajor || d0.b_kmajor != d1.b_kmajor ||
      !pair_ok(d0) || !pair_ok(d1)) {
    const cudaError_t e = gemm(d0, st);
    return e != cudaSuccess ? e : gemm(d1, st);
  }
  if (d0.a_kmajor && d0.b_kmajor) return launch_pair<false, false, EPI_F32_ACC>(d0, st, &d1);
  if (d0.a_kmajor && !d0.b_kmajor) return launch_pair<false, true, EPI_F32_ACC>(d0, st, &d1);
  if (!d0.a_kmajor && !d0.b_kmajor) return launch_pair<true, true, EPI_F32_ACC>(d0, st, &d1);
  return launch_pair<true, false, EPI_F32_ACC>(d0, st, &d1);
}

namespace {
// One warp per row: combine the row's (max, sum exp) slab partials in a
// fixed order (lane-strided, then a butterfly), LSE and the row loss.
__global__ void ce_finish_kernel(const float2* __restrict__ part, int64_t nparts, const float* __restrict__ tlogit,
                                 const int32_t* __restrict__ tgt, int64_t M, float* __restrict__ lse,
                                 float* __restrict__ row_loss) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const float2* p = part + row * nparts;
  float m = -INFINITY, s = 0.f;
  for (int64_t i = lane; i < nparts; i += 32) {
    const float2 q = p[i];
    if (q.x == -INFINITY) continue;
    const float nm = fmaxf(m, q.x);
    s = s * __expf(m - nm) + q.y * __expf(q.x - nm);
    m = nm;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - nm));
    m = nm;
  }
  if (lane == 0) {
    const float l = m + logf(s);
    if (lse) lse[row] = l;
    const int32_t t = tgt[row];
    row_loss[row] = t >= 0 ? l - tlogit[row] : 0.f;
  }
}
}  // namespace

cudaError_t ce_finish(const float* part, int64_t nparts, const float* tlogit, const int32_t* tgt, int64_t M,
                      float* lse, float* row_loss, cudaStream_t st) {
  if (M <= 0) return cudaSuccess;
  ce_finish_kernel<<<static_cast<unsigned>((M * 32 + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const float2*>(part), nparts, tlogit, tgt, M, lse, row_loss);
  return cudaGetLastError();
}

bool gemm_swiglu_ok(int64_t M, int64_t N, int64_t K) {
  const int64_t pair_tiles = ((M + 255) / 256) * (N / 256);
  const int mode = gemm_mode();
  return mode != 1 && N % 256 == 0 && M > 128 && K > 0 && (mode == 2 || pair_tiles >= gemm_num_sms() / 4);
}

bool gemm_rope_ok(int64_t M, int64_t N, int64_t K, int64_t dh, int64_t col_k, int64_t col_v) {
  const int64_t pair_tiles = ((M + 255) / 256) * (N / 256);
  const int mode = gemm_mode();
  return mode != 1 && dh == 128 && N % 256 == 0 && col_k % 256 == 0 && col_v % 256 == 0 && col_k <= col_v &&
         col_v <= N && M > 128 && K > 0 && (mode == 2 || pair_tiles >= gemm_num_sms() / 4);
}

// 0 = auto (CTA pairs when large), 1 = single-CTA only, 2 = CTA pairs whenever M, N > 128 (tests).
int& gemm_mode_ref() {
  static int m = [] {
    const char* e = std::getenv("CF_GEMM_MODE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}
int gemm_mode() { return gemm_mode_ref(); }
void set_gemm_mode(int m) { gemm_mode_ref() = m; }

}  // namespace cfk
