// Measures tcgen05.mma issue-to-completion throughput (cycles per
// instruction, one CTA per SM, all SMs busy) for M=128 x N x K=16 bf16 with
// A from shared memory (SS) or from TMEM (TS).  Operand contents are
// irrelevant (throughput probe).  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O2 -o mma_probe tools/mma_probe.cu
#include <cstdio>

#include "../paper_2503_02356_b200/csrc/kernels/common.cuh"

using namespace cfk;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) probe(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = umma_idesc_bf16(128, N, 0, 0);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 65536);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (TS)
          umma_bf16_ts(tmem, tmem + 384 + k * 8, umma_desc_sw128(b0 + (k & 3) * 32, 16, 1024), id, 1u);
        else
          umma_bf16(tmem, umma_desc_sw128(a0 + (k & 3) * 32, 16, 1024), umma_desc_sw128(b0 + (k & 3) * 32, 16, 1024),
                    id, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

template <int N, bool TS>
void run(const char* name, int sms) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  auto k = probe<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int reps = 2000;
  k<<<sms, 128, 131072>>>(reps, d);
  k<<<sms, 128, 131072>>>(reps, d);
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double per = avg / (reps * 8.0);
  printf("%-22s %7.1f cycles/MMA  -> %6.0f flop/cycle/SM (peak 8192)  err=%s\n", name, per,
         2.0 * 128 * N * 16 / per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// cta_group::2 (CTA pair, M = 256): does a pair issue N = 64 MMAs at the
// full rate, i.e. is the 1-CTA N = 64 shortfall a per-instruction floor or a
// per-CTA operand-read limit?
__device__ __forceinline__ uint32_t cta_rank_() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe2(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && cta_rank_() == 0) {
    constexpr uint32_t id = umma_idesc_bf16(256, N, 0, 0);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 65536);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint64_t bd = umma_desc_sw128(b0 + (k & 3) * 32, 16, 1024);
        if (TS)
          asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(tmem + 384 + k * 8),
                       "l"(bd), "r"(id) : "memory");
        else
          asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem),
                       "l"(umma_desc_sw128(a0 + (k & 3) * 32, 16, 1024)), "l"(bd), "r"(id) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)), "h"(static_cast<uint16_t>(3)) : "memory");
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x / 2] = t1 - t0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int N, bool TS>
void run2(const char* name, int sms) {
  long long* d;
  const int pairs = sms / 2;
  cudaMalloc(&d, pairs * sizeof(long long));
  auto k = probe2<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int reps = 2000;
  k<<<pairs * 2, 128, 131072>>>(reps, d);
  k<<<pairs * 2, 128, 131072>>>(reps, d);
  long long h[256];
  cudaMemcpy(h, d, pairs * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < pairs; ++i) avg += h[i];
  avg /= pairs;
  const double per = avg / (reps * 8.0);
  printf("%-22s %7.1f cycles/MMA  -> %6.0f flop/cycle/SM (peak 8192)  err=%s\n", name, per,
         2.0 * 256 * N * 16 / per / 2, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>("M128 N64  SS", sms);
  run<64, true>("M128 N64  TS", sms);
  run<128, false>("M128 N128 SS", sms);
  run<128, true>("M128 N128 TS", sms);
  run<256, false>("M128 N256 SS", sms);
  run<256, true>("M128 N256 TS", sms);
  run<32, true>("M128 N32  TS", sms);
  run<96, true>("M128 N96  TS", sms);
  run2<64, false>("pair M256 N64  SS", sms);
  run2<64, true>("pair M256 N64  TS", sms);
  run2<128, true>("pair M256 N128 TS", sms);
  run2<32, true>("pair M256 N32  TS", sms);
  return 0;
}
