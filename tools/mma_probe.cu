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

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>("M128 N64  SS", sms);
  run<64, true>("M128 N64  TS", sms);
  run<128, false>("M128 N128 SS", sms);
  run<128, true>("M128 N128 TS", sms);
  run<256, false>("M128 N256 SS", sms);
  run<256, true>("M128 N256 TS", sms);
  return 0;
}
