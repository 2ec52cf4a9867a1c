// Probe: which 1-D fp32 tensor-map encodings does the driver accept?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  float* x;
  cudaMalloc(&x, 4003 * sizeof(float));
  CUtensorMap m;
  cuuint64_t dims[1] = {4003}, dims2[2] = {4003, 1};
  cuuint64_t strides[1] = {4003 * 4};
  cuuint32_t box[1] = {64}, box2[2] = {64, 1}, es[1] = {1}, es2[2] = {1, 1};
  for (int p = 0; p < 2; ++p) {
    auto prom = p ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    CUresult r1 = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, x, dims, nullptr, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, x, dims, strides, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r3 = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims2, strides, box2, es2,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("prom %d: rank1 null strides %d, rank1 strides %d, rank2 %d\n", p, r1, r2, r3);
  }
  return 0;
}
