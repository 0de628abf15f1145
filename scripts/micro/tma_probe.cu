// Probe: can this process encode tensor maps (driver entry point + parameters)?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>

int main() {
  double* d = nullptr;
  cudaMalloc(&d, 4096);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  printf("entry point: err %d (%s) status %d ptr %p\n", (int)e, cudaGetErrorString(e), (int)q, p);
  if (!p) return 1;
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap m;
  const cuuint64_t dims1[1] = {256};
  const cuuint32_t box1[1] = {128};
  const cuuint32_t es1[1] = {1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dims1, nullptr, box1, es1,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("1d f64 box 128, strides null: %d\n", (int)r);
  const cuuint64_t st[1] = {0};
  r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, d, dims1, st, box1, es1,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("1d f64 box 128, no promotion: %d\n", (int)r);
  const cuuint64_t dims2[2] = {4, 256};
  const cuuint64_t st2[1] = {16};
  const cuuint32_t box2[2] = {4, 128};
  const cuuint32_t es2[2] = {1, 1};
  r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims2, st2, box2, es2,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("2d f32 rows: %d\n", (int)r);
  return 0;
}
