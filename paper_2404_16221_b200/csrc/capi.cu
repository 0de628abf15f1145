// C-ABI meta entry points: version, struct-layout check, error reporting.
#include <stdio.h>
#include <string.h>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"

namespace vr {

static thread_local char g_err[512] = "";

void set_error(const char* msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}

int num_sms() {
  static int n = 0;  // B200: 148
  if (n == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      n = v;
    else
      n = 148;
  }
  return n;
}

#ifdef VR_CHECKED
static int (*g_checkers[16])() = {};
static int g_n_checkers = 0;
int register_checker(int (*f)()) {
  if (g_n_checkers < 16) g_checkers[g_n_checkers++] = f;
  return g_n_checkers;
}
#endif

int check_launch(const char* where) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return VR_ERR_CUDA;
  }
  return VR_OK;
}

namespace tma {

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

bool encode_pairs(CUtensorMap* map, const double* base, uint64_t n, uint32_t box_pairs) {
  auto fn = encoder();
  if (!fn || !base || n == 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0 || box_pairs > 256)
    return false;
  // 16-byte rows of two float64 (as four 32-bit words): a tile's innermost start must be
  // 16-byte aligned (an odd 8-byte start raised "illegal instruction",
  // scripts/micro/tma_min2.cu), so chunks start at the even sample at or below theirs
  const cuuint64_t dims[2] = {4, (n + 1) / 2};  // (the caller's array holds 2 * that)
  const cuuint64_t strides[1] = {16};
  const cuuint32_t boxd[2] = {4, box_pairs};
  const cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<double*>(base), dims, strides,
            boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_rows(CUtensorMap* map, const float* base, uint64_t n, uint32_t row, uint32_t box) {
  auto fn = encoder();
  if (!fn || !base || n == 0 || reinterpret_cast<uintptr_t>(base) % 16 != 0 ||
      (row * 4) % 16 != 0)
    return false;
  const cuuint64_t dims[2] = {row, n};
  const cuuint64_t strides[1] = {(cuuint64_t)row * 4};
  const cuuint32_t boxd[2] = {row, box};
  const cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
            boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tma

}  // namespace vr

extern "C" int vr_tma_available(void) {
  CUtensorMap m;
  static double probe[32];
  double* d = nullptr;
  if (cudaMalloc(&d, 256) != cudaSuccess) return 0;
  const bool ok = vr::tma::encode_pairs(&m, d, 32, 8);
  cudaFree(d);
  (void)probe;
  return ok ? 1 : 0;
}

extern "C" int vr_abi_version(void) { return VR_ABI_VERSION; }

extern "C" int vr_struct_sizes(int64_t* out) {
  if (!out) return VR_ERR_BAD_ARG;
  out[0] = (int64_t)sizeof(VrTree);
  out[1] = (int64_t)sizeof(VrAnalyticField);
  out[2] = (int64_t)sizeof(VrVoxelDesc);
  out[3] = (int64_t)sizeof(VrHashGridDesc);
  out[4] = (int64_t)sizeof(VrBlob);
  return VR_OK;
}

extern "C" const char* vr_last_error(void) { return vr::g_err; }

extern "C" int vr_check_failures(void) {
#ifdef VR_CHECKED
  cudaDeviceSynchronize();
  int total = 0;
  for (int i = 0; i < vr::g_n_checkers; ++i) total += vr::g_checkers[i]();
  return total;
#else
  return -1;  // release build: no checks compiled in
#endif
}

extern "C" int vr_device_sync(void) {
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    vr::set_error(cudaGetErrorString(e));
    return VR_ERR_CUDA;
  }
  return VR_OK;
}
