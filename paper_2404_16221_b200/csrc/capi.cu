// C-ABI meta entry points: version, struct-layout check, error reporting.
#include <stdio.h>
#include <string.h>

#include "common.cuh"

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

}  // namespace vr

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
