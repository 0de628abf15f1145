// Microbenchmark: random gathers from an L2-resident table (32 MB).
//   mode 0: one 16-byte load per lane (aligned pair)
//   mode 1: lane pairs, 8 bytes each, same 16-byte pair   (one request per pair?)
//   mode 2: lane pairs, 8 bytes each, same 32-byte sector, straddling its 16-byte halves
//   mode 3: lane pairs, 8 bytes each, different sectors
//   mode 4: one 8-byte load per lane
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(256) k(const float2* __restrict__ tab, uint32_t mask_sectors,
                                         int iters, float* out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t s = hash32(tid * 7919u + 1u);
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    s = hash32(s + it);
    if (MODE == 0) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(tab + (size_t)(s & mask_sectors) * 4));
      acc += v.x + v.w;
    } else if (MODE == 4) {
      const float2 v = __ldg(tab + (size_t)(s & mask_sectors) * 4 + (s >> 30));
      acc += v.x;
    } else {
      const uint32_t sl = __shfl_sync(0xffffffffu, s, lane & ~1u);
      const size_t sec = (size_t)(sl & mask_sectors) * 4;  // 4 entries of 8 B per sector
      size_t e;
      if (MODE == 1) e = sec + (lane & 1);
      else if (MODE == 2) e = sec + 1 + (lane & 1);
      else e = (size_t)((hash32(sl) ^ (lane & 1) * 0x9e3779b9u) & mask_sectors) * 4;
      const float2 v = __ldg(tab + e);
      acc += v.x;
    }
  }
  if (acc == 12345.f) out[tid] = acc;
}

int main() {
  const size_t n_sectors = (32u << 20) / 32;  // 32 MB
  float2* tab;
  float* out;
  cudaMalloc(&tab, n_sectors * 32);
  cudaMalloc(&out, 1 << 24);
  cudaMemset(tab, 0, n_sectors * 32);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 256, grid = sms * 8;
  for (int mode = 0; mode < 5; ++mode) {
    auto launch = [&] {
      if (mode == 0) k<0><<<grid, 256>>>(tab, n_sectors - 1, iters, out);
      if (mode == 1) k<1><<<grid, 256>>>(tab, n_sectors - 1, iters, out);
      if (mode == 2) k<2><<<grid, 256>>>(tab, n_sectors - 1, iters, out);
      if (mode == 3) k<3><<<grid, 256>>>(tab, n_sectors - 1, iters, out);
      if (mode == 4) k<4><<<grid, 256>>>(tab, n_sectors - 1, iters, out);
    };
    launch();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double lanes = 5.0 * grid * 256.0 * iters;
    printf("mode %d: %.3f ms  %.1f G lane-loads/s  (%.3f per SM-clk) %s\n", mode, ms / 5,
           lanes / (ms * 1e6), lanes / (ms * 1e-3) / sms / 1.965e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
