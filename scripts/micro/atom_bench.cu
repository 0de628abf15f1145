// Microbenchmark: random 16-byte float adds into a 128 MB table.
//   mode 0: red.global.add.v4.f32 (LSU)
//   mode 1: cp.reduce.async.bulk .add.f32 16 B from smem (TMA / bulk-copy engine)
//   mode 2: half and half
//   mode 3: red.global.add.v2.f32 x2 (8-byte pieces)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(256) k(float* tab, uint32_t mask_pairs, int iters) {
  __shared__ __align__(16) float4 slot[256][4];
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t s = hash32(tid * 7919u + 1u);
  for (int it = 0; it < iters; ++it) {
    s = hash32(s + it);
    float* dst = tab + (size_t)(s & mask_pairs) * 4;
    const float v = 1e-3f;
    bool use_bulk = MODE == 1 || (MODE == 2 && (it & 1));
    if (MODE >= 4) {
      // lanes cooperating on one sector: the group leader's random pair index is shared
      const int gs = MODE == 5 ? 4 : 2;
      const uint32_t lane = threadIdx.x & 31, lead = lane & ~(uint32_t)(gs - 1);
      const uint32_t sl = __shfl_sync(0xffffffffu, s, lead);
      float* base = tab + (size_t)((sl & mask_pairs) & ~1u) * 4;  // 32-byte aligned
      if (MODE == 4) {  // 2 lanes x v2 into one 16-byte pair
        asm volatile("red.global.add.v2.f32 [%0], {%1, %1};" ::"l"(base + 2 * (lane & 1)), "f"(v) : "memory");
      } else if (MODE == 5) {  // 4 lanes x v2 into one 32-byte sector
        asm volatile("red.global.add.v2.f32 [%0], {%1, %1};" ::"l"(base + 2 * (lane & 3)), "f"(v) : "memory");
      } else if (MODE == 6) {  // 2 lanes x v4 into one 32-byte sector
        asm volatile("red.global.add.v4.f32 [%0], {%1, %1, %1, %1};" ::"l"(base + 4 * (lane & 1)), "f"(v) : "memory");
      } else {  // MODE 7: 2 lanes x v2 straddling the sector's 16-byte halves (bytes 8..23)
        asm volatile("red.global.add.v2.f32 [%0], {%1, %1};" ::"l"(base + 2 + 2 * (lane & 1)), "f"(v) : "memory");
      }
    } else if (MODE == 3) {
      asm volatile("red.global.add.v2.f32 [%0], {%1, %1};" ::"l"(dst), "f"(v) : "memory");
      asm volatile("red.global.add.v2.f32 [%0], {%1, %1};" ::"l"(dst + 2), "f"(v) : "memory");
    } else if (!use_bulk) {
      asm volatile("red.global.add.v4.f32 [%0], {%1, %1, %1, %1};" ::"l"(dst), "f"(v) : "memory");
    } else {
      const int q = (it >> (MODE == 2 ? 1 : 0)) & 3;
      if (it >= 8) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
      slot[threadIdx.x][q] = make_float4(v, v, v, v);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&slot[threadIdx.x][q]);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 16;"
                   ::"l"(dst), "r"(sa) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t n_pairs = 1u << 23;  // 8M x 16 B = 128 MB
  float* tab;
  cudaMalloc(&tab, n_pairs * 16);
  cudaMemset(tab, 0, n_pairs * 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 256;
  for (size_t np : {(size_t)1 << 18, (size_t)1 << 21, n_pairs}) {
  const int blocks_per_sm = 8;
  {
    const int grid = sms * blocks_per_sm;
    for (int mode = 0; mode < 8; ++mode) {
      auto launch = [&] {
        if (mode == 0) k<0><<<grid, 256>>>(tab, np - 1, iters);
        if (mode == 1) k<1><<<grid, 256>>>(tab, np - 1, iters);
        if (mode == 2) k<2><<<grid, 256>>>(tab, np - 1, iters);
        if (mode == 3) k<3><<<grid, 256>>>(tab, np - 1, iters);
        if (mode == 4) k<4><<<grid, 256>>>(tab, np - 1, iters);
        if (mode == 5) k<5><<<grid, 256>>>(tab, np - 1, iters);
        if (mode == 6) k<6><<<grid, 256>>>(tab, np - 1, iters);
        if (mode == 7) k<7><<<grid, 256>>>(tab, np - 1, iters);
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
      // 16-byte adds: modes 4/5 move 8 B per lane
      const double ops = 5.0 * grid * 256.0 * iters * ((mode == 4 || mode == 5 || mode == 7) ? 0.5 : 1.0);
      printf("table %zu MB mode %d: %.2f ms  %.1f G 16B-adds/s  (%.3f per SM-clk @1.965GHz) err=%s\n",
             np * 16 >> 20, mode, ms / 5, ops / (ms * 1e6), ops / (ms * 1e-3) / sms / 1.965e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  }
  return 0;
}
