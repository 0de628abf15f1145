// Layout check for tcgen05.mma kind::f16 with A in TMEM ("TS" mode): D[128 x N] = A . B^T,
// A [128 x K] fp16 written to TMEM with tcgen05.st (lane m = row m, 32-bit column j holds
// A[m][2j] (low half) and A[m][2j+1] (high half)), B [N x K] fp16 in shared memory in the
// repo's SWIZZLE_NONE K-major core-matrix layout.  Compares with a CPU product.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include "../../paper_2404_16221_b200/csrc/tc.cuh"

using namespace vr::tc;

constexpr int M = 128, N = 64, K = 32;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                 "r"(r[6]), "r"(r[7]) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
               ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__global__ void k(const __half* A, const __half* B, float* D) {
  __shared__ __align__(1024) uint8_t sb[N * K * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x;
  for (int idx = t; idx < N * (K / 8); idx += blockDim.x) {  // B rows into core-matrix layout
    const int o = idx / (K / 8), cb = idx % (K / 8);
    *reinterpret_cast<uint4*>(sb + tile_off(N, o, cb * 8)) =
        *reinterpret_cast<const uint4*>(B + o * K + cb * 8);
  }
  if (t < 32) tmem_alloc(&slot, 128);
  if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t lane_base = (uint32_t)((t >> 5) * 32) << 16;
  // A row t into TMEM columns [64, 64 + K/2)
  uint32_t r[8];
  for (int c0 = 0; c0 < K / 2; c0 += 8) {
    for (int j = 0; j < 8; ++j) {
      __half2 h = __halves2half2(A[t * K + 2 * (c0 + j)], A[t * K + 2 * (c0 + j) + 1]);
      r[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    tmem_st8(tmem + lane_base + 64 + c0, r);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (t == 0) {
    tc_fence_after();
    const uint32_t id = idesc_f16(M, N, 0, 0);
    for (int kb = 0; kb < K / 16; ++kb)
      mma_ts(tmem + 0, tmem + 64 + kb * 8, desc_k(smem_u32(sb), N, 2 * kb), id, kb > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[16];
  for (int c = 0; c < N; c += 16) {
    tmem_ld16(tmem + lane_base + c, v);
    for (int j = 0; j < 16; ++j) D[t * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) { tc_fence_after(); tmem_dealloc(tmem, 128); }
}

int main() {
  __half hA[M * K], hB[N * K];
  float fA[M * K], fB[N * K];
  srand(1);
  for (int i = 0; i < M * K; ++i) { fA[i] = (rand() % 17 - 8) / 8.f; hA[i] = __float2half(fA[i]); }
  for (int i = 0; i < N * K; ++i) { fB[i] = (rand() % 17 - 8) / 8.f; hB[i] = __float2half(fB[i]); }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dA, dB, dD);
  static float D[M * N];
  cudaError_t e = cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int kk = 0; kk < K; ++kk) ref += (double)fA[m * K + kk] * fB[n * K + kk];
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
    }
  printf("TS-mode MMA: %s, max abs err %.3g (D[0][0]=%g)\n", cudaGetErrorString(e), maxerr, D[0]);
  return maxerr < 1e-3 ? 0 : 1;
}
