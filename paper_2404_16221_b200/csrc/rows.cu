// Active rows of a backward pass (vr_capi.h vr_active_rows): the ordered list of samples
// whose upstream gradient dsig_rgb[i] (float4) is non-zero.  A sample with an exactly zero
// upstream gradient contributes exactly zero to d(enc) and to every weight gradient, so the
// MLP backward and the hash-grid scatter skip it; behind an opaque surface the float32
// transmittance underflows to 0 and most samples are such rows (c4 steady state: 75 % of
// the NeRF samples, 95 % of the proposal samples).
//
// Three launches, no host sync: k_rows_mark (per 4096-sample chunk: a 16-bit mask per
// thread and the chunk's count), k_rows_scan (one block: exclusive scan of the chunk
// counts, the total into *n_rows) and k_rows_write (per chunk: block scan of the masks,
// indices written in increasing order).  The list is ordered so the backward's tiles keep
// the samples' ray order (coalesced enc / direction loads, deterministic tile contents).
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace vr {

constexpr int AR_THREADS = 256, AR_PER = 16, AR_CHUNK = AR_THREADS * AR_PER;
constexpr int AR_SCAN_THREADS = 1024;

__device__ __forceinline__ bool row_active(const float4* __restrict__ dsr, int64_t i) {
  const float4 g = __ldcs(dsr + i);
  return g.x != 0.f || g.y != 0.f || g.z != 0.f || g.w != 0.f;  // NaN counts as active
}

// element k of thread t in chunk b: sample b * AR_CHUNK + k * AR_THREADS + t (coalesced)
__global__ void __launch_bounds__(AR_THREADS)
    k_rows_mark(const float4* __restrict__ dsr, int64_t n, uint16_t* __restrict__ masks,
                int32_t* __restrict__ counts) {
  const int64_t base = (int64_t)blockIdx.x * AR_CHUNK + threadIdx.x;
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < AR_PER; ++k) {
    const int64_t i = base + (int64_t)k * AR_THREADS;
    if (i < n && row_active(dsr, i)) mask |= 1u << k;
  }
  masks[(int64_t)blockIdx.x * AR_THREADS + threadIdx.x] = (uint16_t)mask;
  __shared__ int32_t tot;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  const int32_t c = (int32_t)__reduce_add_sync(0xffffffffu, (unsigned)__popc(mask));
  if ((threadIdx.x & 31) == 0) atomicAdd(&tot, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(AR_SCAN_THREADS)
    k_rows_scan(int32_t* __restrict__ counts, int64_t chunks, int32_t* __restrict__ n_rows) {
  using Scan = cub::BlockScan<int32_t, AR_SCAN_THREADS>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < chunks; c0 += AR_SCAN_THREADS) {
    const int64_t c = c0 + threadIdx.x;
    const int32_t v = c < chunks ? counts[c] : 0;
    int32_t ex, total;
    Scan(tmp).ExclusiveSum(v, ex, total);
    const int32_t base = carry;
    if (c < chunks) counts[c] = base + ex;
    __syncthreads();  // every thread has read carry and tmp
    if (threadIdx.x == 0) carry = base + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_rows = carry;
}

// All 16 rounds' warp counts at once (16 ballots per warp into shared memory, one barrier),
// then each thread places its elements: round k's elements precede round k + 1's, and
// within a round the warps' in order (two barriers per chunk instead of 32).
__global__ void __launch_bounds__(AR_THREADS)
    k_rows_write(const uint16_t* __restrict__ masks, const int32_t* __restrict__ offsets,
                 int64_t n, int32_t* __restrict__ rows) {
  constexpr int NW = AR_THREADS / 32;
  __shared__ int32_t cnt[AR_PER][NW];  // round k, warp w: active elements
  __shared__ int32_t base_k[AR_PER];   // round k's first output slot (relative)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t mask = masks[(int64_t)blockIdx.x * AR_THREADS + threadIdx.x];
  const int64_t base = (int64_t)blockIdx.x * AR_CHUNK + threadIdx.x;
  uint32_t bal[AR_PER];
#pragma unroll
  for (int k = 0; k < AR_PER; ++k) {
    bal[k] = __ballot_sync(0xffffffffu, (mask >> k) & 1u);
    if (lane == 0) cnt[k][warp] = __popc(bal[k]);
  }
  __syncthreads();
  if (threadIdx.x < AR_PER) {  // per round: the total, then an exclusive scan below
    int32_t t = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += cnt[threadIdx.x][w];
    base_k[threadIdx.x] = t;
  }
  __syncthreads();
  const int32_t out0 = offsets[blockIdx.x];
  int32_t run = 0;
#pragma unroll
  for (int k = 0; k < AR_PER; ++k) {
    int32_t before = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) before += w < warp ? cnt[k][w] : 0;
    if ((mask >> k) & 1u)
      rows[out0 + run + before + __popc(bal[k] & ((1u << lane) - 1u))] =
          (int32_t)(base + (int64_t)k * AR_THREADS);
    run += base_k[k];
  }
}

static int64_t ar_chunks(int64_t n) { return (n + AR_CHUNK - 1) / AR_CHUNK; }

}  // namespace vr

using namespace vr;

extern "C" size_t vr_active_rows_workspace_bytes(int64_t n) {
  if (n < 0) return 0;
  const int64_t c = ar_chunks(n);
  return (size_t)(c * sizeof(int32_t) + 255) / 256 * 256 + (size_t)c * AR_THREADS * 2;
}

extern "C" int vr_active_rows(const float* dsr, int64_t n, int32_t* rows, int32_t* n_rows,
                              void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || n > INT32_MAX || !n_rows || (n > 0 && (!dsr || !rows)) ||
      ws_bytes < vr_active_rows_workspace_bytes(n) || (n > 0 && !ws)) {
    set_error("vr_active_rows: bad argument");
    return VR_ERR_BAD_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    cudaMemsetAsync(n_rows, 0, sizeof(int32_t), s);
    return check_launch("vr_active_rows");
  }
  const int64_t c = ar_chunks(n);
  int32_t* counts = reinterpret_cast<int32_t*>(ws);
  uint16_t* masks = reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(ws) +
                                                (c * sizeof(int32_t) + 255) / 256 * 256);
  k_rows_mark<<<(unsigned)c, AR_THREADS, 0, s>>>(reinterpret_cast<const float4*>(dsr), n, masks,
                                                 counts);
  k_rows_scan<<<1, AR_SCAN_THREADS, 0, s>>>(counts, c, n_rows);
  k_rows_write<<<(unsigned)c, AR_THREADS, 0, s>>>(masks, counts, n, rows);
  return check_launch("vr_active_rows");
}
