// TMA (cp.async.bulk.tensor) staging of contiguous per-sample arrays into shared memory.
//
// The K4 walks read each chunk of 32 K consecutive samples (t0, t1 float64, sig_rgb
// float4) once; as per-lane global loads of K consecutive samples every load instruction
// of a warp spans 32 K elements (uncoalesced within the instruction) and its latency sits in
// the walk.  One elected lane instead issues three tensor copies per chunk into a warp-
// private double buffer (the next chunk's copies fly while the current chunk is walked),
// completion tracked by an mbarrier with the transaction byte count.
//
// Host side: tensor maps are encoded per call (cuTensorMapEncodeTiled through the runtime's
// driver entry point) and passed as __grid_constant__ kernel parameters.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace vr {
namespace tma {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// generic-proxy accesses of a buffer before the async proxy overwrites it
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

// one lane of a converged warp (elect.sync): the issuing lane of the TMA copies
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n"
      : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// host: a float64 array of n elements (allocated with an even count >= n) as ceil(n / 2)
// rows of two (box: box_pairs rows; load with
// load_2d(dst, map, 0, first_pair)); n rows of `row` float32 (box: `box` rows; load with
// load_2d(dst, map, 0, first_row)).  A tile's innermost start must be 16-byte aligned on this
// hardware (scripts/micro/tma_min2.cu), hence rows.  False when the driver entry point is
// missing or the base is not 16-byte aligned (callers take the plain-load path).
bool encode_pairs(CUtensorMap* map, const double* base, uint64_t n, uint32_t box_pairs);
bool encode_rows(CUtensorMap* map, const float* base, uint64_t n, uint32_t row, uint32_t box);

}  // namespace tma
}  // namespace vr
