// Minimal sm_100a tensor-core toolkit (inline PTX): TMEM alloc, tcgen05.mma kind::f16,
// commit -> mbarrier, tcgen05.ld, fences, and the shared-memory operand layout.
//
// Operand layout (SWIZZLE_NONE canonical core matrices).  A [R rows x C cols] fp16
// tile is stored as C/8 column blocks of R x 16 bytes:
//     byte(r, c) = (c / 8) * (R * 16) + r * 16 + (c % 8) * 2
// Read with K = c it is a K-major operand (SBO = 128 B between 8-row groups, LBO =
// R*16 B between 8-column blocks); read with K = r it is an MN-major operand (SBO =
// R*16 between 8-column groups, LBO = 128 B between 8-row groups).  One layout thus
// serves both the forward GEMMs (K = features) and the weight-gradient GEMMs
// (K = samples) without transposes.  Row-per-thread 16-byte stores are bank-conflict
// free (consecutive threads -> consecutive 16 B).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace vr {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__host__ __device__ constexpr uint32_t tile_off(int R, int r, int c) {
  return (uint32_t)((c >> 3) * (R * 16) + r * 16 + (c & 7) * 2);
}

// Shared-memory matrix descriptor (sm_100 "version 1", no swizzle).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// K-major view of an R-row tile, starting at column block kb (8 columns per block)
__device__ __forceinline__ uint64_t desc_k(uint32_t base, int R, int kb) {
  return sdesc(base + (uint32_t)(kb * R * 16), (uint32_t)(R * 16), 128u);
}
// MN-major view (K = rows) of an R-row tile, starting at row block kb (8 rows per block)
__device__ __forceinline__ uint64_t desc_mn(uint32_t base, int R, int kb) {
  return sdesc(base + (uint32_t)(kb * 128), 128u, (uint32_t)(R * 16));
}

// Instruction descriptor, kind::f16: fp16 A/B, fp32 D.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// The suspend-time hint lets the hardware park a waiting warp until the phase completes
// (or the hint expires) instead of returning at once: a spinning try_wait loop cost ~20 %
// of the MLP kernels' issued instructions (SYNCS + BRA), slots the other CTA's epilogue
// warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(a), "r"(phase), "r"(1000000u)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// whole warp: allocate ncols TMEM columns, base address written to *slot
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// 32 lanes x 32-bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// store 8 consecutive columns (one 16-byte chunk) of row r
__device__ __forceinline__ void st_row8(uint8_t* tile, int R, int r, int cb, const __half* h8) {
  *reinterpret_cast<uint4*>(tile + tile_off(R, r, cb * 8)) = *reinterpret_cast<const uint4*>(h8);
}
__device__ __forceinline__ void ld_row8(const uint8_t* tile, int R, int r, int cb, __half* h8) {
  *reinterpret_cast<uint4*>(h8) = *reinterpret_cast<const uint4*>(tile + tile_off(R, r, cb * 8));
}

}  // namespace tc
}  // namespace vr
