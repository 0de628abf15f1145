// K3 on the 5th-generation tensor cores: the per-region density + colour MLP as
// tcgen05.mma (kind::f16, fp32 accumulation in TMEM), one thread issuing, operands in
// shared memory (layout in tc.cuh), results read back with tcgen05.ld.
//
// Semantics are identical to the CUDA-core reference kernels in mlp.cu (same fp16
// quantisation points, fp32 accumulation).  A 128-sample tile is M = 128; sample row r
// lives in TMEM lane r, so the epilogues are row-per-thread (TPR threads per row, each
// owning a slice of the columns; warp w reads lanes 32*(w%4) and column half w/4).
//
// Forward, per tile (TMEM: 128 columns):
//   P <- enc                                  [128 x 32]
//   D[0:64)   = P . W1d^T  -> relu -> Q       [128 x 64]
//   D[64:80)  = Q . W2d^T  -> sigma, geo ;  P <- [geo | SH(d)]
//   D[0:64)   = P . W1c^T  -> relu -> Q
//   D[0:64)   = Q . W2c^T  -> relu -> P
//   D[64:80)  = P . W3c^T  -> sigmoid -> rgb
//
// Backward, per tile (TMEM: 256 columns; weight-gradient accumulators stay in TMEM for
// the CTA's whole persistent loop and are flushed once at the end):
//   recompute the forward keeping h1d, cin, h1c, h2c in smem (enc is re-staged from
//   global memory for the last stage, so its slot is reused for cin);
//   for each layer the upstream gradient G (fp32 registers) is written to smem as an
//   fp16 hi part and an fp16 lo part (G = hi + lo to ~22 bits) and ONE round issues
//       dX  = Ghi . W  + Glo . W   (M = 128, A K-major, B = W read MN-major)
//       dW += [Ghi | Glo]^T X      (one MMA, both operands MN-major, K = 128 samples).
//   The weight-gradient MMA stacks hi and lo instead of issuing two M = 64 MMAs (an
//   M = 64 dispatch costs as much as M = 128): for 64-wide G the hi and lo tiles are
//   adjacent in smem and form one M = 128 A operand (accumulator rows 64..127 hold the lo
//   products); for 16-wide G the lo part sits in columns 16..31 of the hi tile and the
//   stacked operand is B with N = 32.  The halves are summed when the accumulators are
//   flushed.
//   Activations and weights are exactly fp16 by definition of the model, so the
//   backward is accurate to fp32 accumulation.  |g| >= 65504 raises VR_FLAG_OVERFLOW.
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "hashgrid.cuh"
#include "tc.cuh"

namespace vr {

using namespace tc;

namespace mlp {

constexpr int TILE = 128;
// weight tiles in smem (bytes)
constexpr uint32_t OW1D = 0, OW2D = OW1D + 64 * 32 * 2, OW1C = OW2D + 16 * 64 * 2,
                   OW2C = OW1C + 64 * 32 * 2, OW3C = OW2C + 64 * 64 * 2,
                   WBYTES = OW3C + 16 * 64 * 2;  // 20480

__device__ __forceinline__ void stage_one(const __half* __restrict__ Wg, uint8_t* s, int OUT,
                                          int IN) {
  const int nchunk = OUT * (IN / 8);
  for (int idx = threadIdx.x; idx < nchunk; idx += blockDim.x) {
    const int o = idx / (IN / 8), cb = idx % (IN / 8);
    const uint4 v = *reinterpret_cast<const uint4*>(Wg + o * IN + cb * 8);
    *reinterpret_cast<uint4*>(s + tile_off(OUT, o, cb * 8)) = v;
  }
}

template <bool DENS = false>
__device__ __forceinline__ void stage_weights(const __half* __restrict__ W, uint8_t* s) {
  stage_one(W + VR_MLP_W1D, s + OW1D, 64, 32);
  stage_one(W + VR_MLP_W2D, s + OW2D, 16, 64);
  if (DENS) return;  // the density branch reads W1d, W2d only
  stage_one(W + VR_MLP_W1C, s + OW1C, 64, 32);
  stage_one(W + VR_MLP_W2C, s + OW2C, 64, 64);
  stage_one(W + VR_MLP_W3C, s + OW3C, 16, 64);
}

// D[128 x N] = A[128 x K] . B^T,  A = activation tile (K-major), B = weight tile
// [N rows x K cols] (K-major)
__device__ __forceinline__ void issue_fwd(uint32_t a, int K, uint32_t b, int N, uint32_t d) {
  const uint32_t id = idesc_f16(TILE, N, 0, 0);
  for (int kb = 0; kb < K / 16; ++kb)
    mma_f16(d, desc_k(a, TILE, 2 * kb), desc_k(b, N, 2 * kb), id, kb > 0 ? 1u : 0u);
}

// D[128 x N] (+)= G[128 x K] . W[K x N]: G K-major, W tile [K rows(out) x N cols(in)]
// read MN-major.
__device__ __forceinline__ void issue_dgrad(uint32_t g, int K, uint32_t w, int N, uint32_t d,
                                            bool accumulate) {
  const uint32_t id = idesc_f16(TILE, N, 0, 1);
  for (int kb = 0; kb < K / 16; ++kb)
    mma_f16(d, desc_k(g, TILE, 2 * kb), desc_mn(w, K, 2 * kb), id,
            (accumulate || kb > 0) ? 1u : 0u);
}

// Acc[M x N] (+)= A^T . B over the 128 samples: A tile [128 x M] (cols = M), B tile
// [128 x N] (cols = N), both MN-major with K = rows (an M = 128 A spans two adjacent
// 64-column tiles, an N = 32 B the first 32 columns of one tile).
__device__ __forceinline__ void issue_wgrad(uint32_t a, int M, uint32_t b, int N, uint32_t d,
                                            bool accumulate) {
  const uint32_t id = idesc_f16(M, N, 1, 1);
  for (int kb = 0; kb < TILE / 16; ++kb)
    mma_f16(d, desc_mn(a, TILE, 2 * kb), desc_mn(b, TILE, 2 * kb), id,
            (accumulate || kb > 0) ? 1u : 0u);
}

__device__ __forceinline__ void sh16f(float x, float y, float z, float* o) {
  const float xy = x * y, xz = x * z, yz = y * z, x2 = x * x, y2 = y * y, z2 = z * z;
  o[0] = 0.28209479177387814f;
  o[1] = -0.48860251190291987f * y;
  o[2] = 0.48860251190291987f * z;
  o[3] = -0.48860251190291987f * x;
  o[4] = 1.0925484305920792f * xy;
  o[5] = -1.0925484305920792f * yz;
  o[6] = 0.94617469575755997f * z2 - 0.31539156525251999f;
  o[7] = -1.0925484305920792f * xz;
  o[8] = 0.54627421529603959f * x2 - 0.54627421529603959f * y2;
  o[9] = 0.59004358992664352f * y * (-3.0f * x2 + y2);
  o[10] = 2.8906114426405538f * xy * z;
  o[11] = 0.45704579946446572f * y * (1.0f - 5.0f * z2);
  o[12] = 0.3731763325901154f * z * (5.0f * z2 - 3.0f);
  o[13] = 0.45704579946446572f * x * (1.0f - 5.0f * z2);
  o[14] = 1.4453057213202769f * z * (x2 - y2);
  o[15] = 0.59004358992664352f * x * (-x2 + 3.0f * y2);
}

// 8 fp32 -> one 16-byte fp16 chunk (column block cb of row r)
__device__ __forceinline__ void put8(uint8_t* tile, int r, int cb, const float* v) {
  uint4 q;
  __half2* h = reinterpret_cast<__half2*>(&q);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
  *reinterpret_cast<uint4*>(tile + tile_off(TILE, r, cb * 8)) = q;
}
// ReLU on the packed fp16 pair: fp16(max(x, 0)) == max(fp16(x), 0) (rounding is monotonic
// and keeps the sign), done by the conversion itself (cvt.rn.relu.f16x2.f32: one F2FP per
// pair, no separate max).  .x = a, .y = b as __floats2half2_rn; the first PTX source
// operand fills the upper half.
__device__ __forceinline__ __half2 relu_h2(float a, float b) {
  uint32_t u;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(u) : "f"(b), "f"(a));
  return *reinterpret_cast<__half2*>(&u);
}
// the same value as a conversion then HMNMX2: kept in the backward's forward recompute (which
// writes the activations to shared memory), where the folded form measured slower — c4
// k_mlp_bwd_tc 22.1 vs 22.5 ms per step (bench events), 16.0 vs 16.8 ms (ncu, serialised)
__device__ __forceinline__ __half2 relu_h2_max(float a, float b) {
  return __hmax2(__floats2half2_rn(a, b), __float2half2_rn(0.f));
}
__device__ __forceinline__ void put_relu8(uint8_t* tile, int r, int cb, const float* v) {
  uint4 q;
  __half2* h = reinterpret_cast<__half2*>(&q);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = relu_h2_max(v[2 * j], v[2 * j + 1]);
  *reinterpret_cast<uint4*>(tile + tile_off(TILE, r, cb * 8)) = q;
}
// g[j] = v[j] if the (post-relu, fp16) activation of column block cb is non-zero
__device__ __forceinline__ void relu_mask8(const uint8_t* tile, int r, int cb, const float* v,
                                           float* g) {
  const uint4 q = *reinterpret_cast<const uint4*>(tile + tile_off(TILE, r, cb * 8));
  const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    g[2 * j] = (u[j] & 0x7FFFu) ? v[2 * j] : 0.f;
    g[2 * j + 1] = (u[j] & 0x7FFF0000u) ? v[2 * j + 1] : 0.f;
  }
}
// weight-gradient flush: global add, and the value joins the non-finite check
__device__ __forceinline__ void flush_add(float* dst, float v, float& nonfinite) {
  atomicAdd(dst, v);
  nonfinite += v;
}

// fp16 hi/lo split of 8 gradients into Gh / Gl (column block cb).  An operand that
// overflows fp16 (inf) is not tested here: it makes the stage's MMA results non-finite,
// which the d(enc) and weight-gradient checks at the end of the tile / kernel catch.
__device__ __forceinline__ void put_grad8(uint8_t* Gh, uint8_t* Gl, int r, int cb, const float* g) {
  uint4 qh, ql;
  __half2* hh = reinterpret_cast<__half2*>(&qh);
  __half2* hl = reinterpret_cast<__half2*>(&ql);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 h = __floats2half2_rn(g[2 * j], g[2 * j + 1]);
    const float2 f = __half22float2(h);
    hh[j] = h;
    hl[j] = __floats2half2_rn(g[2 * j] - f.x, g[2 * j + 1] - f.y);
  }
  *reinterpret_cast<uint4*>(Gh + tile_off(TILE, r, cb * 8)) = qh;
  *reinterpret_cast<uint4*>(Gl + tile_off(TILE, r, cb * 8)) = ql;
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// Thread geometry: TPR threads per tile row.  warp w covers TMEM lanes 32*(w%4) and
// column slice w/4.
template <int TPR>
struct Geo {
  static constexpr int NT = TILE * TPR;
  __device__ static int row() { return ((threadIdx.x >> 5) & 3) * 32 + (threadIdx.x & 31); }
  __device__ static int part() { return TPR == 1 ? 0 : (int)(threadIdx.x >> 7); }
  __device__ static uint32_t lane_base() {
    return (uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16;
  }
};

// stage this thread's share of the 32 encoding features of row r (sample i, or zeros)
template <int TPR>
__device__ __forceinline__ void stage_enc(uint8_t* tile, int r, int part,
                                          const __half2* __restrict__ enc, int64_t n, int64_t i,
                                          bool valid) {
  constexpr int LV = 16 / TPR;
  uint4 q[LV / 4];
  __half2* h = reinterpret_cast<__half2*>(q);
#pragma unroll
  for (int l = 0; l < LV; ++l)
    h[l] = valid ? enc[(int64_t)(part * LV + l) * n + i] : __floats2half2_rn(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < LV / 4; ++c)
    *reinterpret_cast<uint4*>(tile + tile_off(TILE, r, (part * LV / 4 + c) * 8)) = q[c];
}

// one MMA round for a CTA-wide tile pipeline: make smem writes visible to the tensor
// core, issue from thread 0, wait for completion
// `overlap` runs on every thread after the MMAs are issued and before waiting for them
// (independent SIMT work hidden under the tensor-core latency).
struct NoOverlap {
  __device__ __forceinline__ void operator()(int) const {}
};

template <class F, class O = NoOverlap>
__device__ __forceinline__ void mma_round(uint64_t* bar, uint32_t& phase, F issue,
                                          const O& overlap = O(), int round = 0) {
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_fence_after();
    issue();
    mma_commit(bar);
  }
  overlap(round);
  mbar_wait(bar, phase);
  phase ^= 1u;
  __syncwarp();
  tc_fence_after();
}

struct FwdRow {
  float sigma, od0, rgb[3];  // valid in part 0
};

// Forward chain of one tile.  X0 = enc (pre-staged); activations go to X1 (h1d),
// X2 (cin), X3 (h1c), X4 (h2c) — X2 may alias X0, X3 may alias X1, X4 may alias X2.
// d0: 64 scratch columns, d1: 16 scratch columns.
// DENS: density branch only (a proposal field: its colour head is never used) — rounds
// L1d and L2d, no cin.
template <int TPR, bool DENS = false, class O = NoOverlap>
__device__ __forceinline__ FwdRow forward_tile(uint8_t* sw, uint8_t* X0, uint8_t* X1, uint8_t* X2,
                                               uint8_t* X3, uint8_t* X4, uint32_t tm_row,
                                               uint32_t tmem, uint32_t d0, uint32_t d1,
                                               uint64_t* bar, uint32_t& phase, float dx,
                                               float dy, float dz, const O& ov = O()) {
  using G = Geo<TPR>;
  const int r = G::row(), part = G::part();
  constexpr int C64 = 64 / TPR;  // columns of a 64-wide layer per thread
  const uint32_t sW = smem_u32(sw);
  float v[16];
  FwdRow out = {0.f, 0.f, {0.f, 0.f, 0.f}};
  // L1d
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X0), 32, sW + OW1D, 64, tmem + d0); }, ov, 0);
#pragma unroll
  for (int c = part * C64; c < (part + 1) * C64; c += 16) {
    tmem_ld16(tm_row + d0 + c, v);
    put_relu8(X1, r, c / 8, v);
    put_relu8(X1, r, c / 8 + 1, v + 8);
  }
  // L2d -> sigma, geo (part 0) ; SH(d) (last part)
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X1), 64, sW + OW2D, 16, tmem + d1); }, ov, 1);
  if (part == 0) {
    tmem_ld16(tm_row + d1, v);
    out.od0 = v[0];
    out.sigma = expf(fminf(fmaxf(v[0], -15.f), 15.f));
    if (!DENS) {
      put8(X2, r, 0, v);
      put8(X2, r, 1, v + 8);
    }
  }
  if (DENS) return out;
  if (part == TPR - 1) {
    sh16f(dx, dy, dz, v);
    put8(X2, r, 2, v);
    put8(X2, r, 3, v + 8);
  }
  // L1c
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X2), 32, sW + OW1C, 64, tmem + d0); }, ov, 2);
#pragma unroll
  for (int c = part * C64; c < (part + 1) * C64; c += 16) {
    tmem_ld16(tm_row + d0 + c, v);
    put_relu8(X3, r, c / 8, v);
    put_relu8(X3, r, c / 8 + 1, v + 8);
  }
  // L2c
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X3), 64, sW + OW2C, 64, tmem + d0); }, ov, 3);
#pragma unroll
  for (int c = part * C64; c < (part + 1) * C64; c += 16) {
    tmem_ld16(tm_row + d0 + c, v);
    put_relu8(X4, r, c / 8, v);
    put_relu8(X4, r, c / 8 + 1, v + 8);
  }
  // L3c
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X4), 64, sW + OW3C, 16, tmem + d1); }, ov, 4);
  if (part == 0) {
    tmem_ld16(tm_row + d1, v);
#pragma unroll
    for (int c = 0; c < 3; ++c) out.rgb[c] = 1.f / (1.f + expf(-v[c]));
  }
  return out;
}

__device__ __forceinline__ void load_dir(const double* __restrict__ rays, int64_t stride,
                                         const int32_t* __restrict__ rid, int64_t i, bool valid,
                                         float& dx, float& dy, float& dz) {
  dx = dy = dz = 0.f;
  if (valid) {
    const int64_t r = checked_ray(rid[i], stride);
    dx = (float)__ldg(rays + 3 * stride + r);
    dy = (float)__ldg(rays + 4 * stride + r);
    dz = (float)__ldg(rays + 5 * stride + r);
  }
}

// ---- forward kernel ---------------------------------------------------------------------
// The forward keeps its activations in TMEM: every layer's A operand is written there by
// the epilogue (tcgen05.st, lane = row, 32-bit column j = features 2j, 2j+1) and read by a
// "TS" tcgen05.mma (A from TMEM, weights from shared memory) — no activation round trip
// through shared memory, whose bandwidth the small-K SS MMAs were bound by (ncu: tensor
// pipe ~50 % active at 16 % of peak FLOP/s).  TMEM per CTA (128 columns, 4 CTAs/SM):
// D [0,64) accumulator, A1 [64,96) and A2 [96,128) activation buffers.
constexpr int FWD_TPR = 1;
constexpr uint32_t F_BAR = WBYTES, F_SMEM = F_BAR + 16;
constexpr uint32_t TF_D = 0, TF_A1 = 64, TF_A2 = 96, TF_COLS = 128;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
                 "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t h2bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// D[128 x N] = A[128 x K] . B^T with A in TMEM (K/2 columns at a_tmem), B a weight tile
__device__ __forceinline__ void issue_fwd_ts(uint32_t a_tmem, int K, uint32_t b, int N,
                                             uint32_t d) {
  const uint32_t id = idesc_f16(TILE, N, 0, 0);
  for (int kb = 0; kb < K / 16; ++kb) {
    const uint64_t bd = desc_k(b, N, 2 * kb);
    const uint32_t acc = kb > 0 ? 1u : 0u;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                 ::"r"(d), "r"(a_tmem + (uint32_t)(kb * 8)), "l"(bd), "r"(id), "r"(acc));
  }
}

// one TS round: the TMEM stores of every thread are complete and visible, thread 0 issues
__device__ __forceinline__ void ts_round(uint64_t* bar, uint32_t& phase, uint32_t a, int K,
                                         uint32_t b, int N, uint32_t d) {
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_fence_after();
    issue_fwd_ts(a, K, b, N, d);
    mma_commit(bar);
  }
  mbar_wait(bar, phase);
  phase ^= 1u;
  __syncwarp();
  tc_fence_after();
}

// ReLU + fp16 of the 64-wide D into an activation buffer (32 TMEM columns)
__device__ __forceinline__ void epi_relu64(uint32_t tm_row, uint32_t dst) {
  float v[16];
  uint32_t q[8];
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    tmem_ld16(tm_row + TF_D + c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      q[j] = h2bits(relu_h2(v[2 * j], v[2 * j + 1]));
    tmem_st8(tm_row + dst + c / 2, q);
  }
}

// Forward chain of one 128-sample tile; enc (K = 32) is already in A2.
template <bool DENS>
__device__ __forceinline__ FwdRow forward_tile_ts(uint32_t sW, uint32_t tmem, uint32_t tm_row,
                                                  uint64_t* bar, uint32_t& phase, float dx,
                                                  float dy, float dz) {
  FwdRow out = {0.f, 0.f, {0.f, 0.f, 0.f}};
  float v[16];
  uint32_t q[8];
  ts_round(bar, phase, tmem + TF_A2, 32, sW + OW1D, 64, tmem + TF_D);  // L1d
  epi_relu64(tm_row, TF_A1);
  ts_round(bar, phase, tmem + TF_A1, 64, sW + OW2D, 16, tmem + TF_D);  // L2d
  tmem_ld16(tm_row + TF_D, v);
  out.od0 = v[0];
  out.sigma = expf(fminf(fmaxf(v[0], -15.f), 15.f));
  if (DENS) return out;
  // cin = [geo (16) | SH(d) (16)] -> A2
#pragma unroll
  for (int j = 0; j < 8; ++j) q[j] = h2bits(__floats2half2_rn(v[2 * j], v[2 * j + 1]));
  tmem_st8(tm_row + TF_A2, q);
  sh16f(dx, dy, dz, v);
#pragma unroll
  for (int j = 0; j < 8; ++j) q[j] = h2bits(__floats2half2_rn(v[2 * j], v[2 * j + 1]));
  tmem_st8(tm_row + TF_A2 + 8, q);
  ts_round(bar, phase, tmem + TF_A2, 32, sW + OW1C, 64, tmem + TF_D);  // L1c
  epi_relu64(tm_row, TF_A1);
  ts_round(bar, phase, tmem + TF_A1, 64, sW + OW2C, 64, tmem + TF_D);  // L2c
  epi_relu64(tm_row, TF_A2);
  ts_round(bar, phase, tmem + TF_A2, 64, sW + OW3C, 16, tmem + TF_D);  // L3c
  tmem_ld8(tm_row + TF_D, v);
#pragma unroll
  for (int c = 0; c < 3; ++c) out.rgb[c] = 1.f / (1.f + expf(-v[c]));
  return out;
}

// Hash-grid encoding of this thread's row (FUSED forward): 16 levels gathered from the
// region's table, rounded to fp16, returned packed (16 half2) and (optionally) written
// to enc_out for the backward.  dir returned as float for the SH encoding.
__device__ __forceinline__ void encode_row(const VrHashGridDesc& g, const float2* __restrict__ table,
                                           const double* __restrict__ rays, int64_t stride,
                                           const double* __restrict__ t0,
                                           const double* __restrict__ t1,
                                           const int32_t* __restrict__ rid, int64_t n, int64_t i,
                                           bool valid, uint32_t* q,
                                           __half2* __restrict__ enc_out, float& dx, float& dy,
                                           float& dz) {
  __half2* h = reinterpret_cast<__half2*>(q);
  dx = dy = dz = 0.f;
  if (valid) {
    const int64_t ray = checked_ray(rid[i], stride);
    const double m = sample_mid(t0[i], t1[i]);
    double o[3], d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o[a] = __ldg(rays + a * stride + ray);
      d[a] = __ldg(rays + (3 + a) * stride + ray);
    }
    dx = (float)d[0];
    dy = (float)d[1];
    dz = (float)d[2];
    float u[3];
    norm_pos_od(g, box_inv(g), o, d, m, u);
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      Corners c;
      level_corners(g, l, u, c);
      const float2 f = gather_level(table + g.offset[l], c);
      h[l] = __floats2half2_rn(f.x, f.y);
    }
    if (enc_out) {
#pragma unroll
      for (int l = 0; l < 16; ++l) enc_out[(int64_t)l * n + i] = h[l];
    }
  } else {
#pragma unroll
    for (int l = 0; l < 16; ++l) h[l] = __floats2half2_rn(0.f, 0.f);
  }
}

// FUSED = true: the kernel computes the hash encoding itself (K2 + K3 in one pass);
// otherwise it reads enc (level-major half2) produced by vr_hash_fwd.  DENS: density
// branch only.
template <bool FUSED, bool DENS = false>
__global__ void __launch_bounds__(TILE * FWD_TPR, 4)
    k_mlp_fwd_tc(const __half* __restrict__ W, const __half2* __restrict__ enc,
                 const double* __restrict__ rays, int64_t stride, const int32_t* __restrict__ rid,
                 int64_t n, float4* __restrict__ out, const VrHashGridDesc g,
                 const float2* __restrict__ table, const double* __restrict__ t0,
                 const double* __restrict__ t1, __half2* __restrict__ enc_out) {
  using G = Geo<FWD_TPR>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sw = smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + F_BAR);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + F_BAR + 8);
  stage_weights(W, sw);
  if (threadIdx.x < 32) tmem_alloc(slot, TF_COLS);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  fence_async_smem();  // weights visible to the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t tm_row = tmem + G::lane_base();
  const uint32_t sW = smem_u32(sw);
  const int r = G::row();
  uint32_t phase = 0;
  const int64_t n_tiles = ceil_div(n, TILE);
  // !FUSED: the next tile's encodings and ray direction are loaded one tile ahead (raw,
  // converted at use) and its ray index two tiles ahead, so no tile waits on a global
  // load chain (rid -> rays) before its first MMA
  uint32_t qn[16];
  double dn[3] = {0.0, 0.0, 0.0};
  int32_t rid_ahead = 0;
  auto load_rid = [&](int64_t tile) -> int32_t {  // predicated load, no select (see bwd)
    const int64_t i = tile * TILE + r;
    int32_t v = 0;
    if (!DENS && tile < n_tiles && i < n) v = __ldg(rid + i);
    return v;
  };
  auto prefetch = [&](int64_t tile, int32_t ray) {
    const int64_t i = tile * TILE + r;
    const bool ok = tile < n_tiles && i < n;
    // colour MLP: zero, then predicated loads into the registers (a select between the
    // load and zero would wait for the load here instead of at the next tile: 10.7 -> 10.1
    // ms at c4); the 2-round density MLP is faster with the select form (4.8 vs 5.9 ms)
    if (DENS) {
#pragma unroll
      for (int l = 0; l < 16; ++l) qn[l] = ok ? h2bits(enc[(int64_t)l * n + i]) : 0u;
    } else {
#pragma unroll
      for (int l = 0; l < 16; ++l) qn[l] = 0u;
      if (ok) {
        const uint32_t* e32 = reinterpret_cast<const uint32_t*>(enc);
#pragma unroll
        for (int l = 0; l < 16; ++l) qn[l] = __ldg(e32 + (int64_t)l * n + i);
      }
    }
    if (!DENS && ok) {
      const int64_t rr = checked_ray(ray, stride);
#pragma unroll
      for (int a = 0; a < 3; ++a) dn[a] = __ldg(rays + (3 + a) * stride + rr);
    }
  };
  if (!FUSED && (int64_t)blockIdx.x < n_tiles) {
    prefetch(blockIdx.x, load_rid(blockIdx.x));
    rid_ahead = load_rid(blockIdx.x + (int64_t)gridDim.x);
  }
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t i = tile * TILE + r;
    const bool valid = i < n;
    float dx = 0.f, dy = 0.f, dz = 0.f;
    uint32_t q[16];
    if (FUSED) {
      encode_row(g, table, rays, stride, t0, t1, rid, n, i, valid, q, enc_out, dx, dy, dz);
    } else {
#pragma unroll
      for (int l = 0; l < 16; ++l) q[l] = qn[l];
      if (!DENS && valid) {
        dx = (float)dn[0];
        dy = (float)dn[1];
        dz = (float)dn[2];
      }
      prefetch(tile + gridDim.x, rid_ahead);
      rid_ahead = load_rid(tile + 2 * (int64_t)gridDim.x);
    }
    tmem_st8(tm_row + TF_A2, q);  // enc -> A2 (the previous tile's last MMA is complete)
    tmem_st8(tm_row + TF_A2 + 8, q + 8);
    const FwdRow f = forward_tile_ts<DENS>(sW, tmem, tm_row, bar, phase, dx, dy, dz);
    if (valid) out[i] = make_float4(f.sigma, f.rgb[0], f.rgb[1], f.rgb[2]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, TF_COLS);
  }
}

// ---- backward kernel --------------------------------------------------------------------
// 256 threads (2 per tile row), 2 CTAs per SM.  Smem per CTA: weights 20 KB + A (enc,
// then cin) 8 KB + X1 h1d 16 KB + X3 h1c 16 KB + X4 h2c 16 KB + Gh 16 KB + Gl 16 KB.
constexpr int BWD_TPR = 2;
// Density-only kernels (proposal fields) need W1d / W2d, enc, h1d and G only, and 128 TMEM
// columns (W1d, W2d^T accumulators + scratch): 62 KB of smem, 3 CTAs per SM instead of 2.
template <bool DENS>
struct BwdLayout {
  static constexpr uint32_t W = DENS ? OW1C : WBYTES;
  static constexpr uint32_t A = W, X1 = A + TILE * 32 * 2;
  static constexpr uint32_t X3 = DENS ? X1 : X1 + TILE * 64 * 2;  // unused when DENS
  static constexpr uint32_t X4 = DENS ? X1 : X3 + TILE * 64 * 2;  // unused when DENS
  static constexpr uint32_t GH = (DENS ? X1 : X4) + TILE * 64 * 2, GL = GH + TILE * 64 * 2;
  static constexpr uint32_t BAR = GL + TILE * 64 * 2, WMAX = BAR + 32, SMEM = WMAX + 32;
  static constexpr uint32_t D0 = DENS ? 64 : 192, COLS = DENS ? 128 : 256;
  static constexpr int CTAS = DENS ? 3 : 2;
};
constexpr uint32_t B_A = BwdLayout<false>::A, B_X1 = BwdLayout<false>::X1,
                   B_X3 = BwdLayout<false>::X3, B_X4 = BwdLayout<false>::X4,
                   B_GH = BwdLayout<false>::GH, B_GL = BwdLayout<false>::GL,
                   B_BAR = BwdLayout<false>::BAR, B_WMAX = BwdLayout<false>::WMAX,
                   B_SMEM = BwdLayout<false>::SMEM;
// TMEM columns: weight-gradient accumulators, then scratch.  W1d, W1c, W2c: M = 128
// (rows 0..63 hi, 64..127 lo products); W2d^T, W3c^T: M = 64, columns [hi 16 | lo 16].
// The forward's second scratch slice aliases the first (its results are consumed before
// the next round is issued).
constexpr uint32_t T_W1D = 0, T_W2DT = 32, T_W1C = 64, T_W2C = 96, T_W3CT = 160, T_D0 = 192,
                   T_D1 = T_D0, T_COLS = 256;
static_assert(B_GL == B_GH + TILE * 64 * 2, "stacked wgrad operand needs Gl right after Gh");

// Inputs of one row for one tile, prefetched into registers one tile ahead.  The loads are
// only ISSUED here; every use of a loaded value (the direction's float conversion, the
// gradient scale, the position) happens when the tile is processed, so the thread does not
// wait on them inside the prefetch (measured: the conversions right after the loads were
// the top long-scoreboard stalls of the c4 backward).  The sample's ray index, which the
// direction loads depend on, is loaded one tile earlier still (rid_ahead).
struct RowIn {
  __half2 enc[16 / BWD_TPR];
  double d[3];   // ray direction (raw float64)
  float u[3];    // normalised hash-grid position (FUSED backward only)
  float4 gin;    // upstream gradient, unscaled
};

template <bool FUSED, bool DENS>
__device__ __forceinline__ void fetch_row(RowIn& x, const __half2* __restrict__ enc,
                                          const double* __restrict__ rays, int64_t stride,
                                          int32_t ray, const float4* __restrict__ dsr, int64_t n,
                                          int64_t i, bool valid, int part,
                                          const VrHashGridDesc& g,
                                          const double* __restrict__ t0,
                                          const double* __restrict__ t1,
                                          const float* __restrict__ pos) {
  constexpr int LV = 16 / BWD_TPR;
  // zero first, then predicated loads straight into the registers (a select between the
  // loaded value and zero would wait for the load right here)
#pragma unroll
  for (int l = 0; l < LV; ++l) x.enc[l] = __floats2half2_rn(0.f, 0.f);
  x.gin = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) {
#pragma unroll
    for (int l = 0; l < LV; ++l) x.enc[l] = __ldg(enc + (int64_t)(part * LV + l) * n + i);
    if (part == 0) x.gin = __ldg(dsr + i);
  }
  x.d[0] = x.d[1] = x.d[2] = 0.0;
  x.u[0] = x.u[1] = x.u[2] = 0.f;
  if (valid && !DENS) {  // the density branch has no view direction
    const int64_t r = checked_ray(ray, stride);
#pragma unroll
    for (int a = 0; a < 3; ++a) x.d[a] = __ldg(rays + (3 + a) * stride + r);
    if (FUSED && pos == nullptr) {  // positions recomputed from the ray (no forward store)
      double o[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) o[a] = __ldg(rays + a * stride + r);
      norm_pos_od(g, box_inv(g), o, x.d, sample_mid(t0[i], t1[i]), x.u);
    } else if (FUSED) {  // positions written by the hash-grid forward
      x.u[0] = __ldcs(pos + i);
      x.u[1] = __ldcs(pos + n + i);
      x.u[2] = __ldcs(pos + 2 * n + i);
    }
  }
}

__device__ __forceinline__ void put_enc(uint8_t* tile, int r, int part, const RowIn& x) {
  constexpr int LV = 16 / BWD_TPR;
  const uint4* q = reinterpret_cast<const uint4*>(x.enc);
#pragma unroll
  for (int c = 0; c < LV / 4; ++c)
    *reinterpret_cast<uint4*>(tile + tile_off(TILE, r, (part * LV / 4 + c) * 8)) = q[c];
}

// FUSED = true: instead of writing d(enc) to global memory, each thread scatters its
// row's hash-grid gradients (its 8 levels) straight from the last epilogue (K3 + K2
// backward in one pass); the atomics overlap other tiles' tensor-core rounds.
template <bool FUSED, bool DENS = false>
__global__ void __launch_bounds__(TILE * BWD_TPR, BwdLayout<DENS>::CTAS)
    k_mlp_bwd_tc(const __half* __restrict__ W, const __half2* __restrict__ enc,
                 const double* __restrict__ rays, int64_t stride, const int32_t* __restrict__ rid,
                 int64_t n, const float4* __restrict__ dsr, const float4* __restrict__ sig,
                 float* __restrict__ gW,
                 float2* __restrict__ denc, int32_t* err, const VrHashGridDesc hg,
                 const RepPlan plan, const double* __restrict__ t0,
                 const double* __restrict__ t1, float2* __restrict__ grad_table,
                 float2* __restrict__ rep_ws, const float* __restrict__ pos,
                 const int32_t* __restrict__ rows, const int32_t* __restrict__ n_rows) {
  using G = Geo<BWD_TPR>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sw = smem;
  using LY = BwdLayout<DENS>;
  constexpr uint32_t T_D0 = LY::D0, T_D1 = LY::D0, T_COLS = LY::COLS;
  uint8_t* A = smem + LY::A;   // enc during L1d, cin afterwards
  uint8_t* X1 = smem + LY::X1;
  uint8_t* X3 = smem + LY::X3;
  uint8_t* X4 = smem + LY::X4;  // h2c, then enc (re-staged) for the last stage
  uint8_t* Gh = smem + LY::GH;
  uint8_t* Gl = smem + LY::GL;
  uint64_t* barA = reinterpret_cast<uint64_t*>(smem + LY::BAR);  // forward / dgrad MMAs
  uint64_t* barB = barA + 1;                                     // wgrad MMAs
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + LY::BAR + 16);
  const int r = G::row(), part = G::part();
  const int lane = threadIdx.x & 31, wq = (threadIdx.x >> 5) & 3;
  stage_weights<DENS>(W, sw);
  if (threadIdx.x < 32) tmem_alloc(slot, T_COLS);
  if (threadIdx.x == 0) {
    mbar_init(barA, 1);
    mbar_init(barB, 1);
    fence_barrier_init();
  }
  // Active rows: with a row list (vr_active_rows) the tiles are cut from rows[0, m) — the
  // samples whose upstream gradient is non-zero — instead of [0, n); compact position j
  // stands for sample rows[j], and d(enc) is written at compact position j.
  const int64_t n_act = rows ? (int64_t)__ldg(n_rows) : n;
  const int64_t n_tiles = ceil_div(n_act, TILE);
  auto sample_of = [&](int64_t j) -> int64_t {  // the gradient-scale pre-pass
    if (!rows) return j;
    const int64_t i = __ldg(rows + j);
    return VR_CHECK(i >= 0 && i < n) ? i : 0;  // (checked build: a bad row list entry)
  };
  // Gradient scale of this CTA (a power of two, so exact both ways): the fp16 hi + lo
  // split of G keeps 22 significant bits only while lo = G - fp16(G) is an fp16 normal,
  // i.e. |G| >= 2^-3; below that lo's absolute precision is 2^-24 (measured: d(enc) at
  // 4e-5 relative for the typical |G| ~ 1e-3 of a sum-of-squares loss).  The upstream
  // magnitudes of the row's first two stages (|drgb| * rgb (1 - rgb) <= |drgb| / 4 and
  // |dsigma| * sigma, sigma = the forward's output) over the CTA's rows set S so that
  // their maximum lands at 2^4 — 2^12 of headroom below fp16's 65504 for the growth
  // through the four weight matrices (overflow is flagged, VR_FLAG_GRAD_OVERFLOW).  The
  // weight-gradient accumulators are per CTA, so one scale per CTA is exact: d(enc) and
  // the flushed weight gradients are multiplied by 1/S.
  float gscale = 1.f, ginv = 1.f;
  if (sig) {
    uint32_t* wmax = reinterpret_cast<uint32_t*>(smem + LY::WMAX);
    float m = 0.f;
    // four of this thread's tiles per iteration, their loads independent (the row-list
    // lookup and the two loads behind it were a serial latency chain per tile)
    constexpr int PU = 4;
    const int64_t tstep = 2 * (int64_t)gridDim.x;
    for (int64_t t0_ = blockIdx.x + (int64_t)part * gridDim.x; t0_ < n_tiles; t0_ += PU * tstep) {
      int64_t ii[PU];
#pragma unroll
      for (int k = 0; k < PU; ++k) {
        const int64_t j = (t0_ + k * tstep) * TILE + r;
        ii[k] = j < n_act ? sample_of(j) : -1;
      }
      float4 g4[PU];
      float sg[PU];
#pragma unroll
      for (int k = 0; k < PU; ++k) {
        g4[k] = ii[k] >= 0 ? __ldg(dsr + ii[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
        sg[k] = ii[k] >= 0 ? __ldg(&sig[ii[k]].x) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < PU; ++k) {
        const float a = fabsf(g4[k].x * sg[k]);
        m = fmaxf(m, DENS ? a : fmaxf(a, 0.25f * fmaxf(fabsf(g4[k].y),
                                                       fmaxf(fabsf(g4[k].z), fabsf(g4[k].w)))));
      }
    }
    // non-negative floats order like their bit patterns (NaN above inf)
    const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
    if (lane == 0) wmax[threadIdx.x >> 5] = wm;
    __syncthreads();
    uint32_t mb = 0;
#pragma unroll
    for (int k = 0; k < TILE * BWD_TPR / 32; ++k) mb = max(mb, wmax[k]);
    const float mx = __uint_as_float(mb);
    if (mx > 0.f && isfinite(mx)) {
      int k;
      frexpf(mx, &k);  // 2^(k-1) <= mx < 2^k
      const int e = min(64, max(-64, 4 - k));
      gscale = ldexpf(1.f, e);
      ginv = ldexpf(1.f, -e);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t tm_row = tmem + G::lane_base();
  const uint32_t sW = smem_u32(sw);
  const uint32_t sA = smem_u32(A), sX1 = smem_u32(X1), sX3 = smem_u32(X3), sX4 = smem_u32(X4),
                 sGh = smem_u32(Gh), sGl = smem_u32(Gl), sGh16 = sGh + 2 * TILE * 16;
  uint32_t phA = 0, phB = 0;
  bool wgrad_pending = false;
  float nonfinite = 0.f;  // sum of this thread's d(enc) values: inf / NaN if any is
  bool acc = false;  // weight-gradient accumulators hold data
  constexpr int C64 = 64 / BWD_TPR, C16 = 16 / BWD_TPR;
  const int c64 = part * C64, c16 = part * C16;

  // one backward stage: wait until the previous wgrad released G, write G = hi + lo,
  // issue dX = G.W (commit -> barA) then dW += G^T X (commit -> barB), wait for dX only;
  // the wgrad MMAs overlap the following epilogue.
  auto stage = [&](const float* g, int width_here, int col0, bool total16, auto issue_dgrad_fn,
                   auto issue_wgrad_fn, auto overlap_fn) {
    if (wgrad_pending) {
      mbar_wait(barB, phB);
      phB ^= 1u;
    }
    for (int c = 0; c < width_here; c += 8)  // 16-wide G: lo part -> Gh columns 16..31
      put_grad8(Gh, total16 ? Gh + 2 * TILE * 16 : Gl, r, (col0 + c) / 8, g + c);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
      tc_fence_after();
      issue_dgrad_fn();
      mma_commit(barA);
      issue_wgrad_fn();
      mma_commit(barB);
    }
    wgrad_pending = true;
    overlap_fn();
    mbar_wait(barA, phA);
    phA ^= 1u;
    __syncwarp();
    tc_fence_after();
  };

  // deferred hash-grid scatter of the previous tile (FUSED): its d(enc) (this thread's
  // 8 levels) and position are parked in registers and one level is scattered in each of
  // the next tile's first 8 tensor-core waits (5 forward rounds, backward stages 1-3), so
  // the atomics stream through the whole tile instead of bunching up
  bool pending = false;
  float pk[16], pu[3];
  const int gwarp = blockIdx.x * (TILE * BWD_TPR / 32) + (threadIdx.x >> 5);
  // lane pairs (scatter_half): lanes 2j, 2j+1 hold rows r, r+1; each of the rows is
  // scattered by both lanes, lane p adding the corners with cx = p
  auto scatter_one = [&](int j) {
    if (FUSED && pending) {
      const int p = lane & 1;
      const float2 mine = make_float2(pk[2 * j], pk[2 * j + 1]);
      const float2 other = make_float2(__shfl_xor_sync(0xffffffffu, mine.x, 1),
                                       __shfl_xor_sync(0xffffffffu, mine.y, 1));
      float uo[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) uo[a] = __shfl_xor_sync(0xffffffffu, pu[a], 1);
      // pass 0: the even lane's row, pass 1: the odd lane's row
      const float2 d0 = p ? other : mine, d1 = p ? mine : other;
      const float* u0 = p ? uo : pu;
      const float* u1 = p ? pu : uo;
      const int l = 8 * part + j;
      if (d0.x != 0.f || d0.y != 0.f)
        scatter_half(hg, plan, l, u0, d0, p, gwarp, grad_table, rep_ws);
      if (d1.x != 0.f || d1.y != 0.f)
        scatter_half(hg, plan, l, u1, d1, p, gwarp, grad_table, rep_ws);
    }
  };
  auto scatter_ov = [&](int round) { scatter_one(round); };

  RowIn nxt;
  // inputs are prefetched one tile ahead; the ray index they depend on one tile earlier
  // (rid_a), and the sample index that depends on (a row list) one tile earlier still
  // Both lookups are predicated loads into a pre-set int32 register (no select and no
  // widening right after the load, which would wait for it at the issue point — ncu showed
  // the row-list load as the top stall of the sparse backward before); the values are
  // consumed a tile later.
  auto index_of = [&](int64_t tile) -> int32_t {
    const int64_t j = tile * TILE + r;
    int32_t v = -1;
    if (tile < n_tiles && j < n_act) v = rows ? __ldg(rows + j) : (int32_t)j;
    if (rows && !VR_CHECK(v < n)) v = 0;  // (checked build only: a bad row-list entry)
    return v;
  };
  auto load_rid = [&](int32_t i) -> int32_t {
    int32_t v = 0;
    if (!DENS && i >= 0) v = __ldg(rid + i);
    return v;
  };
  const int64_t G1 = gridDim.x;
  int32_t i_a = -1, i_b = -1;  // sample index of this row in the next tile / the one after
  int32_t rid_a = 0;           // ray index of this row in the next tile
  if ((int64_t)blockIdx.x < n_tiles) {
    const int32_t i0 = index_of(blockIdx.x);
    fetch_row<FUSED, DENS>(nxt, enc, rays, stride, load_rid(i0), dsr, n, i0, i0 >= 0, part, hg,
                           t0, t1, pos);
    i_a = index_of(blockIdx.x + G1);
    rid_a = load_rid(i_a);
    i_b = index_of(blockIdx.x + 2 * G1);
  }
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += G1) {
    const int64_t jrow = tile * TILE + r;  // compact position (== the sample without a list)
    const bool valid = jrow < n_act;
    const RowIn cur = nxt;
    if (tile + G1 < n_tiles) {  // prefetch the next tile's inputs (loads only)
      fetch_row<FUSED, DENS>(nxt, enc, rays, stride, rid_a, dsr, n, i_a, i_a >= 0, part, hg, t0,
                             t1, pos);
      rid_a = load_rid(i_b);
      i_a = i_b;
      i_b = index_of(tile + 3 * G1);
    }
    if (wgrad_pending) {  // the previous tile's last wgrad reads X4/Gh/Gl
      mbar_wait(barB, phB);
      phB ^= 1u;
      wgrad_pending = false;
    }
    put_enc(A, r, part, cur);
    // forward recompute: A(enc) -> X1(h1d) -> A(cin) -> X3(h1c) -> X4(h2c)
    const FwdRow f = forward_tile<BWD_TPR, DENS>(sw, A, X1, A, X3, X4, tm_row, tmem, T_D0, T_D1,
                                                 barA, phA, (float)cur.d[0], (float)cur.d[1],
                                                 (float)cur.d[2], scatter_ov);
    const float4 gin = make_float4(cur.gin.x * gscale, cur.gin.y * gscale, cur.gin.z * gscale,
                                   cur.gin.w * gscale);
    float g[C64];
    float v[16];
    const bool a_w = acc;
    if (DENS) {  // density branch only: no colour-head stages, enc still in A
#pragma unroll
      for (int j = 0; j < C16; ++j) g[j] = 0.f;
      if (part == 0 && f.od0 > -15.f && f.od0 < 15.f) g[0] = gin.x * f.sigma;
      stage(g, C16, c16, true,
            [&] {
              issue_dgrad(sGh, 16, sW + OW2D, 64, tmem + T_D0, false);  // dod . W2d
              issue_dgrad(sGh16, 16, sW + OW2D, 64, tmem + T_D0, true);
            },
            [&] { issue_wgrad(sX1, 64, sGh, 32, tmem + T_W2DT, a_w); }, [] {});
#pragma unroll
      for (int c = 0; c < C64; c += 16) {
        tmem_ld16(tm_row + T_D0 + c64 + c, v);
        relu_mask8(X1, r, (c64 + c) / 8, v, g + c);
        relu_mask8(X1, r, (c64 + c) / 8 + 1, v + 8, g + c + 8);
      }
      stage(g, C64, c64, false,
            [&] {
              issue_dgrad(sGh, 64, sW + OW1D, 32, tmem + T_D0, false);  // denc = dh1d . W1d
              issue_dgrad(sGl, 64, sW + OW1D, 32, tmem + T_D0, true);
            },
            [&] { issue_wgrad(sGh, 128, sA, 32, tmem + T_W1D, a_w); }, [] {});
      tmem_ld16(tm_row + T_D0 + 16 * part, v);
      if (valid) {
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          denc[(int64_t)(8 * part + j / 2) * n + jrow] = make_float2(v[j] * ginv, v[j + 1] * ginv);
          nonfinite += v[j] + v[j + 1];
        }
      }
      acc = true;
      continue;
    }

    // stage 1, colour head: g_o = drgb * rgb (1 - rgb) padded to 16 columns
#pragma unroll
    for (int j = 0; j < C16; ++j) g[j] = 0.f;
    if (part == 0) {
      g[0] = gin.y * f.rgb[0] * (1.f - f.rgb[0]);
      g[1] = gin.z * f.rgb[1] * (1.f - f.rgb[1]);
      g[2] = gin.w * f.rgb[2] * (1.f - f.rgb[2]);
    }
    stage(g, C16, c16, true,
          [&] {
            issue_dgrad(sGh, 16, sW + OW3C, 64, tmem + T_D0, false);  // g_o . W3c
            issue_dgrad(sGh16, 16, sW + OW3C, 64, tmem + T_D0, true);
          },
          [&] { issue_wgrad(sX4, 64, sGh, 32, tmem + T_W3CT, a_w); },  // dW3c^T += h2c^T g_o
          [&] { scatter_one(5); });
    // dh2c = (g_o . W3c) * relu'(h2c)
#pragma unroll
    for (int c = 0; c < C64; c += 16) {
      tmem_ld16(tm_row + T_D0 + c64 + c, v);
      relu_mask8(X4, r, (c64 + c) / 8, v, g + c);
      relu_mask8(X4, r, (c64 + c) / 8 + 1, v + 8, g + c + 8);
    }
    stage(g, C64, c64, false,
          [&] {
            issue_dgrad(sGh, 64, sW + OW2C, 64, tmem + T_D0, false);  // dh2c . W2c
            issue_dgrad(sGl, 64, sW + OW2C, 64, tmem + T_D0, true);
          },
          [&] { issue_wgrad(sGh, 128, sX3, 64, tmem + T_W2C, a_w); },  // dW2c += dh2c^T h1c
          [&] { scatter_one(6); });
    // dh1c = (dh2c . W2c) * relu'(h1c)
#pragma unroll
    for (int c = 0; c < C64; c += 16) {
      tmem_ld16(tm_row + T_D0 + c64 + c, v);
      relu_mask8(X3, r, (c64 + c) / 8, v, g + c);
      relu_mask8(X3, r, (c64 + c) / 8 + 1, v + 8, g + c + 8);
    }
    // the stage-1 wgrad (reads X4) is complete once stage() below has waited on barB;
    // enc is re-staged into X4 after that, before stage 5 needs it
    stage(g, C64, c64, false,
          [&] {
            issue_dgrad(sGh, 64, sW + OW1C, 32, tmem + T_D0, false);  // dh1c . W1c
            issue_dgrad(sGl, 64, sW + OW1C, 32, tmem + T_D0, true);
          },
          [&] { issue_wgrad(sGh, 128, sA, 32, tmem + T_W1C, a_w); },  // dW1c += dh1c^T cin
          [&] { scatter_one(7); });
    put_enc(X4, r, part, cur);
    // d od = dcin[0:16]; + dsigma * sigma on od0 (trunc-exp inside the clamp range)
    tmem_ld8(tm_row + T_D0 + c16, v);
#pragma unroll
    for (int j = 0; j < C16; ++j) g[j] = v[j];
    if (part == 0 && f.od0 > -15.f && f.od0 < 15.f) g[0] += gin.x * f.sigma;
    stage(g, C16, c16, true,
          [&] {
            issue_dgrad(sGh, 16, sW + OW2D, 64, tmem + T_D0, false);  // dod . W2d
            issue_dgrad(sGh16, 16, sW + OW2D, 64, tmem + T_D0, true);
          },
          [&] { issue_wgrad(sX1, 64, sGh, 32, tmem + T_W2DT, a_w); },  // dW2d^T += h1d^T dod
          [] {});
    // dh1d = (dod . W2d) * relu'(h1d)
#pragma unroll
    for (int c = 0; c < C64; c += 16) {
      tmem_ld16(tm_row + T_D0 + c64 + c, v);
      relu_mask8(X1, r, (c64 + c) / 8, v, g + c);
      relu_mask8(X1, r, (c64 + c) / 8 + 1, v + 8, g + c + 8);
    }
    stage(g, C64, c64, false,
          [&] {
            issue_dgrad(sGh, 64, sW + OW1D, 32, tmem + T_D0, false);  // denc = dh1d . W1d
            issue_dgrad(sGl, 64, sW + OW1D, 32, tmem + T_D0, true);
          },
          [&] { issue_wgrad(sGh, 128, sX4, 32, tmem + T_W1D, a_w); },  // dW1d += dh1d^T enc
          [] {});
    // d(enc) of this thread's levels part*8 .. part*8+7
    tmem_ld16(tm_row + T_D0 + 16 * part, v);
    if (valid) {
#pragma unroll
      for (int j = 0; j < 16; ++j) nonfinite += v[j];
    }
    if (FUSED) {
#pragma unroll
      for (int j = 0; j < 16; ++j) pk[j] = valid ? v[j] * ginv : 0.f;
      pu[0] = cur.u[0];
      pu[1] = cur.u[1];
      pu[2] = cur.u[2];
      pending = true;
    } else if (valid) {
#pragma unroll
      for (int j = 0; j < 16; j += 2)
        denc[(int64_t)(8 * part + j / 2) * n + jrow] = make_float2(v[j] * ginv, v[j + 1] * ginv);
    }
    acc = true;
  }
  if (wgrad_pending) {
    mbar_wait(barB, phB);
    phB ^= 1u;
  }
  if (FUSED && pending) {  // the CTA's last tile
#pragma unroll
    for (int j = 0; j < 8; ++j) scatter_one(j);
  }
  // ---- flush the weight-gradient accumulators (M = 64: row 16q+t at lane 32q+t) -----
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (acc) {
    // M = 128 accumulators: row 32*wq + lane (rows >= 64 hold the lo products of row - 64)
    const int m2 = (wq * 32 + lane) & 63;
    // M = 64 accumulators: row 16q+t at lane 32q+t; columns [hi 16 | lo 16]
    const int m = wq * 16 + lane;  // valid for lane < 16
    float v[16], w[16];
    // this warp's column half of each accumulator
    tmem_ld16(tm_row + T_W1D + 16 * part, v);
    for (int j = 0; j < 16; ++j) flush_add(gW + VR_MLP_W1D + m2 * 32 + 16 * part + j, v[j] * ginv, nonfinite);
    tmem_ld8(tm_row + T_W2DT + 8 * part, v);
    tmem_ld8(tm_row + T_W2DT + 16 + 8 * part, w);
    if (lane < 16)
      for (int j = 0; j < 8; ++j)
        flush_add(gW + VR_MLP_W2D + (8 * part + j) * 64 + m, (v[j] + w[j]) * ginv, nonfinite);
    if (!DENS) {  // the colour accumulators (never written in a density-only kernel)
      tmem_ld16(tm_row + T_W1C + 16 * part, v);
      for (int j = 0; j < 16; ++j)
        flush_add(gW + VR_MLP_W1C + m2 * 32 + 16 * part + j, v[j] * ginv, nonfinite);
#pragma unroll
      for (int c = 0; c < 32; c += 16) {
        tmem_ld16(tm_row + T_W2C + 32 * part + c, v);
        for (int j = 0; j < 16; ++j)
          flush_add(gW + VR_MLP_W2C + m2 * 64 + 32 * part + c + j, v[j] * ginv, nonfinite);
      }
      if (part == 0) {
        tmem_ld8(tm_row + T_W3CT, v);
        tmem_ld8(tm_row + T_W3CT + 16, w);
        if (lane < 16)
          for (int j = 0; j < 3; ++j)
            flush_add(gW + VR_MLP_W3C + j * 64 + m, (v[j] + w[j]) * ginv, nonfinite);
      }
    }
  }
  // an fp16 gradient operand that overflowed (or a non-finite upstream) left inf / NaN in
  // d(enc) or in a weight-gradient accumulator
  if (__any_sync(0xffffffffu, !isfinite(nonfinite)) && lane == 0)
    atomicOr(err, VR_FLAG_GRAD_OVERFLOW);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, T_COLS);
  }
}

}  // namespace mlp
}  // namespace vr

using namespace vr;

namespace {

// set on every launch (a host call of ~1 us): no process-wide flag, so any device and any
// host thread get the attribute on the context they launch in
template <class K>
int set_smem(K kernel, uint32_t bytes, const char* who) {
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess) {
    set_error(who);
    return VR_ERR_CUDA;
  }
  return VR_OK;
}

template <bool FUSED, bool DENS = false>
int launch_fwd(const void* w, const void* enc, const double* rays, int64_t stride,
               const int32_t* rid, int64_t n, float* out, const VrHashGridDesc* g,
               const float* table, const double* t0, const double* t1, void* enc_out,
               void* stream) {
  int rc = set_smem(mlp::k_mlp_fwd_tc<FUSED, DENS>, mlp::F_SMEM, "mlp fwd: smem attribute");
  if (rc != VR_OK) return rc;
  VrHashGridDesc gd;
  if (g) gd = *g; else memset(&gd, 0, sizeof(gd));
  const int64_t tiles = ceil_div(n, mlp::TILE);
  const int grid = (int)(tiles < VR_NUM_SMS * 4 ? tiles : VR_NUM_SMS * 4);
  mlp::k_mlp_fwd_tc<FUSED, DENS><<<grid, mlp::TILE * mlp::FWD_TPR, mlp::F_SMEM,
                                   (cudaStream_t)stream>>>(
      (const __half*)w, (const __half2*)enc, rays, stride, rid, n, reinterpret_cast<float4*>(out),
      gd, reinterpret_cast<const float2*>(table), t0, t1, (__half2*)enc_out);
  return check_launch("vr_mlp_fwd_tc");
}

template <bool FUSED, bool DENS = false>
int launch_bwd(const void* w, const void* enc, const double* rays, int64_t stride,
               const int32_t* rid, int64_t n, const float* dsr, const float* sig, float* gW,
               float* denc, int32_t* err, const VrHashGridDesc* g, const double* t0, const double* t1,
               float* grad_table, void* ws, size_t ws_bytes, const float* pos,
               const int32_t* rows, const int32_t* n_rows, void* stream, int max_ctas = 0) {
  using LY = mlp::BwdLayout<DENS>;
  if (n > INT32_MAX) {  // the prefetch pipeline carries sample indices as int32
    set_error("vr_mlp_bwd_tc: more than 2^31 - 1 samples in one call");
    return VR_ERR_BAD_ARG;
  }
  int rc = set_smem(mlp::k_mlp_bwd_tc<FUSED, DENS>, LY::SMEM, "mlp bwd: smem attribute");
  if (rc != VR_OK) return rc;
  VrHashGridDesc gd;
  RepPlan plan;
  int64_t ws_entries = 0, red = 0;
  memset(&plan, 0, sizeof(plan));
  if (g) {
    gd = *g;
    plan = hash_rep_plan(g, &ws_entries, &red);
    if (!ws || ws_bytes < (size_t)ws_entries * sizeof(float2)) plan.n_rep = 0;
  } else {
    memset(&gd, 0, sizeof(gd));
  }
  const int64_t tiles = ceil_div(n, mlp::TILE);
  const int full = VR_NUM_SMS * LY::CTAS;
  const int cap = max_ctas > 0 && max_ctas < full ? max_ctas : full;
  const int grid = (int)(tiles < cap ? tiles : cap);
  mlp::k_mlp_bwd_tc<FUSED, DENS><<<grid, mlp::TILE * mlp::BWD_TPR, LY::SMEM,
                                   (cudaStream_t)stream>>>(
      (const __half*)w, (const __half2*)enc, rays, stride, rid, n,
      reinterpret_cast<const float4*>(dsr), reinterpret_cast<const float4*>(sig), gW,
      reinterpret_cast<float2*>(denc), err, gd, plan, t0, t1,
      reinterpret_cast<float2*>(grad_table),
      reinterpret_cast<float2*>(ws), pos, rows, n_rows);
  rc = check_launch("vr_mlp_bwd_tc");
  if (rc != VR_OK || !FUSED) return rc;
  return hash_rep_reduce(&gd, plan, red, grad_table, ws, stream);
}

}  // namespace

extern "C" int vr_mlp_fwd_tc(const void* w, const void* enc, const double* rays, int64_t stride,
                             const int32_t* rid, int64_t n, float* out, void* stream) {
  if (n < 0 || !w) {
    set_error("vr_mlp_fwd_tc: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  return launch_fwd<false>(w, enc, rays, stride, rid, n, out, nullptr, nullptr, nullptr, nullptr,
                           nullptr, stream);
}

extern "C" int vr_mlp_bwd_tc(const void* w, const void* enc, const double* rays, int64_t stride,
                             const int32_t* rid, int64_t n, const float* dsr, const float* sig,
                             float* gW, float* denc, int32_t* err, int32_t max_ctas,
                             const int32_t* rows, const int32_t* n_rows, void* stream) {
  if (n < 0 || !w || !gW || !denc || !err || (!rows != !n_rows)) {
    set_error("vr_mlp_bwd_tc: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  return launch_bwd<false>(w, enc, rays, stride, rid, n, dsr, sig, gW, denc, err, nullptr,
                           nullptr, nullptr, nullptr, nullptr, 0, nullptr, rows, n_rows, stream,
                           max_ctas);
}

// density branch only (proposal fields): sigma of the same MLP, rgb = 0; the backward takes
// dL/dsigma (dsig_rgb[i].x) and writes d(enc) and the density weights' gradients only
extern "C" int vr_mlp_fwd_tc_density(const void* w, const void* enc, int64_t n, float* out,
                                     void* stream) {
  if (n < 0 || !w || (n > 0 && (!enc || !out))) {
    set_error("vr_mlp_fwd_tc_density: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  return launch_fwd<false, true>(w, enc, nullptr, 0, nullptr, n, out, nullptr, nullptr, nullptr,
                                 nullptr, nullptr, stream);
}

extern "C" int vr_mlp_bwd_tc_density(const void* w, const void* enc, const double* rays,
                                     int64_t stride, const int32_t* rid, int64_t n,
                                     const float* dsr, const float* sig, float* gW, float* denc,
                                     int32_t* err, int32_t max_ctas, const int32_t* rows,
                                     const int32_t* n_rows, void* stream) {
  if (n < 0 || !w || !gW || !denc || !err || (!rows != !n_rows)) {
    set_error("vr_mlp_bwd_tc_density: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  return launch_bwd<false, true>(w, enc, rays, stride, rid, n, dsr, sig, gW, denc, err, nullptr,
                                 nullptr, nullptr, nullptr, nullptr, 0, nullptr, rows, n_rows,
                                 stream, max_ctas);
}

extern "C" int vr_field_fwd_tc(const VrHashGridDesc* g, const float* table, const void* w,
                               const double* rays, int64_t stride, const double* t0,
                               const double* t1, const int32_t* rid, int64_t n, void* enc_out,
                               float* out, void* stream) {
  if (!valid_grid(g) || g->n_levels != 16 || n < 0 || !w || !table) {
    set_error("vr_field_fwd_tc: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  return launch_fwd<true>(w, nullptr, rays, stride, rid, n, out, g, table, t0, t1, enc_out,
                          stream);
}

extern "C" int vr_field_bwd_tc(const VrHashGridDesc* g, const void* w, const void* enc,
                               const double* rays, int64_t stride, const double* t0,
                               const double* t1, const int32_t* rid, int64_t n, const float* dsr,
                               const float* sig, float* gW, float* grad_table, void* ws,
                               size_t ws_bytes, int32_t* err, const float* pos,
                               const int32_t* rows, const int32_t* n_rows, void* stream) {
  if (!valid_grid(g) || g->n_levels != 16 || n < 0 || !w || !enc || !gW || !grad_table || !err ||
      (!rows != !n_rows)) {
    set_error("vr_field_bwd_tc: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  return launch_bwd<true>(w, enc, rays, stride, rid, n, dsr, sig, gW, nullptr, err, g, t0, t1,
                          grad_table, ws, ws_bytes, pos, rows, n_rows, stream);
}
