// K3 on the 5th-generation tensor cores: the per-region density + colour MLP as
// tcgen05.mma (kind::f16, fp32 accumulation in TMEM), one elected thread issuing,
// operands in shared memory (layout in tc.cuh), results read back with tcgen05.ld.
//
// Semantics are identical to the CUDA-core reference kernels in mlp.cu (same fp16
// quantisation points, fp32 accumulation): one 128-sample tile is M = 128 and each
// thread owns one sample row for the epilogues.
//
// Forward, per tile (TMEM: 128 columns):
//   P <- enc                                  [128 x 32]
//   D0[0:64)   = P  . W1d^T   -> relu -> Q    [128 x 64]
//   D0[64:80)  = Q  . W2d^T   -> sigma, geo ; P <- [geo | SH(d)]
//   D0[0:64)   = P  . W1c^T   -> relu -> Q
//   D0[64:128) = Q  . W2c^T   -> relu -> P
//   D0[0:16)   = P  . W3c^T   -> sigmoid -> rgb
//
// Backward, per tile (TMEM: 256 columns; weight-gradient accumulators live in TMEM
// for the CTA's whole persistent loop and are flushed once at the end):
//   recompute the forward keeping X0=enc, X1=h1d, X2=cin, X3=h1c, X4=h2c in smem;
//   for each layer the upstream gradient G (fp32 in registers) is written to smem as
//   an fp16 hi part and then an fp16 lo part (G = hi + lo to ~22 bits), each pass
//   issuing  dW += G^T X  (M = 64, both operands MN-major, K = 128 samples)  and
//            dX  = G . W  (M = 128, A K-major, B = W read MN-major).
//   Activations and weights are exactly fp16 by definition of the model, so the
//   backward is accurate to fp32 accumulation.  Gradients with |g| >= 65504 cannot be
//   represented and raise VR_FLAG_OVERFLOW (no silent saturation).
#include "common.cuh"
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

__device__ __forceinline__ void stage_weights(const __half* __restrict__ W, uint8_t* s) {
  stage_one(W + VR_MLP_W1D, s + OW1D, 64, 32);
  stage_one(W + VR_MLP_W2D, s + OW2D, 16, 64);
  stage_one(W + VR_MLP_W1C, s + OW1C, 64, 32);
  stage_one(W + VR_MLP_W2C, s + OW2C, 64, 64);
  stage_one(W + VR_MLP_W3C, s + OW3C, 16, 64);
}

// D[128 x N] (+)= A[128 x K] . B^T,  A = activation tile (K-major), B = weight tile
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

// Acc[M=64 x N] += A^T . B over the 128 samples: A tile [128 x 64] (cols = M),
// B tile [128 x N] (cols = N), both MN-major with K = rows.
__device__ __forceinline__ void issue_wgrad(uint32_t a, uint32_t b, int N, uint32_t d,
                                            bool accumulate) {
  const uint32_t id = idesc_f16(64, N, 1, 1);
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

// write 16 fp32 values (cols c0..c0+15 of row r) as fp16 into a tile
__device__ __forceinline__ void put16(uint8_t* tile, int r, int c0, const float* v) {
  __align__(16) __half h[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) h[j] = __float2half_rn(v[j]);
  st_row8(tile, TILE, r, c0 / 8, h);
  st_row8(tile, TILE, r, c0 / 8 + 1, h + 8);
}
__device__ __forceinline__ void get16(const uint8_t* tile, int r, int c0, float* v) {
  __align__(16) __half h[16];
  ld_row8(tile, TILE, r, c0 / 8, h);
  ld_row8(tile, TILE, r, c0 / 8 + 1, h + 8);
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __half2float(h[j]);
}

// stage the 32 encoding features of row r (sample i, or zeros)
__device__ __forceinline__ void stage_enc(uint8_t* tile, int r, const __half2* __restrict__ enc,
                                          int64_t n, int64_t i, bool valid) {
  __align__(16) __half2 h[16];
#pragma unroll
  for (int l = 0; l < 16; ++l) h[l] = valid ? enc[(int64_t)l * n + i] : __floats2half2_rn(0.f, 0.f);
  const __half* hh = reinterpret_cast<const __half*>(h);
#pragma unroll
  for (int cb = 0; cb < 4; ++cb) st_row8(tile, TILE, r, cb, hh + 8 * cb);
}

// one MMA round: make this thread's smem writes visible to the tensor core, issue,
// wait for completion
template <class F>
__device__ __forceinline__ void mma_round(uint64_t* bar, uint32_t& phase, F issue) {
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_fence_after();
    issue();
    mma_commit(bar);
  }
  mbar_wait(bar, phase);
  phase ^= 1u;
  __syncwarp();
  tc_fence_after();
}

struct FwdRow {
  float sigma, od0, rgb[3];
};

// The forward chain for one tile.  Activation tiles: X0 (enc, pre-staged), X1, X2, X3,
// X4 (may alias: the forward-only kernel ping-pongs two buffers).  d0/d1 = TMEM
// column bases of two scratch accumulators (64 and 16+ columns).
__device__ __forceinline__ FwdRow forward_tile(uint8_t* sw, uint8_t* X0, uint8_t* X1, uint8_t* X2,
                                               uint8_t* X3, uint8_t* X4, uint32_t tm_row,
                                               uint32_t tmem, uint32_t d0, uint32_t d1,
                                               uint64_t* bar, uint32_t& phase, float dx,
                                               float dy, float dz) {
  const int r = threadIdx.x;
  const uint32_t sW = smem_u32(sw);
  float v[16];
  // L1d
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X0), 32, sW + OW1D, 64, tmem + d0); });
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    tmem_ld16(tm_row + d0 + c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.f);
    put16(X1, r, c, v);
  }
  // L2d
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X1), 64, sW + OW2D, 16, tmem + d1); });
  FwdRow out;
  tmem_ld16(tm_row + d1, v);
  out.od0 = v[0];
  out.sigma = expf(fminf(fmaxf(v[0], -15.f), 15.f));
  put16(X2, r, 0, v);
  sh16f(dx, dy, dz, v);
  put16(X2, r, 16, v);
  // L1c
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X2), 32, sW + OW1C, 64, tmem + d0); });
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    tmem_ld16(tm_row + d0 + c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.f);
    put16(X3, r, c, v);
  }
  // L2c
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X3), 64, sW + OW2C, 64, tmem + d0); });
#pragma unroll
  for (int c = 0; c < 64; c += 16) {
    tmem_ld16(tm_row + d0 + c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = fmaxf(v[j], 0.f);
    put16(X4, r, c, v);
  }
  // L3c
  mma_round(bar, phase, [&] { issue_fwd(smem_u32(X4), 64, sW + OW3C, 16, tmem + d1); });
  tmem_ld16(tm_row + d1, v);
#pragma unroll
  for (int c = 0; c < 3; ++c) out.rgb[c] = 1.f / (1.f + expf(-v[c]));
  return out;
}

__device__ __forceinline__ void load_dir(const double* __restrict__ rays, int64_t stride,
                                         const int32_t* __restrict__ rid, int64_t i, bool valid,
                                         float& dx, float& dy, float& dz) {
  dx = dy = dz = 0.f;
  if (valid) {
    const int64_t r = rid[i];
    dx = (float)__ldg(rays + 3 * stride + r);
    dy = (float)__ldg(rays + 4 * stride + r);
    dz = (float)__ldg(rays + 5 * stride + r);
  }
}

// ---- forward kernel ---------------------------------------------------------------------
constexpr uint32_t F_P = WBYTES, F_Q = F_P + TILE * 64 * 2, F_BAR = F_Q + TILE * 64 * 2,
                   F_SMEM = F_BAR + 16;

__global__ void __launch_bounds__(TILE, 4)
    k_mlp_fwd_tc(const __half* __restrict__ W, const __half2* __restrict__ enc,
                 const double* __restrict__ rays, int64_t stride, const int32_t* __restrict__ rid,
                 int64_t n, float4* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sw = smem;
  uint8_t* P = smem + F_P;
  uint8_t* Q = smem + F_Q;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + F_BAR);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + F_BAR + 8);
  const int warp = threadIdx.x >> 5;
  stage_weights(W, sw);
  if (warp == 0) tmem_alloc(slot, 128);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t tm_row = tmem + ((uint32_t)(warp * 32) << 16);
  uint32_t phase = 0;
  const int64_t n_tiles = ceil_div(n, TILE);
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t i = tile * TILE + threadIdx.x;
    const bool valid = i < n;
    stage_enc(P, threadIdx.x, enc, n, i, valid);
    float dx, dy, dz;
    load_dir(rays, stride, rid, i, valid, dx, dy, dz);
    // P(enc) -> Q(h1d) -> P(cin) -> Q(h1c) -> P(h2c)
    const FwdRow f = forward_tile(sw, P, Q, P, Q, P, tm_row, tmem, 0, 64, bar, phase, dx, dy, dz);
    if (valid) out[i] = make_float4(f.sigma, f.rgb[0], f.rgb[1], f.rgb[2]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

// ---- backward kernel --------------------------------------------------------------------
constexpr uint32_t B_X0 = WBYTES, B_X1 = B_X0 + TILE * 32 * 2, B_X2 = B_X1 + TILE * 64 * 2,
                   B_X3 = B_X2 + TILE * 32 * 2, B_X4 = B_X3 + TILE * 64 * 2,
                   B_G = B_X4 + TILE * 64 * 2, B_BAR = B_G + TILE * 64 * 2, B_SMEM = B_BAR + 16;
// TMEM columns: weight-gradient accumulators (M = 64) then scratch
constexpr uint32_t T_W1D = 0, T_W2DT = 32, T_W1C = 48, T_W2C = 80, T_W3CT = 144, T_D0 = 160,
                   T_D1 = 224, T_COLS = 256;

// write the hi or lo fp16 part of a gradient row (width multiple of 16) into G
template <int WIDTH>
__device__ __forceinline__ void put_grad(uint8_t* G, int r, const float* g, bool lo, int& flags) {
#pragma unroll
  for (int c = 0; c < WIDTH; c += 16) {
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float x = g[c + j];
      const float hi = __half2float(__float2half_rn(x));
      if (!lo && !(fabsf(x) < 65504.f)) flags |= VR_FLAG_OVERFLOW;
      v[j] = lo ? (x - hi) : hi;
    }
    put16(G, r, c, v);
  }
}

__global__ void __launch_bounds__(TILE, 2)
    k_mlp_bwd_tc(const __half* __restrict__ W, const __half2* __restrict__ enc,
                 const double* __restrict__ rays, int64_t stride, const int32_t* __restrict__ rid,
                 int64_t n, const float4* __restrict__ dsr, float* __restrict__ gW,
                 float2* __restrict__ denc, int32_t* err) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sw = smem;
  uint8_t* X0 = smem + B_X0;
  uint8_t* X1 = smem + B_X1;
  uint8_t* X2 = smem + B_X2;
  uint8_t* X3 = smem + B_X3;
  uint8_t* X4 = smem + B_X4;
  uint8_t* G = smem + B_G;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + B_BAR);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + B_BAR + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = threadIdx.x;
  stage_weights(W, sw);
  if (warp == 0) tmem_alloc(slot, T_COLS);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t tm_row = tmem + ((uint32_t)(warp * 32) << 16);
  const uint32_t sW = smem_u32(sw);
  const uint32_t sX0 = smem_u32(X0), sX1 = smem_u32(X1), sX2 = smem_u32(X2),
                 sX3 = smem_u32(X3), sX4 = smem_u32(X4), sG = smem_u32(G);
  uint32_t phase = 0;
  int flags = 0;
  bool acc = false;  // weight-gradient accumulators hold data
  const int64_t n_tiles = ceil_div(n, TILE);
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t i = tile * TILE + r;
    const bool valid = i < n;
    stage_enc(X0, r, enc, n, i, valid);
    float dx, dy, dz;
    load_dir(rays, stride, rid, i, valid, dx, dy, dz);
    const FwdRow f =
        forward_tile(sw, X0, X1, X2, X3, X4, tm_row, tmem, T_D0, T_D1, bar, phase, dx, dy, dz);
    const float4 gin = valid ? dsr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float g[64];
    float v[16];

    // ---- colour head: g_o = drgb * rgb (1 - rgb), padded to 16 ----------------------
#pragma unroll
    for (int j = 0; j < 16; ++j) g[j] = 0.f;
    g[0] = gin.y * f.rgb[0] * (1.f - f.rgb[0]);
    g[1] = gin.z * f.rgb[1] * (1.f - f.rgb[1]);
    g[2] = gin.w * f.rgb[2] * (1.f - f.rgb[2]);
    for (int pass = 0; pass < 2; ++pass) {
      put_grad<16>(G, r, g, pass == 1, flags);
      const bool a_w = acc || pass == 1;
      mma_round(bar, phase, [&] {
        issue_wgrad(sX4, sG, 16, tmem + T_W3CT, a_w);            // dW3c^T += h2c^T g_o
        issue_dgrad(sG, 16, sW + OW3C, 64, tmem + T_D0, pass == 1);  // g_o . W3c
      });
    }
    // dh2c = (g_o . W3c) * relu'(h2c)
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      tmem_ld16(tm_row + T_D0 + c, v);
      float h[16];
      get16(X4, r, c, h);
#pragma unroll
      for (int j = 0; j < 16; ++j) g[c + j] = h[j] > 0.f ? v[j] : 0.f;
    }
    for (int pass = 0; pass < 2; ++pass) {
      put_grad<64>(G, r, g, pass == 1, flags);
      const bool a_w = acc || pass == 1;
      mma_round(bar, phase, [&] {
        issue_wgrad(sG, sX3, 64, tmem + T_W2C, a_w);             // dW2c += dh2c^T h1c
        issue_dgrad(sG, 64, sW + OW2C, 64, tmem + T_D0, pass == 1);  // dh2c . W2c
      });
    }
    // dh1c = (dh2c . W2c) * relu'(h1c)
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      tmem_ld16(tm_row + T_D0 + c, v);
      float h[16];
      get16(X3, r, c, h);
#pragma unroll
      for (int j = 0; j < 16; ++j) g[c + j] = h[j] > 0.f ? v[j] : 0.f;
    }
    for (int pass = 0; pass < 2; ++pass) {
      put_grad<64>(G, r, g, pass == 1, flags);
      const bool a_w = acc || pass == 1;
      mma_round(bar, phase, [&] {
        issue_wgrad(sG, sX2, 32, tmem + T_W1C, a_w);             // dW1c += dh1c^T cin
        issue_dgrad(sG, 64, sW + OW1C, 32, tmem + T_D0, pass == 1);  // dh1c . W1c
      });
    }
    // d od = dcin[0:16]; + dsigma * sigma on od0 (trunc-exp inside the clamp range)
    tmem_ld16(tm_row + T_D0, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) g[j] = v[j];
    if (f.od0 > -15.f && f.od0 < 15.f) g[0] += gin.x * f.sigma;
    for (int pass = 0; pass < 2; ++pass) {
      put_grad<16>(G, r, g, pass == 1, flags);
      const bool a_w = acc || pass == 1;
      mma_round(bar, phase, [&] {
        issue_wgrad(sX1, sG, 16, tmem + T_W2DT, a_w);            // dW2d^T += h1d^T dod
        issue_dgrad(sG, 16, sW + OW2D, 64, tmem + T_D0, pass == 1);  // dod . W2d
      });
    }
    // dh1d = (dod . W2d) * relu'(h1d)
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      tmem_ld16(tm_row + T_D0 + c, v);
      float h[16];
      get16(X1, r, c, h);
#pragma unroll
      for (int j = 0; j < 16; ++j) g[c + j] = h[j] > 0.f ? v[j] : 0.f;
    }
    for (int pass = 0; pass < 2; ++pass) {
      put_grad<64>(G, r, g, pass == 1, flags);
      const bool a_w = acc || pass == 1;
      mma_round(bar, phase, [&] {
        issue_wgrad(sG, sX0, 32, tmem + T_W1D, a_w);             // dW1d += dh1d^T enc
        issue_dgrad(sG, 64, sW + OW1D, 32, tmem + T_D0, pass == 1);  // denc = dh1d . W1d
      });
    }
    // denc -> global, level-major float2
#pragma unroll
    for (int c = 0; c < 32; c += 16) {
      tmem_ld16(tm_row + T_D0 + c, v);
      if (valid) {
#pragma unroll
        for (int j = 0; j < 16; j += 2)
          denc[(int64_t)((c + j) / 2) * n + i] = make_float2(v[j], v[j + 1]);
      }
    }
    acc = true;
  }
  // ---- flush the weight-gradient accumulators (M = 64: rows 16w+t at lanes 32w+t) ------
  if (acc) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int m = warp * 16 + lane;  // valid for lane < 16
    float v[16];
#pragma unroll
    for (int c = 0; c < 32; c += 16) {
      tmem_ld16(tm_row + T_W1D + c, v);
      if (lane < 16)
        for (int j = 0; j < 16; ++j) atomicAdd(gW + VR_MLP_W1D + m * 32 + c + j, v[j]);
    }
    tmem_ld16(tm_row + T_W2DT, v);
    if (lane < 16)
      for (int j = 0; j < 16; ++j) atomicAdd(gW + VR_MLP_W2D + j * 64 + m, v[j]);
#pragma unroll
    for (int c = 0; c < 32; c += 16) {
      tmem_ld16(tm_row + T_W1C + c, v);
      if (lane < 16)
        for (int j = 0; j < 16; ++j) atomicAdd(gW + VR_MLP_W1C + m * 32 + c + j, v[j]);
    }
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      tmem_ld16(tm_row + T_W2C + c, v);
      if (lane < 16)
        for (int j = 0; j < 16; ++j) atomicAdd(gW + VR_MLP_W2C + m * 64 + c + j, v[j]);
    }
    tmem_ld16(tm_row + T_W3CT, v);
    if (lane < 16)
      for (int j = 0; j < 3; ++j) atomicAdd(gW + VR_MLP_W3C + j * 64 + m, v[j]);
  }
  flags = (int)__reduce_or_sync(0xffffffffu, (unsigned)flags);
  if (flags && lane == 0) atomicOr(err, flags);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, T_COLS);
  }
}

}  // namespace mlp
}  // namespace vr

using namespace vr;

static int mlp_grid(int64_t n, int per_sm) {
  const int64_t tiles = ceil_div(n, vr::mlp::TILE);
  int64_t g = (int64_t)VR_NUM_SMS * per_sm;
  return (int)(tiles < g ? tiles : g);
}

extern "C" int vr_mlp_fwd_tc(const void* w, const void* enc, const double* rays, int64_t stride,
                             const int32_t* rid, int64_t n, float* out, void* stream) {
  if (n < 0 || !w) {
    set_error("vr_mlp_fwd_tc: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(mlp::k_mlp_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mlp::F_SMEM) != cudaSuccess) {
      set_error("vr_mlp_fwd_tc: smem attribute");
      return VR_ERR_CUDA;
    }
    attr = true;
  }
  mlp::k_mlp_fwd_tc<<<mlp_grid(n, 4), mlp::TILE, mlp::F_SMEM, (cudaStream_t)stream>>>(
      (const __half*)w, (const __half2*)enc, rays, stride, rid, n, reinterpret_cast<float4*>(out));
  return check_launch("vr_mlp_fwd_tc");
}

extern "C" int vr_mlp_bwd_tc(const void* w, const void* enc, const double* rays, int64_t stride,
                             const int32_t* rid, int64_t n, const float* dsr, float* gW,
                             float* denc, int32_t* err, void* stream) {
  if (n < 0 || !w || !gW || !denc || !err) {
    set_error("vr_mlp_bwd_tc: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(mlp::k_mlp_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)mlp::B_SMEM) != cudaSuccess) {
      set_error("vr_mlp_bwd_tc: smem attribute");
      return VR_ERR_CUDA;
    }
    attr = true;
  }
  mlp::k_mlp_bwd_tc<<<mlp_grid(n, 2), mlp::TILE, mlp::B_SMEM, (cudaStream_t)stream>>>(
      (const __half*)w, (const __half2*)enc, rays, stride, rid, n,
      reinterpret_cast<const float4*>(dsr), gW, reinterpret_cast<float2*>(denc), err);
  return check_launch("vr_mlp_bwd_tc");
}
