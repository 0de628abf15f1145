// K3 — per-region density + colour MLP (Instant-NGP layout; no reference
// code, restated in oracle/hashmlp_oracle.py).  CUDA-core implementation: one thread
// per sample, 128-sample tiles, fp16 quantisation points identical to the tensor-core
// path (weights fp16; enc, hidden activations, geo features and SH stored as fp16;
// fp32 accumulation).
//
//   density:  h1d = relu(W1d enc)            32 -> 64
//             od  = W2d h1d                  64 -> 16,  sigma = exp(clamp(od0, -15, 15))
//   colour:   cin = [fp16(od[0:16]), SH4(d)] 32
//             h1c = relu(W1c cin)            32 -> 64
//             h2c = relu(W2c h1c)            64 -> 64
//             rgb = sigmoid(W3c h2c)         64 -> 3
// dsigma/d od0 = sigma (trunc-exp convention, zero outside the clamp range).
#include "common.cuh"

namespace vr {

constexpr int MLP_TILE = 128;

__device__ __forceinline__ float q16(float x) { return __half2float(__float2half_rn(x)); }

// Real spherical harmonics up to degree 3 (16 coefficients), tiny-cuda-nn ordering.
__device__ __forceinline__ void sh16(float x, float y, float z, float* o) {
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

struct MlpSmemW {
  float w[VR_MLP_NPARAMS];
};

__device__ __forceinline__ void load_weights(const __half* __restrict__ wg, float* ws) {
  for (int i = threadIdx.x; i < VR_MLP_NPARAMS; i += blockDim.x) ws[i] = __half2float(wg[i]);
}

template <int OUT, int IN>
__device__ __forceinline__ void matvec(const float* __restrict__ W, const float* x, float* y) {
#pragma unroll 4
  for (int j = 0; j < OUT; ++j) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < IN; ++k) acc += W[j * IN + k] * x[k];
    y[j] = acc;
  }
}

struct FwdAct {
  float sigma, od0, rgb[3];
};

// Forward for one sample; optionally records the fp16-rounded activations into
// row-per-thread shared arrays (for the backward tile GEMMs).
template <bool RECORD>
__device__ __forceinline__ FwdAct mlp_forward_one(const float* __restrict__ ws,
                                                  const __half2* __restrict__ enc, int64_t n,
                                                  int64_t i, float dx, float dy, float dz,
                                                  __half* s_enc, __half* s_h1d, __half* s_cin,
                                                  __half* s_h1c, __half* s_h2c) {
  float x[32];
#pragma unroll
  for (int l = 0; l < 16; ++l) {
    const float2 v = __half22float2(enc[(int64_t)l * n + i]);
    x[2 * l] = v.x;
    x[2 * l + 1] = v.y;
  }
  float h[64];
  matvec<64, 32>(ws + VR_MLP_W1D, x, h);
#pragma unroll
  for (int j = 0; j < 64; ++j) h[j] = q16(fmaxf(h[j], 0.f));
  float od[16];
  matvec<16, 64>(ws + VR_MLP_W2D, h, od);
  if (RECORD) {
#pragma unroll
    for (int k = 0; k < 32; ++k) s_enc[k] = __float2half_rn(x[k]);
#pragma unroll
    for (int k = 0; k < 64; ++k) s_h1d[k] = __float2half_rn(h[k]);
  }
  FwdAct a;
  a.od0 = od[0];
  a.sigma = expf(fminf(fmaxf(od[0], -15.f), 15.f));
  float cin[32];
#pragma unroll
  for (int k = 0; k < 16; ++k) cin[k] = q16(od[k]);
  float sh[16];
  sh16(dx, dy, dz, sh);
#pragma unroll
  for (int k = 0; k < 16; ++k) cin[16 + k] = q16(sh[k]);
  matvec<64, 32>(ws + VR_MLP_W1C, cin, h);
#pragma unroll
  for (int j = 0; j < 64; ++j) h[j] = q16(fmaxf(h[j], 0.f));
  if (RECORD) {
#pragma unroll
    for (int k = 0; k < 32; ++k) s_cin[k] = __float2half_rn(cin[k]);
#pragma unroll
    for (int k = 0; k < 64; ++k) s_h1c[k] = __float2half_rn(h[k]);
  }
  float h2[64];
  matvec<64, 64>(ws + VR_MLP_W2C, h, h2);
#pragma unroll
  for (int j = 0; j < 64; ++j) h2[j] = q16(fmaxf(h2[j], 0.f));
  float oc[3];
  matvec<3, 64>(ws + VR_MLP_W3C, h2, oc);
#pragma unroll
  for (int c = 0; c < 3; ++c) a.rgb[c] = 1.f / (1.f + expf(-oc[c]));
  if (RECORD) {
#pragma unroll
    for (int k = 0; k < 64; ++k) s_h2c[k] = __float2half_rn(h2[k]);
  }
  return a;
}

__device__ __forceinline__ void ray_dir(const double* __restrict__ rays, int64_t stride, int64_t r,
                                        float& dx, float& dy, float& dz) {
  dx = (float)__ldg(rays + 3 * stride + r);
  dy = (float)__ldg(rays + 4 * stride + r);
  dz = (float)__ldg(rays + 5 * stride + r);
}

__global__ void __launch_bounds__(MLP_TILE)
    k_mlp_fwd(const __half* __restrict__ wg, const __half2* __restrict__ enc,
              const double* __restrict__ rays, int64_t stride, const int32_t* __restrict__ rid,
              int64_t n, float4* __restrict__ out) {
  __shared__ MlpSmemW sw;
  load_weights(wg, sw.w);
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float dx, dy, dz;
    ray_dir(rays, stride, rid[i], dx, dy, dz);
    const FwdAct a = mlp_forward_one<false>(sw.w, enc, n, i, dx, dy, dz, nullptr, nullptr,
                                            nullptr, nullptr, nullptr);
    out[i] = make_float4(a.sigma, a.rgb[0], a.rgb[1], a.rgb[2]);
  }
}

// Row strides padded to odd 32-bit word counts so row-per-thread accesses are
// bank-conflict free: fp16 rows of 32/64 values -> 34/66 halves, fp32 rows 65/17.
constexpr int H32 = 34, H64 = 66, S64 = 65, S16 = 17;

struct MlpBwdSmem {
  float w[VR_MLP_NPARAMS];
  __half enc[MLP_TILE * H32];
  __half h1d[MLP_TILE * H64];
  __half cin[MLP_TILE * H32];
  __half h1c[MLP_TILE * H64];
  __half h2c[MLP_TILE * H64];
  float d_o[MLP_TILE * 4];
  float b1[MLP_TILE * S64];
  float b2[MLP_TILE * S64];
  float b3[MLP_TILE * S16];
};

// dW[j][k] += sum_s dH[s][j] X[s][k] over the valid rows of the tile
template <int OUT, int IN, int SD, int SX>
__device__ __forceinline__ void tile_wgrad(const float* dH, const __half* X, int rows,
                                           float* __restrict__ gW) {
  for (int o = threadIdx.x; o < OUT * IN; o += blockDim.x) {
    const int j = o / IN, k = o % IN;
    float acc = 0.f;
    for (int s = 0; s < rows; ++s) acc += dH[s * SD + j] * __half2float(X[s * SX + k]);
    if (acc != 0.f) atomicAdd(gW + o, acc);
  }
}

__global__ void __launch_bounds__(MLP_TILE)
    k_mlp_bwd(const __half* __restrict__ wg, const __half2* __restrict__ enc,
              const double* __restrict__ rays, int64_t stride, const int32_t* __restrict__ rid,
              int64_t n, const float4* __restrict__ dsr, float* __restrict__ gW,
              float2* __restrict__ denc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MlpBwdSmem& sm = *reinterpret_cast<MlpBwdSmem*>(smem_raw);
  load_weights(wg, sm.w);
  __syncthreads();
  const int t = threadIdx.x;
  const float* W1d = sm.w + VR_MLP_W1D;
  const float* W2d = sm.w + VR_MLP_W2D;
  const float* W1c = sm.w + VR_MLP_W1C;
  const float* W2c = sm.w + VR_MLP_W2C;
  const float* W3c = sm.w + VR_MLP_W3C;
  for (int64_t base = (int64_t)blockIdx.x * MLP_TILE; base < n;
       base += (int64_t)gridDim.x * MLP_TILE) {
    const int rows = (int)min((int64_t)MLP_TILE, n - base);
    const int64_t i = base + t;
    const bool act = t < rows;
    FwdAct a = {0.f, 0.f, {0.f, 0.f, 0.f}};
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) {
      float dx, dy, dz;
      ray_dir(rays, stride, rid[i], dx, dy, dz);
      a = mlp_forward_one<true>(sm.w, enc, n, i, dx, dy, dz, sm.enc + t * H32,
                                sm.h1d + t * H64, sm.cin + t * H32, sm.h1c + t * H64,
                                sm.h2c + t * H64);
      g = dsr[i];
      // colour head: d(out) = drgb * rgb (1 - rgb)
      sm.d_o[t * 4 + 0] = g.y * a.rgb[0] * (1.f - a.rgb[0]);
      sm.d_o[t * 4 + 1] = g.z * a.rgb[1] * (1.f - a.rgb[1]);
      sm.d_o[t * 4 + 2] = g.w * a.rgb[2] * (1.f - a.rgb[2]);
      // dh2c = W3c^T d_o * relu'(h2c)   -> b1
      const float* d_o = sm.d_o + t * 4;
      const __half* h2 = sm.h2c + t * H64;
      float* dh2 = sm.b1 + t * S64;
#pragma unroll 4
      for (int k = 0; k < 64; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc += W3c[c * 64 + k] * d_o[c];
        dh2[k] = __half2float(h2[k]) > 0.f ? acc : 0.f;
      }
    }
    __syncthreads();
    tile_wgrad<3, 64, 4, H64>(sm.d_o, sm.h2c, rows, gW + VR_MLP_W3C);
    tile_wgrad<64, 64, S64, H64>(sm.b1, sm.h1c, rows, gW + VR_MLP_W2C);
    if (act) {
      // dh1c = W2c^T dh2c * relu'(h1c)   -> b2
      const float* dh2 = sm.b1 + t * S64;
      const __half* h1 = sm.h1c + t * H64;
      float* dh1 = sm.b2 + t * S64;
#pragma unroll 4
      for (int k = 0; k < 64; ++k) {
        float acc = 0.f;
        for (int j = 0; j < 64; ++j) acc += W2c[j * 64 + k] * dh2[j];
        dh1[k] = __half2float(h1[k]) > 0.f ? acc : 0.f;
      }
      // d od = (W1c^T dh1c)[0:16] (+ dsigma * sigma on od0)   -> b3
      float* dod = sm.b3 + t * S16;
#pragma unroll 4
      for (int k = 0; k < 16; ++k) {
        float acc = 0.f;
        for (int j = 0; j < 64; ++j) acc += W1c[j * 32 + k] * dh1[j];
        dod[k] = acc;
      }
      if (a.od0 > -15.f && a.od0 < 15.f) dod[0] += g.x * a.sigma;
    }
    __syncthreads();
    tile_wgrad<64, 32, S64, H32>(sm.b2, sm.cin, rows, gW + VR_MLP_W1C);
    tile_wgrad<16, 64, S16, H64>(sm.b3, sm.h1d, rows, gW + VR_MLP_W2D);
    __syncthreads();
    if (act) {
      // dh1d = W2d^T dod * relu'(h1d)   -> b1 ; denc = W1d^T dh1d
      const float* dod = sm.b3 + t * S16;
      const __half* hd = sm.h1d + t * H64;
      float* dhd = sm.b1 + t * S64;
#pragma unroll 4
      for (int k = 0; k < 64; ++k) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += W2d[j * 64 + k] * dod[j];
        dhd[k] = __half2float(hd[k]) > 0.f ? acc : 0.f;
      }
#pragma unroll 1
      for (int l = 0; l < 16; ++l) {
        float acc0 = 0.f, acc1 = 0.f;
        for (int j = 0; j < 64; ++j) {
          acc0 += W1d[j * 32 + 2 * l] * dhd[j];
          acc1 += W1d[j * 32 + 2 * l + 1] * dhd[j];
        }
        denc[(int64_t)l * n + i] = make_float2(acc0, acc1);
      }
    }
    __syncthreads();
    tile_wgrad<64, 32, S64, H32>(sm.b1, sm.enc, rows, gW + VR_MLP_W1D);
    __syncthreads();
  }
}

}  // namespace vr

using namespace vr;

extern "C" int vr_mlp_fwd(const void* w, const void* enc, const double* rays, int64_t stride,
                          const int32_t* rid, int64_t n, float* out, void* stream) {
  if (n < 0 || !w) {
    set_error("vr_mlp_fwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_mlp_fwd<<<grid_for(n, MLP_TILE, 8), MLP_TILE, 0, (cudaStream_t)stream>>>(
      (const __half*)w, (const __half2*)enc, rays, stride, rid, n, reinterpret_cast<float4*>(out));
  return check_launch("vr_mlp_fwd");
}

extern "C" int vr_mlp_bwd(const void* w, const void* enc, const double* rays, int64_t stride,
                          const int32_t* rid, int64_t n, const float* dsr, float* gW, float* denc,
                          void* stream) {
  if (n < 0 || !w || !gW || !denc) {
    set_error("vr_mlp_bwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  const int smem = (int)sizeof(MlpBwdSmem);
  if (cudaFuncSetAttribute(k_mlp_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
      cudaSuccess) {
    set_error("vr_mlp_bwd: cannot raise shared memory limit");
    return VR_ERR_CUDA;
  }
  k_mlp_bwd<<<grid_for(n, MLP_TILE, 1), MLP_TILE, smem, (cudaStream_t)stream>>>(
      (const __half*)w, (const __half2*)enc, rays, stride, rid, n,
      reinterpret_cast<const float4*>(dsr), gW, reinterpret_cast<float2*>(denc));
  return check_launch("vr_mlp_bwd");
}
