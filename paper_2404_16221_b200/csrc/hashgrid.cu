// K2 — per-region multiresolution hash-grid encoding (Instant-NGP).
//
// There is no reference implementation; the spec below is
// restated bit-for-bit in oracle/hashmlp_oracle.py:
//   u   = float32((p - box_mn) / (box_mx - box_mn))          float64 ops, one cast
//   pos = u * scale_l + 0.5f        (two float32 roundings, no FMA)
//   g   = clamp(floor(pos), 0, res_l - 2),  f = pos - g
//   corner c = (cx, cy, cz):  idx = dense_l ? x + res*(y + res*z)
//                                           : (x ^ y*2654435761 ^ z*805459861) & (T-1)
//   w_c = (wx * wy) * wz,  feat_l = sum_c w_c * table[offset_l + idx_c]   (F = 2,
//   float32, corner order c = 0..7, no FMA)
// Encodings are written level-major enc[l][n] as half2 so both the gather kernel
// and the MLP read them coalesced.  The backward scatters w_c * dfeat with vector
// float2 atomics (red.global.add.v2.f32 on sm_90+).
#include "common.cuh"

namespace vr {

constexpr int HASH_THREADS = 256;

__device__ __forceinline__ void norm_pos(const VrHashGridDesc& g, const double* __restrict__ rays,
                                         int64_t stride, const double* __restrict__ t0,
                                         const double* __restrict__ t1,
                                         const int32_t* __restrict__ rid, int64_t i, float u[3]) {
  double p[3];
  const int64_t r = rid[i];
  const double m = sample_mid(t0[i], t1[i]);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    p[a] = dadd(__ldg(rays + a * stride + r), dmul(m, __ldg(rays + (3 + a) * stride + r)));
    u[a] = (float)ddiv(dsub(p[a], g.box_mn[a]), dsub(g.box_mx[a], g.box_mn[a]));
  }
}

struct Corners {
  uint32_t idx[8];
  float w[8];
};

__device__ __forceinline__ void level_corners(const VrHashGridDesc& g, int l, const float u[3],
                                              Corners& c) {
  const float scale = g.scale[l];
  const int res = g.res[l];
  int gi[3];
  float fr[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float pos = __fadd_rn(__fmul_rn(u[a], scale), 0.5f);
    float fl = floorf(pos);
    int gg = (int)fl;
    gg = min(max(gg, 0), res - 2);
    gi[a] = gg;
    fr[a] = __fsub_rn(pos, (float)gg);
  }
  const uint32_t mask = (1u << g.log2_T) - 1u;
  const bool dense = g.dense[l] != 0;
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) {
    const int cx = c8 & 1, cy = (c8 >> 1) & 1, cz = (c8 >> 2) & 1;
    const uint32_t x = (uint32_t)(gi[0] + cx), y = (uint32_t)(gi[1] + cy),
                   z = (uint32_t)(gi[2] + cz);
    uint32_t idx;
    if (dense) {
      idx = x + (uint32_t)res * (y + (uint32_t)res * z);
    } else {
      idx = (x ^ (y * 2654435761u) ^ (z * 805459861u)) & mask;
    }
    c.idx[c8] = idx;
    const float wx = cx ? fr[0] : __fsub_rn(1.f, fr[0]);
    const float wy = cy ? fr[1] : __fsub_rn(1.f, fr[1]);
    const float wz = cz ? fr[2] : __fsub_rn(1.f, fr[2]);
    c.w[c8] = __fmul_rn(__fmul_rn(wx, wy), wz);
  }
}

__global__ void __launch_bounds__(HASH_THREADS)
    k_hash_fwd(const VrHashGridDesc g, const float2* __restrict__ table,
               const double* __restrict__ rays, int64_t stride, const double* __restrict__ t0,
               const double* __restrict__ t1, const int32_t* __restrict__ rid, int64_t n,
               __half2* __restrict__ enc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float u[3];
    norm_pos(g, rays, stride, t0, t1, rid, i, u);
#pragma unroll 2
    for (int l = 0; l < g.n_levels; ++l) {
      Corners c;
      level_corners(g, l, u, c);
      const float2* tl = table + g.offset[l];
      float2 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(tl + c.idx[k]);
      // explicit round-to-nearest mul/add (no FMA): features are bit-identical to the
      // float32 restatement in oracle/hashmlp_oracle.py
      float a0 = 0.f, a1 = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a0 = __fadd_rn(a0, __fmul_rn(c.w[k], v[k].x));
        a1 = __fadd_rn(a1, __fmul_rn(c.w[k], v[k].y));
      }
      enc[(int64_t)l * n + i] = __floats2half2_rn(a0, a1);
    }
  }
}

__global__ void __launch_bounds__(HASH_THREADS)
    k_hash_bwd(const VrHashGridDesc g, const double* __restrict__ rays, int64_t stride,
               const double* __restrict__ t0, const double* __restrict__ t1,
               const int32_t* __restrict__ rid, int64_t n, const float2* __restrict__ denc,
               float2* __restrict__ grad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float u[3];
    norm_pos(g, rays, stride, t0, t1, rid, i, u);
#pragma unroll 2
    for (int l = 0; l < g.n_levels; ++l) {
      const float2 d = denc[(int64_t)l * n + i];
      if (d.x == 0.f && d.y == 0.f) continue;
      Corners c;
      level_corners(g, l, u, c);
      float2* gl = grad + g.offset[l];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        atomicAdd(gl + c.idx[k], make_float2(c.w[k] * d.x, c.w[k] * d.y));
    }
  }
}

__global__ void k_hash_idx(const VrHashGridDesc g, const double* __restrict__ rays, int64_t stride,
                           const double* __restrict__ t0, const double* __restrict__ t1,
                           const int32_t* __restrict__ rid, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float u[3];
    norm_pos(g, rays, stride, t0, t1, rid, i, u);
    for (int l = 0; l < g.n_levels; ++l) {
      Corners c;
      level_corners(g, l, u, c);
#pragma unroll
      for (int k = 0; k < 8; ++k) out[((int64_t)l * n + i) * 8 + k] = (int32_t)c.idx[k];
    }
  }
}

static bool valid_grid(const VrHashGridDesc* g) {
  if (!g || g->n_levels < 1 || g->n_levels > VR_MAX_LEVELS || g->log2_T < 1 || g->log2_T > 28)
    return false;
  for (int l = 0; l < g->n_levels; ++l)
    if (g->res[l] < 2) return false;
  return true;
}

}  // namespace vr

using namespace vr;

extern "C" int vr_hash_fwd(const VrHashGridDesc* g, const float* table, const double* rays,
                           int64_t stride, const double* t0, const double* t1, const int32_t* rid,
                           int64_t n, void* enc, void* stream) {
  if (!valid_grid(g) || n < 0) {
    set_error("vr_hash_fwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_hash_fwd<<<grid_for(n, HASH_THREADS, 8), HASH_THREADS, 0, (cudaStream_t)stream>>>(
      *g, reinterpret_cast<const float2*>(table), rays, stride, t0, t1, rid, n,
      reinterpret_cast<__half2*>(enc));
  return check_launch("vr_hash_fwd");
}

extern "C" int vr_hash_bwd(const VrHashGridDesc* g, const double* rays, int64_t stride,
                           const double* t0, const double* t1, const int32_t* rid, int64_t n,
                           const float* denc, float* grad, void* stream) {
  if (!valid_grid(g) || n < 0) {
    set_error("vr_hash_bwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_hash_bwd<<<grid_for(n, HASH_THREADS, 8), HASH_THREADS, 0, (cudaStream_t)stream>>>(
      *g, rays, stride, t0, t1, rid, n, reinterpret_cast<const float2*>(denc),
      reinterpret_cast<float2*>(grad));
  return check_launch("vr_hash_bwd");
}

extern "C" int vr_hash_indices(const VrHashGridDesc* g, const double* rays, int64_t stride,
                               const double* t0, const double* t1, const int32_t* rid, int64_t n,
                               int32_t* out, void* stream) {
  if (!valid_grid(g) || n < 0) {
    set_error("vr_hash_indices: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_hash_idx<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*g, rays, stride, t0, t1, rid,
                                                                   n, out);
  return check_launch("vr_hash_indices");
}
