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
#include <string.h>

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
      // x-adjacent corners whose entries differ only in bit 0 share one 16-byte pair
      // (always for even x on hashed levels, even index on dense levels): one float4
      // gather instead of two float2 (level offsets are multiples of 8 entries).
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const uint32_t a = c.idx[k], b = c.idx[k + 1];
        if ((a ^ b) == 1u) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(tl + (a & ~1u)));
          const float2 lo = make_float2(q.x, q.y), hi = make_float2(q.z, q.w);
          v[k] = (a & 1u) ? hi : lo;
          v[k + 1] = (a & 1u) ? lo : hi;
        } else {
          v[k] = __ldg(tl + a);
          v[k + 1] = __ldg(tl + b);
        }
      }
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

// Coarse dense levels (a few thousand entries hit by every sample of the region) are
// contention-bound under global atomics: their gradients go to R private replicas
// (picked per warp) in a workspace and are summed into the table by k_hash_rep_reduce.
struct RepPlan {
  int32_t n_rep;  // levels 0 .. n_rep-1 are replicated
  int32_t R[VR_MAX_LEVELS];
  int64_t off[VR_MAX_LEVELS];  // workspace offset (entries) of level l's replicas
};

__device__ __forceinline__ void scatter_pair(float2* gl, uint32_t a, uint32_t b, float2 ga,
                                             float2 gb) {
  if ((a ^ b) == 1u) {  // one 16-byte vector atomic for the x-adjacent pair
    const float4 q =
        (a & 1u) ? make_float4(gb.x, gb.y, ga.x, ga.y) : make_float4(ga.x, ga.y, gb.x, gb.y);
    atomicAdd(reinterpret_cast<float4*>(gl + (a & ~1u)), q);
  } else {
    atomicAdd(gl + a, ga);
    atomicAdd(gl + b, gb);
  }
}

__global__ void __launch_bounds__(HASH_THREADS)
    k_hash_bwd(const VrHashGridDesc g, const RepPlan plan, const double* __restrict__ rays,
               int64_t stride, const double* __restrict__ t0, const double* __restrict__ t1,
               const int32_t* __restrict__ rid, int64_t n, const float2* __restrict__ denc,
               float2* __restrict__ grad, float2* __restrict__ ws) {
  const int gwarp = blockIdx.x * (HASH_THREADS / 32) + (threadIdx.x >> 5);
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
      const int64_t size_l = g.offset[l + 1] - g.offset[l];
      float2* gl = (l < plan.n_rep) ? ws + plan.off[l] + (int64_t)(gwarp % plan.R[l]) * size_l
                                    : grad + g.offset[l];
#pragma unroll
      for (int k = 0; k < 8; k += 2)
        scatter_pair(gl, c.idx[k], c.idx[k + 1], make_float2(c.w[k] * d.x, c.w[k] * d.y),
                     make_float2(c.w[k + 1] * d.x, c.w[k + 1] * d.y));
    }
  }
}

// grad[level l entry e] += sum_r ws[l][r][e]; the replicas are zeroed for the next use
__global__ void k_hash_rep_reduce(const VrHashGridDesc g, const RepPlan plan,
                                  float2* __restrict__ grad, float2* __restrict__ ws,
                                  int64_t total) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = t;
    int l = 0;
    while (l < plan.n_rep - 1 && e >= g.offset[l + 1] - g.offset[l]) {
      e -= g.offset[l + 1] - g.offset[l];
      ++l;
    }
    const int64_t size_l = g.offset[l + 1] - g.offset[l];
    float2* w = ws + plan.off[l] + e;
    float2 acc = make_float2(0.f, 0.f);
    for (int r = 0; r < plan.R[l]; ++r) {
      const float2 v = w[r * size_l];
      acc.x += v.x;
      acc.y += v.y;
      w[r * size_l] = make_float2(0.f, 0.f);
    }
    float2* gp = grad + g.offset[l] + e;
    gp->x += acc.x;
    gp->y += acc.y;
  }
}

static RepPlan rep_plan(const VrHashGridDesc* g, int64_t* ws_entries, int64_t* red_entries) {
  RepPlan p;
  memset(&p, 0, sizeof(p));
  int64_t off = 0, red = 0;
  for (int l = 0; l < g->n_levels; ++l) {
    const int64_t size_l = g->offset[l + 1] - g->offset[l];
    // measured on c3 (scripts/bench_hash.py): only the coarsest level (17^3 entries) is
    // contention-bound; replicating 24^3 / 32^3 levels costs more than it saves
    if (!g->dense[l] || size_l > 8192) break;
    int R = (int)((int64_t)(1 << 20) / size_l);
    R = R < 1 ? 1 : (R > 64 ? 64 : R);
    p.R[l] = R;
    p.off[l] = off;
    off += (int64_t)R * size_l;
    red += size_l;
    p.n_rep = l + 1;
  }
  *ws_entries = off;
  *red_entries = red;
  return p;
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

extern "C" size_t vr_hash_bwd_workspace_bytes(const VrHashGridDesc* g) {
  if (!valid_grid(g)) return 0;
  int64_t ws = 0, red = 0;
  rep_plan(g, &ws, &red);
  return (size_t)ws * sizeof(float2);
}

extern "C" int vr_hash_bwd(const VrHashGridDesc* g, const double* rays, int64_t stride,
                           const double* t0, const double* t1, const int32_t* rid, int64_t n,
                           const float* denc, float* grad, void* ws, size_t ws_bytes,
                           void* stream) {
  if (!valid_grid(g) || n < 0) {
    set_error("vr_hash_bwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  int64_t ws_entries = 0, red = 0;
  RepPlan plan = rep_plan(g, &ws_entries, &red);
  if (!ws || ws_bytes < (size_t)ws_entries * sizeof(float2)) plan.n_rep = 0;  // plain atomics
  cudaStream_t s = (cudaStream_t)stream;
  k_hash_bwd<<<grid_for(n, HASH_THREADS, 8), HASH_THREADS, 0, s>>>(
      *g, plan, rays, stride, t0, t1, rid, n, reinterpret_cast<const float2*>(denc),
      reinterpret_cast<float2*>(grad), reinterpret_cast<float2*>(ws));
  if (plan.n_rep > 0)
    k_hash_rep_reduce<<<grid_for(red, 256, 4), 256, 0, s>>>(
        *g, plan, reinterpret_cast<float2*>(grad), reinterpret_cast<float2*>(ws), red);
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
