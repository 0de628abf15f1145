// Device building blocks of the multiresolution hash-grid encoding (K2), shared by the
// standalone kernels (hashgrid.cu) and the fused field kernels (mlp_tc.cu).  The
// arithmetic spec is in hashgrid.cu's header and restated in oracle/hashmlp_oracle.py.
#pragma once

#include "common.cuh"

namespace vr {

// u = float32((p - box_mn) / (box_mx - box_mn)) for p = o + m d (float64, no FMA in p).
// The division is exact (correctly rounded) without a division instruction per sample:
// with y = RN(1 / e) (one __drcp_rn per thread, BoxInv) and q0 = RN(a y), the remainder
// r = a - e q0 is exact under an FMA and RN(q0 + r y) is the correctly rounded a / e
// (Markstein's theorem: y within half an ulp of 1/e, q0 within one ulp of a/e; no overflow
// or underflow for positions inside the box's range) — bit-identical to the division, at a
// third of its instructions (the position pass was fp64-division bound).
struct BoxInv {
  double ext[3], inv[3];
};
__device__ __forceinline__ BoxInv box_inv(const VrHashGridDesc& g) {
  BoxInv b;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b.ext[a] = dsub(g.box_mx[a], g.box_mn[a]);
    b.inv[a] = __drcp_rn(b.ext[a]);
  }
  return b;
}
__device__ __forceinline__ double div_exact(double a, double e, double inv) {
  const double q0 = __dmul_rn(a, inv);
  const double r = __fma_rn(-q0, e, a);
  return __fma_rn(r, inv, q0);
}

__device__ __forceinline__ void norm_pos_od(const VrHashGridDesc& g, const BoxInv& bi,
                                            const double o[3], const double d[3], double m,
                                            float u[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double p = dadd(o[a], dmul(m, d[a]));
    u[a] = (float)div_exact(dsub(p, g.box_mn[a]), bi.ext[a], bi.inv[a]);
  }
}

__device__ __forceinline__ void norm_pos(const VrHashGridDesc& g, const BoxInv& bi,
                                         const double* __restrict__ rays,
                                         int64_t stride, const double* __restrict__ t0,
                                         const double* __restrict__ t1,
                                         const int32_t* __restrict__ rid, int64_t i, float u[3]) {
  const int64_t r = checked_ray(rid[i], stride);
  const double m = sample_mid(t0[i], t1[i]);
  double o[3], d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    o[a] = __ldg(rays + a * stride + r);
    d[a] = __ldg(rays + (3 + a) * stride + r);
  }
  norm_pos_od(g, bi, o, d, m, u);
}

struct Corners {
  uint32_t idx[8];
  float w[8];
};

// cell of level l: lower corner gi and fractions fr (two float32 roundings, no FMA)
__device__ __forceinline__ void level_cell(const VrHashGridDesc& g, int l, const float u[3],
                                           int gi[3], float fr[3]) {
  const float scale = g.scale[l];
  const int res = g.res[l];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float pos = __fadd_rn(__fmul_rn(u[a], scale), 0.5f);
    int gg = (int)floorf(pos);
    gg = min(max(gg, 0), res - 2);
    gi[a] = gg;
    fr[a] = __fsub_rn(pos, (float)gg);
  }
}

// table index and trilinear weight of corner c8 = cx + 2 cy + 4 cz
__device__ __forceinline__ void corner(const VrHashGridDesc& g, int l, const int gi[3],
                                       const float fr[3], int c8, uint32_t& idx, float& w) {
  const int res = g.res[l];
  const int cx = c8 & 1, cy = (c8 >> 1) & 1, cz = (c8 >> 2) & 1;
  const uint32_t x = (uint32_t)(gi[0] + cx), y = (uint32_t)(gi[1] + cy),
                 z = (uint32_t)(gi[2] + cz);
  idx = g.dense[l] ? x + (uint32_t)res * (y + (uint32_t)res * z)
                   : (x ^ (y * 2654435761u) ^ (z * 805459861u)) & ((1u << g.log2_T) - 1u);
  const float wx = cx ? fr[0] : __fsub_rn(1.f, fr[0]);
  const float wy = cy ? fr[1] : __fsub_rn(1.f, fr[1]);
  const float wz = cz ? fr[2] : __fsub_rn(1.f, fr[2]);
  w = __fmul_rn(__fmul_rn(wx, wy), wz);
}

__device__ __forceinline__ void level_corners(const VrHashGridDesc& g, int l, const float u[3],
                                              Corners& c) {
  int gi[3];
  float fr[3];
  level_cell(g, l, u, gi, fr);
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) corner(g, l, gi, fr, c8, c.idx[c8], c.w[c8]);
}

// Half of a level's feature: the corners with cx = p (c8 = p, p+2, p+4, p+6), accumulated
// in that order from 0 with round-to-nearest mul/add (no FMA).  feature = half(0) + half(1)
// — the accumulation order every gather implements and oracle/hashmlp_oracle.py restates.
// Lane-pair gathers: lanes 2j and 2j+1 take the two halves of one sample, so the x-adjacent
// corners of a row are read by the same 8-byte load instruction and merge into one L2
// sector request whenever their entries share a 32-byte sector (x mod 4 != 3 on hashed
// levels; measured 2.5x the per-lane rate of 16-byte loads in scripts/micro/gather_bench.cu).
__device__ __forceinline__ float2 gather_half(const VrHashGridDesc& g, int l,
                                              const float2* __restrict__ tl, const float u[3],
                                              int p) {
  int gi[3];
  float fr[3];
  level_cell(g, l, u, gi, fr);
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t idx;
    float w;
    corner(g, l, gi, fr, p + 2 * k, idx, w);
    if (!VR_CHECK((int64_t)idx < g.offset[l + 1] - g.offset[l])) idx = 0;
    const float2 v = __ldg(tl + idx);
    a0 = __fadd_rn(a0, __fmul_rn(w, v.x));
    a1 = __fadd_rn(a1, __fmul_rn(w, v.y));
  }
  return make_float2(a0, a1);
}

// Feature of one level.  x-adjacent corners whose entries differ only in bit 0 share
// one 16-byte pair (always for even x on hashed levels, even index on dense levels):
// one float4 gather instead of two float2 (level offsets are multiples of 8 entries).
// Explicit round-to-nearest mul/add (no FMA): bit-identical to the float32 oracle.
__device__ __forceinline__ float2 gather_level(const float2* __restrict__ tl, const Corners& c) {
  float2 v[8];
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
  // even corners, odd corners, then their sum (the order gather_half pairs implement)
  float e0 = 0.f, e1 = 0.f, o0 = 0.f, o1 = 0.f;
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    e0 = __fadd_rn(e0, __fmul_rn(c.w[k], v[k].x));
    e1 = __fadd_rn(e1, __fmul_rn(c.w[k], v[k].y));
    o0 = __fadd_rn(o0, __fmul_rn(c.w[k + 1], v[k + 1].x));
    o1 = __fadd_rn(o1, __fmul_rn(c.w[k + 1], v[k + 1].y));
  }
  return make_float2(__fadd_rn(e0, o0), __fadd_rn(e1, o1));
}

// Coarse dense levels (a few thousand entries hit by every sample of the region) are
// contention-bound under global atomics: their gradients go to R private replicas
// (picked per warp) in a workspace, summed into the table by k_hash_rep_reduce.
struct RepPlan {
  int32_t n_rep;  // levels 0 .. n_rep-1 are replicated
  int32_t R[VR_MAX_LEVELS];
  int64_t off[VR_MAX_LEVELS];  // workspace offset (entries) of level l's replicas
};

// Half of a level's scatter for lane pairs (as gather_half): lane p adds w_c * d to the
// corners with cx = p.  The partner lane adds the x+1 corner of each row in the same
// 8-byte RED instruction, so entries in one 32-byte sector (x mod 4 != 3) cost one L2
// request (measured: two lanes' 8-byte adds into one sector run at the 16-byte-RED rate,
// scripts/micro/atom_bench.cu modes 4/7) — 1.25 requests per row instead of 1.5.
__device__ __forceinline__ void scatter_half(const VrHashGridDesc& g, const RepPlan& plan, int l,
                                             const float u[3], float2 d, int p, int gwarp,
                                             float2* __restrict__ grad, float2* __restrict__ ws) {
  int gi[3];
  float fr[3];
  level_cell(g, l, u, gi, fr);
  const int64_t size_l = g.offset[l + 1] - g.offset[l];
  float2* gl = (l < plan.n_rep) ? ws + plan.off[l] + (int64_t)(gwarp % plan.R[l]) * size_l
                                : grad + g.offset[l];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t idx;
    float w;
    corner(g, l, gi, fr, p + 2 * k, idx, w);
    if (!VR_CHECK((int64_t)idx < size_l)) continue;
    atomicAdd(gl + idx, make_float2(w * d.x, w * d.y));
  }
}

// host: replica plan + workspace / reduction sizes (entries)
RepPlan hash_rep_plan(const VrHashGridDesc* g, int64_t* ws_entries, int64_t* red_entries);
// host: sum the replicas into grad and zero them (enqueued on stream)
int hash_rep_reduce(const VrHashGridDesc* g, const RepPlan& plan, int64_t red_entries,
                    float* grad, void* ws, void* stream);

}  // namespace vr

namespace vr {
bool valid_grid(const VrHashGridDesc* g);
}  // namespace vr
