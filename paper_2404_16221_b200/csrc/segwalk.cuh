// Lane-serial segmented walks for K4 (composite.cu) and the interlevel loss (interlevel.cu).
//
// A warp owns 32 consecutive (region, ray) segments — a contiguous sample range — and walks
// it in chunks of 32 K samples: lane j takes the K consecutive samples
// [base + K j, base + K j + K) and folds them serially, so the cross-lane work (a
// segmented Hillis-Steele scan of one value per lane, carried across chunks) is paid once
// per 32 K samples instead of once per 32.  The segment composite is a monoid (NeRF-XL's
// own compositing rule, compose_render / compose_distortion segrender.py:93-142, applied to
// sub-ranges of one segment), so a lane's piece of a segment composes with the pieces of
// the lanes before it exactly like packets compose along a ray.
//
// The group's 33 segment offsets sit in shared memory (per warp), so a lane finds the
// segment of its first sample by binary search and steps to the next one by comparison.
#pragma once

#include "common.cuh"

namespace vr {

// largest j < nseg with off[j] <= s: the (non-empty) segment that holds sample s
__device__ __forceinline__ int seg_of(const int64_t* off, int nseg, int64_t s) {
  int j = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const int c = j + step;
    if (c < nseg && off[c] <= s) j = c;
  }
  return j;
}

// stage the group's offsets off[seg0 .. seg0 + nseg] (33 slots; slots past nseg repeat
// the end) into the warp's shared array
__device__ __forceinline__ void stage_offsets(const int64_t* __restrict__ off, int64_t seg0,
                                              int nseg, int lane, int64_t* s_off) {
  s_off[lane] = off[seg0 + min(lane, nseg)];
  if (lane == 0) s_off[32] = off[seg0 + nseg];
  __syncwarp();
}

// The next group's offsets, loaded into registers while the current group is walked (a
// group costs two dependent memory round trips — offsets, then its first chunk): used by
// the T-only walk (2.32 -> 2.27 ms at c4); the forward / backward walks, at 128 registers,
// spilled with it and got slower (5.7 -> 7.0 / 5.6 -> 5.8 ms).
// GroupPrefetch::load(g) issues the loads, stage() stores them for the walk.
struct GroupPrefetch {
  int64_t o, o32;
  int64_t seg0;
  int nseg;
  __device__ __forceinline__ void load(const int64_t* __restrict__ off, int64_t grp,
                                       int64_t n_groups, int64_t n_segs, int lane) {
    seg0 = grp * 32;
    nseg = grp < n_groups ? (int)min((int64_t)32, n_segs - seg0) : 0;
    o = o32 = 0;
    if (grp < n_groups) {
      o = __ldg(off + seg0 + min(lane, nseg));
      if (lane == 0) o32 = __ldg(off + seg0 + nseg);
    }
  }
  __device__ __forceinline__ void stage(int64_t* s_off, int lane) const {
    s_off[lane] = o;
    if (lane == 0) s_off[32] = o32;
    __syncwarp();
  }
};

// ray index of segment seg (segments are region-major, kk * n_rays + r); 32-bit when the
// batch allows (a 64-bit modulo costs ~100 instructions)
__device__ __forceinline__ int64_t seg_ray(int64_t seg, int64_t n_rays, bool narrow) {
  return narrow ? (int64_t)((uint32_t)seg % (uint32_t)n_rays) : seg % n_rays;
}

// The lane's span of a chunk: samples [s0, s0 + cnt), the segment of s0 and whether that
// segment started before s0 (its earlier part belongs to previous lanes / chunks).
struct LaneSpan {
  int64_t s0;
  int cnt, sf;
  bool open_left;
};

template <int K>
__device__ __forceinline__ LaneSpan lane_span(const int64_t* s_off, int nseg, int64_t base,
                                              int64_t s_end, int lane) {
  LaneSpan sp;
  sp.s0 = base + (int64_t)K * lane;
  sp.cnt = (int)max((int64_t)0, min((int64_t)K, s_end - sp.s0));
  sp.sf = sp.cnt > 0 ? seg_of(s_off, nseg, sp.s0) : nseg - 1;
  sp.open_left = sp.cnt > 0 && sp.s0 > s_off[sp.sf];
  return sp;
}

// ---- monoids -----------------------------------------------------------------------
// Forward composite of a run of samples: T = prod keep, C = sum w c, A = sum w,
// D = sum w m, L = sum_ij w_i w_j |m_i - m_j| (weights relative to the run's start).
struct Comp {
  double T, C0, C1, C2, A, D, L;
};
__device__ __forceinline__ Comp comp_id() { return {1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0}; }
// x then y (y behind x): compose_render / compose_distortion
__device__ __forceinline__ Comp comp_cat(const Comp& x, const Comp& y) {
  Comp r;
  r.T = x.T * y.T;
  r.C0 = x.C0 + x.T * y.C0;
  r.C1 = x.C1 + x.T * y.C1;
  r.C2 = x.C2 + x.T * y.C2;
  r.A = x.A + x.T * y.A;
  r.D = x.D + x.T * y.D;
  r.L = x.L + x.T * x.T * y.L + 2.0 * x.T * (x.A * y.D - y.A * x.D);
  return r;
}
// append one sample: w = T alpha, L += 2 w (m A - D) (the O(N) distortion), then the sums
__device__ __forceinline__ void comp_push(Comp& a, double keep, double alpha, const float4& v,
                                          double m) {
  const double w = a.T * alpha;
  a.L += 2.0 * w * (m * a.A - a.D);
  a.C0 += w * (double)v.y;
  a.C1 += w * (double)v.z;
  a.C2 += w * (double)v.w;
  a.A += w;
  a.D += w * m;
  a.T *= keep;
}
__device__ __forceinline__ Comp comp_shfl_up(const Comp& x, int o) {
  Comp r;
  r.T = __shfl_up_sync(0xffffffffu, x.T, o);
  r.C0 = __shfl_up_sync(0xffffffffu, x.C0, o);
  r.C1 = __shfl_up_sync(0xffffffffu, x.C1, o);
  r.C2 = __shfl_up_sync(0xffffffffu, x.C2, o);
  r.A = __shfl_up_sync(0xffffffffu, x.A, o);
  r.D = __shfl_up_sync(0xffffffffu, x.D, o);
  r.L = __shfl_up_sync(0xffffffffu, x.L, o);
  return r;
}
__device__ __forceinline__ Comp comp_shfl(const Comp& x, int src) {
  Comp r;
  r.T = __shfl_sync(0xffffffffu, x.T, src);
  r.C0 = __shfl_sync(0xffffffffu, x.C0, src);
  r.C1 = __shfl_sync(0xffffffffu, x.C1, src);
  r.C2 = __shfl_sync(0xffffffffu, x.C2, src);
  r.A = __shfl_sync(0xffffffffu, x.A, src);
  r.D = __shfl_sync(0xffffffffu, x.D, src);
  r.L = __shfl_sync(0xffffffffu, x.L, src);
  return r;
}

// Prefix state of the backward: T (transmittance), A (opacity), D (depth sum).
struct Pre {
  double T, A, D;
};
__device__ __forceinline__ Pre pre_id() { return {1.0, 0.0, 0.0}; }
__device__ __forceinline__ Pre pre_cat(const Pre& x, const Pre& y) {
  return {x.T * y.T, x.A + x.T * y.A, x.D + x.T * y.D};
}
__device__ __forceinline__ Pre pre_shfl_up(const Pre& x, int o) {
  return {__shfl_up_sync(0xffffffffu, x.T, o), __shfl_up_sync(0xffffffffu, x.A, o),
          __shfl_up_sync(0xffffffffu, x.D, o)};
}
__device__ __forceinline__ Pre pre_shfl(const Pre& x, int src) {
  return {__shfl_sync(0xffffffffu, x.T, src), __shfl_sync(0xffffffffu, x.A, src),
          __shfl_sync(0xffffffffu, x.D, src)};
}

// Segmented inclusive scan over lanes: S_j = E_i ∘ ... ∘ E_j from the last lane i <= j
// whose flag is set (a piece that starts inside its lane).  Cat(x, y): x in front of y.
template <class V, class Cat, class Up>
__device__ __forceinline__ V lane_seg_scan(V s, bool f, int lane, Cat cat, Up up) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V p = up(s, o);
    const bool pf = __shfl_up_sync(0xffffffffu, (int)f, o) != 0;
    if (lane >= o && !f) {
      s = cat(p, s);
      f = pf;
    }
  }
  return s;
}

}  // namespace vr
