// Shared device helpers for the volray B200 kernels (sm_100a).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/vr_capi.h"

#define VR_SLIVER 1e-12 /* quadrature.py:19 */
// SM count of the current device (queried once per process in capi.cu; 148 on B200).
// Persistent grids and grid caps are sized in multiples of it.
#define VR_NUM_SMS (vr::num_sms())

namespace vr {

// Set by every entry point on a launch/argument failure; read by vr_last_error().
void set_error(const char* msg);
int check_launch(const char* where);
int num_sms();

// ---- checked build (-DVR_CHECKED, csrc/build.py --checked) -----------------------------
// compute-sanitizer is not available on this pool, so a debug build of the library adds
// device-side range checks at the hot global accesses (table entries, sample / segment /
// record indices); a failed check skips the access and counts the failure, read back by
// vr_check_failures().  Release builds compile the checks out.
#ifdef VR_CHECKED
static __device__ unsigned int g_check_failures;
#define VR_CHECK(cond) ((cond) ? true : (atomicAdd(&vr::g_check_failures, 1u), false))
int register_checker(int (*read_and_clear)());
static int read_and_clear_checks() {
  unsigned int v = 0, z = 0;
  cudaMemcpyFromSymbol(&v, g_check_failures, sizeof(v));
  cudaMemcpyToSymbol(g_check_failures, &z, sizeof(z));
  return (int)v;
}
static const int g_checker_registered = register_checker(&read_and_clear_checks);
#else
#define VR_CHECK(cond) true
#endif

// ---- exact float64 arithmetic (no FMA contraction) ------------------------------
// The reference computes in numpy float64 without fused multiply-add; these
// intrinsics are never contracted by nvcc, so edges, midpoints and positions are
// bit-identical to the reference (quadrature.py:83, :40, geometry.py:93-94).
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

struct RayD {
  double o[3], d[3], tn, tf;
};

__device__ __forceinline__ RayD load_ray(const double* __restrict__ rays, int64_t stride,
                                         int64_t r) {
  RayD ray;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ray.o[a] = __ldg(rays + a * stride + r);
    ray.d[a] = __ldg(rays + (3 + a) * stride + r);
  }
  ray.tn = __ldg(rays + 6 * stride + r);
  ray.tf = __ldg(rays + 7 * stride + r);
  return ray;
}

// Slab test, exact replica of geometry.ray_box_intersect (geometry.py:109-128):
// axes with d == 0 miss if the origin is outside the slab, else contribute
// (-inf, +inf); result is (max(t_near, max near), min(t_far, min far)) and a
// zero-length overlap is a miss.
__device__ __forceinline__ bool ray_box(const RayD& ray, const double* mn, const double* mx,
                                        double& t_enter, double& t_exit) {
  double near_max = -INFINITY, far_min = INFINITY;
  bool miss = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (ray.d[a] == 0.0) {
      if (ray.o[a] < mn[a] || ray.o[a] > mx[a]) miss = true;
    } else {
      double lo = ddiv(dsub(mn[a], ray.o[a]), ray.d[a]);
      double hi = ddiv(dsub(mx[a], ray.o[a]), ray.d[a]);
      near_max = fmax(near_max, fmin(lo, hi));
      far_min = fmin(far_min, fmax(lo, hi));
    }
  }
  // Python max()/min() keep the first argument on ties.
  t_enter = (near_max > ray.tn) ? near_max : ray.tn;
  t_exit = (far_min < ray.tf) ? far_min : ray.tf;
  return !miss && (t_enter < t_exit);
}

// p = o + m * d, as Ray.points_at (geometry.py:96-97)
__device__ __forceinline__ void point_at(const RayD& ray, double m, double p[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) p[a] = dadd(ray.o[a], dmul(m, ray.d[a]));
}

// partitioner.locate (partitioner.py:166-174): closed root box, p[axis] < plane -> low
__device__ __forceinline__ int locate_point(const VrTree& t, const double p[3], bool& oob) {
  oob = !(p[0] >= t.root_mn[0] && p[1] >= t.root_mn[1] && p[2] >= t.root_mn[2] &&
          p[0] <= t.root_mx[0] && p[1] <= t.root_mx[1] && p[2] <= t.root_mx[2]);
  if (t.n_nodes == 0) return 0;
  int node = 0;
#pragma unroll 1
  for (int depth = 0; depth < VR_MAX_REGIONS; ++depth) {
    int a = t.node_axis[node];
    int c = (p[a] < t.node_plane[node]) ? t.node_low[node] : t.node_high[node];
    if (c < 0) return -c - 1;
    node = c;
  }
  return 0;
}

// a sample's ray index (checked build: within [0, n_rays), else ray 0 and a failure)
__device__ __forceinline__ int64_t checked_ray(int64_t r, int64_t n_rays) {
  return VR_CHECK(r >= 0 && r < n_rays) ? r : 0;
}

__device__ __forceinline__ double sample_mid(double t0, double t1) {
  return dmul(0.5, dadd(t0, t1));  // SampleInterval.__post_init__ (quadrature.py:40)
}

// ---- warp scans (float64 / int) ------------------------------------------------------
__device__ __forceinline__ double warp_incl_sum(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
__device__ __forceinline__ double warp_incl_prod(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v *= n;
  }
  return v;
}
__device__ __forceinline__ int warp_incl_sum_i(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

inline int grid_for(int64_t work, int per_block, int max_blocks_per_sm = 8) {
  int64_t g = ceil_div(work, per_block);
  int64_t cap = (int64_t)VR_NUM_SMS * max_blocks_per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace vr
