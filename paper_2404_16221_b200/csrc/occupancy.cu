// Per-region occupancy grid: the paper trains with an occupancy grid per
// region for empty-space skipping; the reference simulator has none
// (SPEC.md:192).  K1 reads the bits (VrOccupancy, vr_capi.h; the cell formula is in
// sampler.cu occupied()); these kernels maintain them from the region's field:
//
//   vr_occupancy_points  one jittered point per cell of a leaf's res^3 grid, written as
//                        zero-length rays (origin = point) so any region field kernel
//                        evaluates it (t0 = t1 = 0: the sample point is the origin);
//   vr_occupancy_update  density EMA d = max(decay * d, sigma) per cell (Instant-NGP's
//                        grid update), bit = d > threshold, one thread per 32-cell word.
//
// The jitter is an integer hash of (seed, cell, axis) restated bit for bit in
// oracle/volray_oracle.py (occupancy_points).
#include "common.cuh"

namespace vr {

__host__ __device__ __forceinline__ uint32_t occ_hash(uint32_t x) {
  // lowbias32 (Wellons): full-avalanche 32-bit integer hash
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

__global__ void k_occ_points(const double mn0, const double mn1, const double mn2,
                             const double mx0, const double mx1, const double mx2, int G,
                             uint32_t seed, int64_t n, double* __restrict__ rays) {
  const double mn[3] = {mn0, mn1, mn2}, mx[3] = {mx0, mx1, mx2};
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cc[3] = {c % G, (c / G) % G, c / ((int64_t)G * G)};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint32_t h = occ_hash(seed * 0x9E3779B9u + (uint32_t)(c * 3 + a));
      const double u = (double)(h >> 8) * (1.0 / 16777216.0);  // [0, 1), 24 bits
      // mn + ((cell + u) / G) * (mx - mn), no FMA
      const double f = ddiv(dadd((double)cc[a], u), (double)G);
      rays[a * n + c] = dadd(mn[a], dmul(f, dsub(mx[a], mn[a])));
      rays[(3 + a) * n + c] = a == 0 ? 1.0 : 0.0;
    }
    rays[6 * n + c] = 0.0;
    rays[7 * n + c] = 1.0;
  }
}

__global__ void k_occ_update(const float4* __restrict__ sig_rgb, int64_t n, float decay,
                             float threshold, float* __restrict__ density,
                             uint32_t* __restrict__ bits) {
  const int64_t words = (n + 31) / 32;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t c = w * 32 + b;
      if (c >= n) break;
      const float d = fmaxf(density[c] * decay, sig_rgb[c].x);
      density[c] = d;
      if (d > threshold) word |= 1u << b;
    }
    bits[w] = word;
  }
}

}  // namespace vr

using namespace vr;

extern "C" int vr_occupancy_points(const double* box_mn, const double* box_mx, int32_t res,
                                   uint32_t seed, double* rays_dev, void* stream) {
  if (!box_mn || !box_mx || res < 1 || res > 1024 || !rays_dev) {
    set_error("vr_occupancy_points: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n = (int64_t)res * res * res;
  k_occ_points<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      box_mn[0], box_mn[1], box_mn[2], box_mx[0], box_mx[1], box_mx[2], res, seed, n, rays_dev);
  return check_launch("vr_occupancy_points");
}

extern "C" int vr_occupancy_update(const float* sig_rgb_dev, int32_t res, float decay,
                                   float threshold, float* density_dev, uint32_t* bits_dev,
                                   void* stream) {
  if (!sig_rgb_dev || res < 1 || res > 1024 || !density_dev || !bits_dev ||
      !(decay >= 0.f && decay <= 1.f)) {
    set_error("vr_occupancy_update: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n = (int64_t)res * res * res;
  k_occ_update<<<grid_for((n + 31) / 32, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(sig_rgb_dev), n, decay, threshold, density_dev,
      bits_dev);
  return check_launch("vr_occupancy_update");
}
