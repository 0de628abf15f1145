// Grouped-segment helpers shared by K4 (composite.cu) and the interlevel loss
// (interlevel.cu).
#pragma once

#include "common.cuh"

namespace vr {

// ---- grouped K4: one warp per 32 consecutive segments ---------------------------------
// The samples of consecutive segments are contiguous, so a warp walks the group's whole
// sample range 32 samples at a time with segmented warp scans (head flags at segment
// starts); empty segments cost nothing but their identity packet, and no lane idles on
// short segments.  Carries link a segment that spans two chunks.
struct GroupSeg {
  int64_t lo, hi;  // lane j: sample range of segment seg0 + j
};

// index of the segment (0..nseg-1) that contains sample s (largest j with lo[j] <= s)
__device__ __forceinline__ int find_seg(int64_t my_lo, int nseg, int64_t s) {
  int j = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const int cand = j + step;
    const int64_t lo_c = __shfl_sync(0xffffffffu, my_lo, cand < 32 ? cand : 31);
    if (cand < nseg && lo_c <= s) j = cand;
  }
  return j;
}

// segmented inclusive scans of up to 4 doubles sharing the head flags
template <int NV, class Op>
__device__ __forceinline__ void seg_scan(double* v, bool head, int lane, Op op) {
  bool f = head;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double nv[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) nv[k] = __shfl_up_sync(0xffffffffu, v[k], o);
    const bool nf = __shfl_up_sync(0xffffffffu, (int)f, o) != 0;
    if (lane >= o && !f) {
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] = op(nv[k], v[k]);
      f = nf;
    }
  }
}

}  // namespace vr
