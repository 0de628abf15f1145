// Float64 segment aggregation and composition: the reference's per-segment API
// (aggregate_segment / compose_render / compose_distortion, segrender.py:71-142) on the
// GPU for callers that hand in float64 bins or packets — the reference's own hand cases,
// the finite-difference probe (DistributedLossProbe, segrender.py:146-251) — where the
// float32 packets of the training path (K4 / K5, composite.cu) would cost the 1e-15
// agreement those callers expect.  Every multiply / add is round-to-nearest without FMA
// contraction, in the reference's operation order, so composition is bitwise the
// reference's Python float arithmetic; exp() is CUDA's (<= 1 ulp from the host libm).
#include "common.cuh"

namespace vr {

// One thread per segment: composite_samples (quadrature.py:141-165) over the segment's
// bins [off[s], off[s+1]) with local T starting at 1; the distortion by the O(N) prefix
// form sum_i 2 w_i (m_i A_<i - D_<i) (equal to the O(N^2) pairwise sum).
// out[s] = {T, C0, C1, C2, A, D, L, order_t = t0 of the first bin (inf when empty)}.
__global__ void k_segment_aggregate_f64(const double* __restrict__ t0,
                                        const double* __restrict__ t1,
                                        const double* __restrict__ sigma,
                                        const double* __restrict__ rgb,
                                        const int64_t* __restrict__ off, int64_t n_segs,
                                        double* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_segs;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = off[s], hi = off[s + 1];
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, A = 0.0, D = 0.0, L = 0.0;
    for (int64_t i = lo; i < hi; ++i) {
      const double delta = dsub(t1[i], t0[i]);
      const double alpha = dsub(1.0, exp(-dmul(sigma[i], delta)));
      const double w = dmul(T, alpha);
      const double m = sample_mid(t0[i], t1[i]);
      L = dadd(L, dmul(dmul(2.0, w), dsub(dmul(m, A), D)));
      C0 = dadd(C0, dmul(w, rgb[3 * i]));
      C1 = dadd(C1, dmul(w, rgb[3 * i + 1]));
      C2 = dadd(C2, dmul(w, rgb[3 * i + 2]));
      A = dadd(A, w);
      D = dadd(D, dmul(w, m));
      T = dmul(T, dsub(1.0, alpha));
    }
    double* o = out + 8 * s;
    o[0] = T;
    o[1] = C0;
    o[2] = C1;
    o[3] = C2;
    o[4] = A;
    o[5] = D;
    o[6] = L;
    o[7] = hi > lo ? t0[lo] : INFINITY;
  }
}

// One thread per ray: compose_render + compose_distortion (segrender.py:93-142) over the
// ray's n[r] packets, already in (order_t, tile) order, seg[r][k] = {T, C0, C1, C2, A, D,
// L}.  out[r] = {C0, C1, C2, A, D, T, L}; a non-finite packet raises VR_FLAG_NONFINITE,
// L < -1e-12 VR_FLAG_NEG_LOSS (smaller negatives clamp to 0).
__global__ void k_compose_f64(const double* __restrict__ seg, const int32_t* __restrict__ n,
                              int32_t max_segs, int64_t n_rays, double* __restrict__ out,
                              int32_t* err) {
  int flags = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int k_n = min(max(n[r], 0), max_segs);
    const double* p = seg + (int64_t)r * max_segs * 7;
    bool finite = true;
    for (int k = 0; k < k_n; ++k)
      for (int j = 0; j < 7; ++j) finite = finite && isfinite(p[7 * k + j]);
    double T = 1.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, A = 0.0, D = 0.0, L = 0.0;
    for (int k = 0; k < k_n; ++k) {
      const double* q = p + 7 * k;
      const double cross = dsub(dmul(q[5], A), dmul(q[4], D));
      L = dadd(L, dadd(dmul(dmul(T, T), q[6]), dmul(dmul(2.0, T), cross)));
      C0 = dadd(C0, dmul(T, q[1]));
      C1 = dadd(C1, dmul(T, q[2]));
      C2 = dadd(C2, dmul(T, q[3]));
      A = dadd(A, dmul(T, q[4]));
      D = dadd(D, dmul(T, q[5]));
      T = dmul(T, q[0]);
    }
    if (!finite) flags |= VR_FLAG_NONFINITE;
    if (L < 0.0) {
      if (L < -1e-12) flags |= VR_FLAG_NEG_LOSS;
      L = 0.0;
    }
    double* o = out + 7 * r;
    o[0] = C0;
    o[1] = C1;
    o[2] = C2;
    o[3] = A;
    o[4] = D;
    o[5] = T;
    o[6] = L;
  }
  if (flags && err) atomicOr(err, flags);
}

}  // namespace vr

using namespace vr;

extern "C" int vr_segment_aggregate_f64(const double* t0, const double* t1, const double* sigma,
                                        const double* rgb, const int64_t* seg_off,
                                        int64_t n_segs, double* out, void* stream) {
  if (n_segs < 0 || (n_segs > 0 && (!seg_off || !out))) {
    set_error("vr_segment_aggregate_f64: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_segs == 0) return VR_OK;
  k_segment_aggregate_f64<<<grid_for(n_segs, 128), 128, 0, (cudaStream_t)stream>>>(
      t0, t1, sigma, rgb, seg_off, n_segs, out);
  return check_launch("vr_segment_aggregate_f64");
}

extern "C" int vr_compose_f64(const double* seg, const int32_t* n_segs, int32_t max_segs,
                              int64_t n_rays, double* out, int32_t* err, void* stream) {
  if (n_rays < 0 || max_segs < 0 || (n_rays > 0 && (!n_segs || !out))) {
    set_error("vr_compose_f64: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  k_compose_f64<<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(seg, n_segs, max_segs,
                                                                          n_rays, out, err);
  return check_launch("vr_compose_f64");
}
