// Interlevel (proposal) loss for the distributed NeRF-XL step (north_star config 4).
//
// PARITY UNPINNED: neither the reference code nor PAPER.md/SPEC.md define it; the spec is
// restated in oracle/grad_oracle.py (field_loss with a proposal).  Mip-NeRF 360's
// proposal loss on the reference's fixed bins (the proposal is evaluated on the same
// intervals, so its "bound" for bin i is its own weight):
//     L_int = lambda * sum_i max(0, w_i - wh_i)^2 / (w_i + eps)
// with w_i = P_s * T_i alpha_i the NeRF weight (stop-gradient, as in Mip-NeRF 360) and
// wh_i = Ph_s * Th_i alphah_i the proposal weight; P_s / Ph_s are the global NeRF /
// proposal transmittance in front of segment s (from the exchanged packets) and — like
// peers' packets in NeRF-XL's own losses — constants, so each rank's
// proposal gradient is local and there is no gradient collective.
//   dL/dsh_j = Ph_s (Th_{j+1} e_j - sum_{i>j} wh_loc_i e_i),  e_i = dL/dwh_i
//            = -2 lambda max(0, w_i - wh_i) / (w_i + eps)
#include "common.cuh"

namespace vr {

constexpr int IL_WARPS = 8;

// per ray: prefixes (P, Ph) of the NeRF and proposal transmittance before each owned
// segment, folded in the same first-sample order as K5
__global__ void k_prefix(const float4* __restrict__ pk, const float* __restrict__ propT,
                         int n_regions, int64_t n_rays, int own_lo, int own_cnt,
                         float2* __restrict__ prefix) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    int ord[VR_MAX_REGIONS], key[VR_MAX_REGIONS];
    int n = 0;
    for (int k = 0; k < n_regions; ++k) {
      const int kf = __float_as_int(pk[2 * ((int64_t)k * n_rays + r) + 1].w);
      if (kf == INT32_MAX) continue;
      int j = n++;
      while (j > 0 && key[j - 1] > kf) {
        key[j] = key[j - 1];
        ord[j] = ord[j - 1];
        --j;
      }
      key[j] = kf;
      ord[j] = k;
    }
    for (int kk = 0; kk < own_cnt; ++kk) prefix[(int64_t)kk * n_rays + r] = make_float2(1.f, 1.f);
    double P = 1.0, Ph = 1.0;
    for (int s = 0; s < n; ++s) {
      const int64_t idx = (int64_t)ord[s] * n_rays + r;
      const int kk = ord[s] - own_lo;
      if (kk >= 0 && kk < own_cnt)
        prefix[(int64_t)kk * n_rays + r] = make_float2((float)P, (float)Ph);
      P *= (double)pk[2 * idx].x;
      Ph *= (double)propT[idx];
    }
  }
}

struct IlSample {
  double keep, alpha, keeph, alphah, dlt;
};

__device__ __forceinline__ IlSample il_load(const double* __restrict__ t0,
                                            const double* __restrict__ t1,
                                            const float4* __restrict__ sr,
                                            const float4* __restrict__ sp, int64_t i, bool valid) {
  IlSample s = {1.0, 0.0, 1.0, 0.0, 0.0};
  if (valid) {
    s.dlt = t1[i] - t0[i];
    const double x = (double)sr[i].x * s.dlt, xh = (double)sp[i].x * s.dlt;
    s.keep = exp(-x);
    s.alpha = -expm1(-x);
    s.keeph = exp(-xh);
    s.alphah = -expm1(-xh);
  }
  return s;
}

__global__ void __launch_bounds__(IL_WARPS * 32)
    k_interlevel(const double* __restrict__ t0, const double* __restrict__ t1,
                 const float4* __restrict__ sr, const float4* __restrict__ sp,
                 const int64_t* __restrict__ off, const float2* __restrict__ prefix,
                 int64_t n_segs, float lambda, float eps, double* __restrict__ seg_loss,
                 float4* __restrict__ dsp) {
  const int lane = threadIdx.x & 31;
  for (int64_t seg = (int64_t)blockIdx.x * IL_WARPS + (threadIdx.x >> 5); seg < n_segs;
       seg += (int64_t)gridDim.x * IL_WARPS) {
    const int64_t b = off[seg], e = off[seg + 1];
    if (b == e) {
      if (lane == 0) seg_loss[seg] = 0.0;
      continue;
    }
    const float2 pre = prefix[seg];
    const double P = pre.x, Ph = pre.y;
    // sweep 1: loss and S = sum_i wh_loc_i e_i
    double Tc = 1.0, Thc = 1.0, L = 0.0, S = 0.0;
    for (int64_t i0 = b; i0 < e; i0 += 32) {
      const int64_t i = i0 + lane;
      const IlSample s = il_load(t0, t1, sr, sp, i, i < e);
      const double p = warp_incl_prod(s.keep, lane), ph = warp_incl_prod(s.keeph, lane);
      double pe = __shfl_up_sync(0xffffffffu, p, 1), phe = __shfl_up_sync(0xffffffffu, ph, 1);
      if (lane == 0) pe = phe = 1.0;
      const double w = P * Tc * pe * s.alpha;
      const double whl = Thc * phe * s.alphah;
      const double d = fmax(w - Ph * whl, 0.0);
      const double inv = 1.0 / (w + (double)eps);
      L += warp_sum((double)lambda * d * d * inv);
      S += warp_sum(whl * (-2.0 * (double)lambda * d * inv));
      Tc *= __shfl_sync(0xffffffffu, p, 31);
      Thc *= __shfl_sync(0xffffffffu, ph, 31);
    }
    if (lane == 0) seg_loss[seg] = L;
    // sweep 2: per-sample proposal gradients
    Tc = 1.0;
    Thc = 1.0;
    double Sc = 0.0;
    for (int64_t i0 = b; i0 < e; i0 += 32) {
      const int64_t i = i0 + lane;
      const IlSample s = il_load(t0, t1, sr, sp, i, i < e);
      const double p = warp_incl_prod(s.keep, lane), ph = warp_incl_prod(s.keeph, lane);
      double pe = __shfl_up_sync(0xffffffffu, p, 1), phe = __shfl_up_sync(0xffffffffu, ph, 1);
      if (lane == 0) pe = phe = 1.0;
      const double w = P * Tc * pe * s.alpha;
      const double whl = Thc * phe * s.alphah;
      const double d = fmax(w - Ph * whl, 0.0);
      const double ei = -2.0 * (double)lambda * d / (w + (double)eps);
      const double we = whl * ei;
      const double incl = warp_incl_sum(we, lane);
      const double s_gt = S - (Sc + incl);
      const double Thn = Thc * ph;  // local proposal transmittance after sample i
      const double ds = Ph * (Thn * ei - s_gt);
      if (i < e) dsp[i] = make_float4((float)(ds * s.dlt), 0.f, 0.f, 0.f);
      Tc *= __shfl_sync(0xffffffffu, p, 31);
      Thc *= __shfl_sync(0xffffffffu, ph, 31);
      Sc += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

}  // namespace vr

using namespace vr;

extern "C" int vr_prefix_train(const float* pk, const float* prop_T, int32_t n_regions,
                               int64_t n_rays, int32_t own_lo, int32_t own_cnt, float* prefix,
                               void* stream) {
  if (n_regions < 1 || n_regions > VR_MAX_REGIONS || n_rays < 0 || own_lo < 0 || own_cnt < 1 ||
      own_lo + own_cnt > n_regions || !prop_T || !prefix) {
    set_error("vr_prefix_train: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  k_prefix<<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4*>(pk), prop_T, n_regions, n_rays, own_lo, own_cnt,
      reinterpret_cast<float2*>(prefix));
  return check_launch("vr_prefix_train");
}

extern "C" int vr_interlevel(const double* t0, const double* t1, const float* sig_rgb,
                             const float* sig_prop, const int64_t* off, const float* prefix,
                             int64_t n_rays, int32_t region_cnt, float lambda, float eps,
                             double* seg_loss, float* dsig_prop, void* stream) {
  if (n_rays < 0 || region_cnt < 1 || region_cnt > VR_MAX_REGIONS || !(eps > 0.f) || !seg_loss ||
      !dsig_prop) {
    set_error("vr_interlevel: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n_segs = n_rays * region_cnt;
  if (n_segs == 0) return VR_OK;
  k_interlevel<<<grid_for(ceil_div(n_segs, IL_WARPS), 1, 8), IL_WARPS * 32, 0,
                 (cudaStream_t)stream>>>(t0, t1, reinterpret_cast<const float4*>(sig_rgb),
                                         reinterpret_cast<const float4*>(sig_prop), off,
                                         reinterpret_cast<const float2*>(prefix), n_segs, lambda,
                                         eps, seg_loss, reinterpret_cast<float4*>(dsig_prop));
  return check_launch("vr_interlevel");
}
