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
#include <stdlib.h>

#include "common.cuh"
#include "pksrc.cuh"
#include "segscan.cuh"

namespace vr {

constexpr int IL_WARPS = 8;

// per ray: prefixes (P, Ph) of the NeRF and proposal transmittance before each owned
// segment, folded in the same first-sample order as K5
__global__ void k_prefix(const PacketSrc pk, int n_regions, int64_t n_rays, int own_lo,
                         int own_cnt, float2* __restrict__ prefix) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    int ord[VR_MAX_REGIONS], key[VR_MAX_REGIONS];
    int n = 0;
    for (int k = 0; k < n_regions; ++k) {
      const int kf = pk_key(pk, (int64_t)k * n_rays + r);
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
      float4 a, b;
      pk_load(pk, idx, a, b);
      P *= (double)a.x;
      Ph *= (double)pk_extra(pk, idx);
    }
  }
}

// Grouped like K4 (segscan.cuh): one warp per 32 consecutive (region, ray) segments walks
// their contiguous sample range 32 samples at a time with segmented scans, so no lane
// idles on short segments.  Sweep 1: local transmittances (NeRF, proposal), per-segment
// loss L and S = sum_i wh_loc_i e_i, and each sample's gradient up to the S term; sweep 2
// (reads 16 B per sample, no re-evaluation): per-sample proposal gradients.
struct IlChunk {
  bool valid, head, tail, cont;
  int seg;
  double dlt, keep, alpha, alphah, keeph;
  double T, Th;  // local exclusive transmittances (NeRF, proposal)
};

// one lane's inputs of a chunk, loaded one chunk ahead
struct IlIn {
  double a, b;
  float sig, sigh;
};

__device__ __forceinline__ IlIn il_load(const double* __restrict__ t0,
                                        const double* __restrict__ t1,
                                        const float4* __restrict__ sr,
                                        const float4* __restrict__ sp, int64_t s, int64_t s_end) {
  IlIn in = {0.0, 0.0, 0.f, 0.f};
  if (s < s_end) {
    in.a = t0[s];
    in.b = t1[s];
    in.sig = sr[s].x;
    in.sigh = sp[s].x;
  }
  return in;
}

__device__ __forceinline__ IlChunk il_chunk(const IlIn& in, int64_t s, int64_t s_end,
                                            const GroupSeg& gs, int nseg, double cT, double cTh,
                                            int lane) {
  IlChunk c;
  c.valid = s < s_end;
  c.seg = find_seg(gs.lo, nseg, c.valid ? s : s_end - 1);
  const int64_t seg_lo = __shfl_sync(0xffffffffu, gs.lo, c.seg);
  const int64_t seg_hi = __shfl_sync(0xffffffffu, gs.hi, c.seg);
  c.head = (s == seg_lo) || lane == 0;
  c.tail = c.valid && (s + 1 == seg_hi);
  const int seg0 = __shfl_sync(0xffffffffu, c.seg, 0);
  c.cont = (__shfl_sync(0xffffffffu, (int)(s != seg_lo), 0) != 0) && c.seg == seg0;
  c.keep = 1.0;
  c.keeph = 1.0;
  c.dlt = c.alpha = c.alphah = 0.0;
  if (c.valid) {
    c.dlt = in.b - in.a;
    const double x = (double)in.sig * c.dlt, xh = (double)in.sigh * c.dlt;
    // composite_samples' arithmetic (quadrature.py:152-154) and the oracle's: one exp each
    c.alpha = 1.0 - exp(-x);
    c.keep = 1.0 - c.alpha;
    c.alphah = 1.0 - exp(-xh);
    c.keeph = 1.0 - c.alphah;
  }
  double p[2] = {c.keep, c.keeph};
  seg_scan<2>(p, c.head, lane, [](double a, double b) { return a * b; });
  const double pu0 = __shfl_up_sync(0xffffffffu, p[0], 1);
  const double pu1 = __shfl_up_sync(0xffffffffu, p[1], 1);
  c.T = (c.cont ? cT : 1.0) * (c.head ? 1.0 : pu0);
  c.Th = (c.cont ? cTh : 1.0) * (c.head ? 1.0 : pu1);
  return c;
}

// 3 resident blocks (80 registers): c4 10.7 -> 9.5 ms (at 4 blocks / 64 registers the
// spills cost it back: 10.5)
__global__ void __launch_bounds__(IL_WARPS * 32, 3)
    k_interlevel(const double* __restrict__ t0, const double* __restrict__ t1,
                 const float4* __restrict__ sr, const float4* __restrict__ sp,
                 const int64_t* __restrict__ off, const float2* __restrict__ prefix,
                 int64_t n_segs, float lambda, float eps, double* __restrict__ seg_loss,
                 float4* __restrict__ dsp) {
  __shared__ double s_S[IL_WARPS][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Sseg = s_S[wid];
  const double lam = lambda, ep = eps;
  const int64_t n_groups = ceil_div(n_segs, 32);
  for (int64_t grp = (int64_t)blockIdx.x * IL_WARPS + wid; grp < n_groups;
       grp += (int64_t)gridDim.x * IL_WARPS) {
    const int64_t seg0 = grp * 32;
    const int nseg = (int)min((int64_t)32, n_segs - seg0);
    const int64_t my = seg0 + lane;
    GroupSeg gs;
    gs.lo = off[lane < nseg ? my : seg0 + nseg];
    gs.hi = off[lane < nseg ? my + 1 : seg0 + nseg];
    float2 pre = make_float2(1.f, 1.f);
    if (lane < nseg) {
      pre = prefix[my];
      if (gs.lo == gs.hi) seg_loss[my] = 0.0;  // empty segment
    }
    const int64_t s_beg = __shfl_sync(0xffffffffu, gs.lo, 0);
    const int64_t s_end = __shfl_sync(0xffffffffu, gs.hi, nseg - 1);
    if (s_beg == s_end) continue;
    // sweep 1: L and S per segment, and per sample the two terms of its gradient that do
    // not need the segment total S — parked in the sample's dsp slot as two doubles
    //   ds_i dt_i = x_i - y_i S,  x_i = Ph dt_i (Th_{i+1} e_i + S_<=i),  y_i = Ph dt_i
    double cT = 1.0, cTh = 1.0, cL = 0.0, cS = 0.0;
    double2* park = reinterpret_cast<double2*>(dsp);
    IlIn nxt = il_load(t0, t1, sr, sp, s_beg + lane, s_end);
    for (int64_t base = s_beg; base < s_end; base += 32) {
      const IlIn cur = nxt;
      nxt = il_load(t0, t1, sr, sp, base + 32 + lane, s_end);
      const IlChunk c = il_chunk(cur, base + lane, s_end, gs, nseg, cT, cTh, lane);
      const double P = __shfl_sync(0xffffffffu, (double)pre.x, c.seg);
      const double Ph = __shfl_sync(0xffffffffu, (double)pre.y, c.seg);
      const double w = P * c.T * c.alpha;
      const double whl = c.Th * c.alphah;
      const double d = fmax(w - Ph * whl, 0.0);
      const double inv = 1.0 / (w + ep);
      const double ei = -2.0 * lam * d * inv;
      double q[2] = {c.valid ? lam * d * d * inv : 0.0, c.valid ? whl * ei : 0.0};
      seg_scan<2>(q, c.head, lane, [](double a, double b) { return a + b; });
      const double L = (c.cont ? cL : 0.0) + q[0];
      const double S = (c.cont ? cS : 0.0) + q[1];
      const double Thn = c.Th * c.keeph;  // local proposal transmittance after sample i
      if (c.valid) {
        const double y = Ph * c.dlt;
        park[base + lane] = make_double2(y * (Thn * ei + S), y);
      }
      if (c.tail) {
        seg_loss[seg0 + c.seg] = L;
        Sseg[c.seg] = S;
      }
      cT = __shfl_sync(0xffffffffu, c.T * c.keep, 31);
      cTh = __shfl_sync(0xffffffffu, Thn, 31);
      cL = __shfl_sync(0xffffffffu, L, 31);
      cS = __shfl_sync(0xffffffffu, S, 31);
    }
    __syncwarp();
    // sweep 2: dL/dsigma_prop = x_i - y_i S of the sample's segment (no re-evaluation)
    for (int64_t base = s_beg; base < s_end; base += 32) {
      const int64_t s = base + lane;
      const bool valid = s < s_end;
      const int seg = find_seg(gs.lo, nseg, valid ? s : s_end - 1);
      if (valid) {
        const double2 xy = park[s];
        dsp[s] = make_float4((float)(xy.x - xy.y * Sseg[seg]), 0.f, 0.f, 0.f);
      }
    }
    __syncwarp();
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
  PacketSrc src;
  src.pk = reinterpret_cast<const float4*>(pk);
  src.extra = prop_T;
  src.rec = nullptr;
  src.index = nullptr;
  src.width = 0;
  k_prefix<<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(
      src, n_regions, n_rays, own_lo, own_cnt, reinterpret_cast<float2*>(prefix));
  return check_launch("vr_prefix_train");
}

extern "C" int vr_prefix_train_records(const float* recv, const int32_t* index, int32_t n_regions,
                                       int64_t n_rays, int32_t own_lo, int32_t own_cnt,
                                       float* prefix, void* stream) {
  if (n_regions < 1 || n_regions > VR_MAX_REGIONS || n_rays < 0 || own_lo < 0 || own_cnt < 1 ||
      own_lo + own_cnt > n_regions || !prefix || (n_rays > 0 && (!recv || !index))) {
    set_error("vr_prefix_train_records: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  PacketSrc src;  // records of width 10: the proposal T rides in field 9
  src.pk = nullptr;
  src.extra = nullptr;
  src.rec = recv;
  src.index = index;
  src.width = 10;
  k_prefix<<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(
      src, n_regions, n_rays, own_lo, own_cnt, reinterpret_cast<float2*>(prefix));
  return check_launch("vr_prefix_train_records");
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
  // dsig_prop doubles as the first sweep's scratch (a double2 parked in each sample's
  // 16-byte slot): it must be 16-byte aligned and must not alias the read-only inputs
  if (reinterpret_cast<uintptr_t>(dsig_prop) % 16 != 0 ||
      (const void*)dsig_prop == (const void*)sig_prop ||
      (const void*)dsig_prop == (const void*)sig_rgb) {
    set_error("vr_interlevel: dsig_prop must be 16-byte aligned and distinct from the inputs");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n_segs = n_rays * region_cnt;
  if (n_segs == 0) return VR_OK;
  k_interlevel<<<grid_for(ceil_div(n_segs, 32 * IL_WARPS), 1, 8), IL_WARPS * 32, 0, (cudaStream_t)stream>>>(
      t0, t1, reinterpret_cast<const float4*>(sig_rgb), reinterpret_cast<const float4*>(sig_prop),
      off, reinterpret_cast<const float2*>(prefix), n_segs, lambda, eps, seg_loss,
      reinterpret_cast<float4*>(dsig_prop));
  return check_launch("vr_interlevel");
}
