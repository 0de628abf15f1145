// K4 (per-segment composite, fwd + analytic bwd) and K5 (global composite, fwd +
// train fwd/bwd), plus the deterministic loss reduction and the Adam step.
//
// K4 — grouped: one warp per 32 consecutive (region, ray) segments walks their contiguous
// sample range 32 samples at a time with segmented float64 warp scans (segscan.cuh),
// loading the next chunk while scanning the current one.  Forward (composite_samples
// quadrature.py:141-165 and
// aggregate_segment segrender.py:71-90):
//   s_i = sigma_i * delta_i,  keep_i = exp(-s_i),  alpha_i = -expm1(-s_i)
//   T_i = prod_{j<i} keep_j,  w_i = T_i alpha_i
//   C = sum w c, A = sum w, D' = sum w (m - te), T = prod keep
//   L = sum_ij w_i w_j |m_i - m_j| = 2 sum_i w_i (m_i A_<i - D_<i)   (O(N) form of
//       distortion_bruteforce quadrature.py:179-188; equal for sorted midpoints)
// Backward, for adjoints (bT, bC, bA, bD, bL) of the packet:
//   dL/ds_j = -bT T + T_{j+1} v_j - sum_{i>j} w_i v_i
//   v_i = bC.c_i + bA + bD m_i + bL g_i,  g_i = 2 sum_k w_k |m_i - m_k|
//   dL/dsigma_j = delta_j dL/ds_j,  dL/dc_j = w_j bC
// and sum_{i>j} w_i v_i is formed from the segment totals minus inclusive prefixes
// (sum_i w_i g_i = 2L), all in float64.
//
// K5 — one thread per ray: gather the ray's packets from every region, order the
// non-empty ones by their first-sample index (exact stand-in for the reference's
// (order_t, tile) sort, distsim.py:378), fold in float64 (compose_render
// segrender.py:93-110, compose_distortion segrender.py:113-142), and for training
// run the reverse sweep of that fold to get every owned packet's adjoint.
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "segscan.cuh"  // grouped-segment helpers (GroupSeg, find_seg, seg_scan)
#include "segwalk.cuh"  // lane-serial segmented walks (LaneSpan, Comp, Pre, lane_seg_scan)
#include "tma.cuh"      // TMA staging of the walks' per-sample inputs
#include "pksrc.cuh"    // K5's packet source: the dense slab or the exchanged records

namespace vr {

constexpr int SEG_WARPS = 8;
constexpr int SEG_TOT = 7;  // float64 segment totals kept for the backward: T, C[3], A, D, L

__device__ __forceinline__ float order_bits(int32_t first) { return __int_as_float(first); }

struct Carry {
  double T, A, D, L, C0, C1, C2, V;
};

// Per-lane quantities of one chunk of a group (forward sweep).
struct ChunkFwd {
  bool valid, head, tail, cont;
  int seg;
  double keep, alpha, m, dlt;
  float4 v;
  double Ti, Tn, w, a_lt, d_lt, a_incl, d_incl;  // Tn = T_{i+1}
  double l_incl, c_incl[3];
};

// One lane's sample of a chunk, loaded one chunk ahead by the kernels (the scans of the
// current chunk hide the next chunk's load latency).
struct ChunkIn {
  double a, b;
  float4 v;
};

__device__ __forceinline__ ChunkIn chunk_load(const double* __restrict__ t0,
                                              const double* __restrict__ t1,
                                              const float4* __restrict__ sr, int64_t s,
                                              int64_t s_end) {
  ChunkIn in = {0.0, 0.0, make_float4(0.f, 0.f, 0.f, 0.f)};
  if (s < s_end) {
    in.a = t0[s];
    in.b = t1[s];
    in.v = sr[s];
  }
  return in;
}

template <bool TOTALS = true>
__device__ __forceinline__ ChunkFwd chunk_forward(const ChunkIn& in, int64_t s, int64_t s_end,
                                                  const GroupSeg& gs, int nseg, double te_lane,
                                                  const Carry& cin, int lane) {
  ChunkFwd c;
  c.valid = s < s_end;
  c.seg = find_seg(gs.lo, nseg, c.valid ? s : s_end - 1);
  const int64_t seg_lo = __shfl_sync(0xffffffffu, gs.lo, c.seg);
  const int64_t seg_hi = __shfl_sync(0xffffffffu, gs.hi, c.seg);
  const double te = __shfl_sync(0xffffffffu, te_lane, c.seg);
  c.head = (s == seg_lo) || lane == 0;
  c.tail = c.valid && (s + 1 == seg_hi);
  // the chunk's first segment may continue from the previous chunk
  const int seg0 = __shfl_sync(0xffffffffu, c.seg, 0);
  const bool cont = (__shfl_sync(0xffffffffu, (int)(s != seg_lo), 0) != 0) && c.seg == seg0;
  c.keep = 1.0;
  c.alpha = 0.0;
  c.m = 0.0;
  c.dlt = 0.0;
  c.v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c.valid) {
    const double a = in.a, b = in.b;
    c.v = in.v;
    c.dlt = b - a;
    const double x = (double)c.v.x * c.dlt;
    c.keep = exp(-x);
    c.alpha = -expm1(-x);
    c.m = sample_mid(a, b) - te;
  }
  // transmittance
  double p[1] = {c.keep};
  seg_scan<1>(p, c.head, lane, [](double a, double b) { return a * b; });
  const double p_up = __shfl_up_sync(0xffffffffu, p[0], 1);
  const double p_excl = c.head ? 1.0 : p_up;
  const double cT = cont ? cin.T : 1.0;
  c.Ti = cT * p_excl;
  c.Tn = cT * p[0];
  c.w = c.Ti * c.alpha;
  // opacity / depth prefix sums
  double q[2] = {c.w, c.w * c.m};
  seg_scan<2>(q, c.head, lane, [](double a, double b) { return a + b; });
  const double q0_up = __shfl_up_sync(0xffffffffu, q[0], 1);
  const double q1_up = __shfl_up_sync(0xffffffffu, q[1], 1);
  const double cA = cont ? cin.A : 0.0, cD = cont ? cin.D : 0.0;
  c.a_lt = cA + (c.head ? 0.0 : q0_up);
  c.d_lt = cD + (c.head ? 0.0 : q1_up);
  c.a_incl = cA + q[0];
  c.d_incl = cD + q[1];
  c.cont = cont;
  if (TOTALS) {
    // distortion terms and colour
    double r[4] = {c.w * (c.m * c.a_lt - c.d_lt), c.w * (double)c.v.y, c.w * (double)c.v.z,
                   c.w * (double)c.v.w};
    seg_scan<4>(r, c.head, lane, [](double a, double b) { return a + b; });
    c.l_incl = (cont ? cin.L : 0.0) + 2.0 * r[0];
    c.c_incl[0] = (cont ? cin.C0 : 0.0) + r[1];
    c.c_incl[1] = (cont ? cin.C1 : 0.0) + r[2];
    c.c_incl[2] = (cont ? cin.C2 : 0.0) + r[3];
  }
  return c;
}

__device__ __forceinline__ Carry carry_out(const ChunkFwd& c) {
  Carry o;
  o.T = __shfl_sync(0xffffffffu, c.Tn, 31);
  o.A = __shfl_sync(0xffffffffu, c.a_incl, 31);
  o.D = __shfl_sync(0xffffffffu, c.d_incl, 31);
  o.L = __shfl_sync(0xffffffffu, c.l_incl, 31);
  o.C0 = __shfl_sync(0xffffffffu, c.c_incl[0], 31);
  o.C1 = __shfl_sync(0xffffffffu, c.c_incl[1], 31);
  o.C2 = __shfl_sync(0xffffffffu, c.c_incl[2], 31);
  o.V = 0.0;
  return o;
}

__global__ void __launch_bounds__(SEG_WARPS * 32)
    k_segment_fwd_grp(const double* __restrict__ t0, const double* __restrict__ t1,
                      const float4* __restrict__ sr, const int64_t* __restrict__ off,
                      const int32_t* __restrict__ seg_first, const double* __restrict__ ray_te,
                      int64_t n_rays, int64_t n_segs, float4* __restrict__ packets,
                      double* __restrict__ seg_tot) {
  const int lane = threadIdx.x & 31;
  const int64_t n_groups = ceil_div(n_segs, 32);
  for (int64_t grp = (int64_t)blockIdx.x * SEG_WARPS + (threadIdx.x >> 5); grp < n_groups;
       grp += (int64_t)gridDim.x * SEG_WARPS) {
    const int64_t seg0 = grp * 32;
    const int nseg = (int)min((int64_t)32, n_segs - seg0);
    const int64_t my = seg0 + lane;
    GroupSeg gs;
    gs.lo = off[lane < nseg ? my : seg0 + nseg];
    gs.hi = off[lane < nseg ? my + 1 : seg0 + nseg];
    const double te_lane = lane < nseg ? ray_te[my % n_rays] : 0.0;
    const int64_t s_beg = __shfl_sync(0xffffffffu, gs.lo, 0);
    const int64_t s_end = __shfl_sync(0xffffffffu, gs.hi, nseg - 1);
    // empty segments: identity packet
    if (lane < nseg && gs.lo == gs.hi) {
      packets[2 * my] = make_float4(1.f, 0.f, 0.f, 0.f);
      packets[2 * my + 1] = make_float4(0.f, 0.f, 0.f, order_bits(INT32_MAX));
    }
    Carry cin = {1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    ChunkIn nxt = chunk_load(t0, t1, sr, s_beg + lane, s_end);
    for (int64_t base = s_beg; base < s_end; base += 32) {
      const ChunkIn cur = nxt;
      nxt = chunk_load(t0, t1, sr, base + 32 + lane, s_end);
      const ChunkFwd c = chunk_forward(cur, base + lane, s_end, gs, nseg, te_lane, cin, lane);
      if (c.tail) {
        const int64_t seg = seg0 + c.seg;
        packets[2 * seg] = make_float4((float)c.Tn, (float)c.c_incl[0], (float)c.c_incl[1],
                                       (float)c.c_incl[2]);
        packets[2 * seg + 1] = make_float4((float)c.a_incl, (float)c.d_incl, (float)c.l_incl,
                                           order_bits(seg_first[seg]));
        if (seg_tot) {  // float64 totals for the backward (its sweep 1)
          double* st = seg_tot + SEG_TOT * seg;
          st[0] = c.Tn;
          st[1] = c.c_incl[0];
          st[2] = c.c_incl[1];
          st[3] = c.c_incl[2];
          st[4] = c.a_incl;
          st[5] = c.d_incl;
          st[6] = c.l_incl;
        }
      }
      cin = carry_out(c);
    }
  }
}

// Segment transmittance only (the proposal fields' packets: the interlevel loss reads T
// alone): the forward's product scan without the colour / depth / distortion scans, the
// same float64 chain, so T[seg] == (float) of the full packet's T bit for bit.
__global__ void __launch_bounds__(SEG_WARPS * 32)
    k_segment_T_grp(const double* __restrict__ t0, const double* __restrict__ t1,
                    const float4* __restrict__ sr, const int64_t* __restrict__ off,
                    int64_t n_segs, float* __restrict__ T_out) {
  const int lane = threadIdx.x & 31;
  const int64_t n_groups = ceil_div(n_segs, 32);
  const float* sigma = reinterpret_cast<const float*>(sr);
  for (int64_t grp = (int64_t)blockIdx.x * SEG_WARPS + (threadIdx.x >> 5); grp < n_groups;
       grp += (int64_t)gridDim.x * SEG_WARPS) {
    const int64_t seg0 = grp * 32;
    const int nseg = (int)min((int64_t)32, n_segs - seg0);
    const int64_t my = seg0 + lane;
    GroupSeg gs;
    gs.lo = off[lane < nseg ? my : seg0 + nseg];
    gs.hi = off[lane < nseg ? my + 1 : seg0 + nseg];
    const int64_t s_beg = __shfl_sync(0xffffffffu, gs.lo, 0);
    const int64_t s_end = __shfl_sync(0xffffffffu, gs.hi, nseg - 1);
    if (lane < nseg && gs.lo == gs.hi) T_out[my] = 1.f;  // empty segment: identity
    double carry = 1.0;
    for (int64_t base = s_beg; base < s_end; base += 32) {
      const int64_t s = base + lane;
      const bool valid = s < s_end;
      const int seg = find_seg(gs.lo, nseg, valid ? s : s_end - 1);
      const int64_t seg_lo = __shfl_sync(0xffffffffu, gs.lo, seg);
      const int64_t seg_hi = __shfl_sync(0xffffffffu, gs.hi, seg);
      const bool head = (s == seg_lo) || lane == 0;
      const int sg0 = __shfl_sync(0xffffffffu, seg, 0);
      const bool cont = (__shfl_sync(0xffffffffu, (int)(s != seg_lo), 0) != 0) && seg == sg0;
      double keep = 1.0;
      if (valid) {
        const double dlt = t1[s] - t0[s];
        keep = exp(-((double)sigma[4 * s] * dlt));
      }
      double p[1] = {keep};
      seg_scan<1>(p, head, lane, [](double a, double b) { return a * b; });
      const double Tn = (cont ? carry : 1.0) * p[0];
      if (valid && s + 1 == seg_hi) T_out[seg0 + seg] = (float)Tn;
      carry = __shfl_sync(0xffffffffu, Tn, 31);
    }
  }
}

// Grouped K4 backward: sweep 1 = the forward (segment totals into shared memory),
// sweep 2 = per-sample gradients with one more segmented scan for sum_{i>j} w_i v_i.
__global__ void __launch_bounds__(SEG_WARPS * 32)
    k_segment_bwd_grp(const double* __restrict__ t0, const double* __restrict__ t1,
                      const float4* __restrict__ sr, const int64_t* __restrict__ off,
                      const double* __restrict__ ray_te, int64_t n_rays, int64_t n_segs,
                      const float4* __restrict__ dpk, const double* __restrict__ seg_tot,
                      float4* __restrict__ dsr) {
  __shared__ double s_tot[SEG_WARPS][32][6];  // T, A, D, L, Vtot, bT*T per segment
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double(*tot)[6] = s_tot[wid];
  const int64_t n_groups = ceil_div(n_segs, 32);
  for (int64_t grp = (int64_t)blockIdx.x * SEG_WARPS + wid; grp < n_groups;
       grp += (int64_t)gridDim.x * SEG_WARPS) {
    const int64_t seg0 = grp * 32;
    const int nseg = (int)min((int64_t)32, n_segs - seg0);
    const int64_t my = seg0 + lane;
    GroupSeg gs;
    gs.lo = off[lane < nseg ? my : seg0 + nseg];
    gs.hi = off[lane < nseg ? my + 1 : seg0 + nseg];
    const double te_lane = lane < nseg ? ray_te[my % n_rays] : 0.0;
    const int64_t s_beg = __shfl_sync(0xffffffffu, gs.lo, 0);
    const int64_t s_end = __shfl_sync(0xffffffffu, gs.hi, nseg - 1);
    if (s_beg == s_end) continue;
    float4 g0 = make_float4(0.f, 0.f, 0.f, 0.f), g1 = g0;
    if (lane < nseg && gs.lo < gs.hi) {
      g0 = dpk[2 * my];
      g1 = dpk[2 * my + 1];
    }
    // sweep 1: totals (from the forward's float64 totals when it kept them)
    Carry cin = {1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    ChunkIn nxt = {0.0, 0.0, make_float4(0.f, 0.f, 0.f, 0.f)};
    if (!seg_tot) nxt = chunk_load(t0, t1, sr, s_beg + lane, s_end);
    if (seg_tot) {
      if (lane < nseg && gs.lo < gs.hi) {
        const double* st = seg_tot + SEG_TOT * my;
        const double Tn = st[0], c0 = st[1], c1 = st[2], c2 = st[3], a = st[4], d = st[5],
                     l = st[6];
        tot[lane][0] = Tn;
        tot[lane][1] = a;
        tot[lane][2] = d;
        tot[lane][3] = l;
        tot[lane][4] = (double)g0.y * c0 + (double)g0.z * c1 + (double)g0.w * c2 +
                       (double)g1.x * a + (double)g1.y * d + 2.0 * (double)g1.z * l;
        tot[lane][5] = (double)g0.x * Tn;
      }
    }
    for (int64_t base = s_beg; !seg_tot && base < s_end; base += 32) {
      const ChunkIn cur = nxt;
      nxt = chunk_load(t0, t1, sr, base + 32 + lane, s_end);
      const ChunkFwd c =
          chunk_forward<true>(cur, base + lane, s_end, gs, nseg, te_lane, cin, lane);
      if (c.tail) {
        tot[c.seg][0] = c.Tn;
        tot[c.seg][1] = c.a_incl;
        tot[c.seg][2] = c.d_incl;
        tot[c.seg][3] = c.l_incl;
        // Vtot = bC.C + bA A + bD D + 2 bL L  (adjoints of this segment)
        const float4 a0 = dpk[2 * (seg0 + c.seg)], a1 = dpk[2 * (seg0 + c.seg) + 1];
        tot[c.seg][4] = (double)a0.y * c.c_incl[0] + (double)a0.z * c.c_incl[1] +
                        (double)a0.w * c.c_incl[2] + (double)a1.x * c.a_incl +
                        (double)a1.y * c.d_incl + 2.0 * (double)a1.z * c.l_incl;
        tot[c.seg][5] = (double)a0.x * c.Tn;
      }
      cin = carry_out(c);
    }
    __syncwarp();
    // sweep 2: per-sample gradients
    cin = {1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    nxt = chunk_load(t0, t1, sr, s_beg + lane, s_end);
    for (int64_t base = s_beg; base < s_end; base += 32) {
      const ChunkIn cur = nxt;
      nxt = chunk_load(t0, t1, sr, base + 32 + lane, s_end);
      const ChunkFwd c =
          chunk_forward<false>(cur, base + lane, s_end, gs, nseg, te_lane, cin, lane);
      const float bC0 = __shfl_sync(0xffffffffu, g0.y, c.seg);
      const float bC1 = __shfl_sync(0xffffffffu, g0.z, c.seg);
      const float bC2 = __shfl_sync(0xffffffffu, g0.w, c.seg);
      const float bA = __shfl_sync(0xffffffffu, g1.x, c.seg);
      const float bD = __shfl_sync(0xffffffffu, g1.y, c.seg);
      const float bL = __shfl_sync(0xffffffffu, g1.z, c.seg);
      const double A_tot = tot[c.seg][1], D_tot = tot[c.seg][2], V_tot = tot[c.seg][4],
                   bTT = tot[c.seg][5];
      const double a_gt = A_tot - c.a_incl, d_gt = D_tot - c.d_incl;
      const double g = 2.0 * (c.m * c.a_lt - c.d_lt + d_gt - c.m * a_gt);
      const double vi = (double)bC0 * c.v.y + (double)bC1 * c.v.z + (double)bC2 * c.v.w +
                        (double)bA + (double)bD * c.m + (double)bL * g;
      double q[1] = {c.w * vi};
      seg_scan<1>(q, c.head, lane, [](double a, double b) { return a + b; });
      const double v_incl = (c.cont ? cin.V : 0.0) + q[0];
      const double ds = -bTT + c.Tn * vi - (V_tot - v_incl);
      if (c.valid)
        dsr[base + lane] = make_float4((float)(ds * c.dlt), (float)(c.w * bC0),
                                       (float)(c.w * bC1), (float)(c.w * bC2));
      cin = carry_out(c);
      cin.V = __shfl_sync(0xffffffffu, v_incl, 31);
    }
    __syncwarp();
  }
}

// ---- K5 ---------------------------------------------------------------------------------
struct Pk {
  double T, C[3], A, D, L;
};

__device__ __forceinline__ Pk load_pk(const PacketSrc& src, int64_t idx) {
  float4 a, b;
  pk_load(src, idx, a, b);
  Pk p;
  p.T = a.x;
  p.C[0] = a.y;
  p.C[1] = a.z;
  p.C[2] = a.w;
  p.A = b.x;
  p.D = b.y;
  p.L = b.z;
  return p;
}

template <bool TRAIN>
__global__ void k_global(const PacketSrc pk, int n_regions, int64_t n_rays,
                         const double* __restrict__ ray_te, float bg0, float bg1, float bg2,
                         int clip_bg, const float* __restrict__ targets, float lambda_dist,
                         int own_lo, int own_cnt, float* __restrict__ out,
                         double* __restrict__ ray_loss, float4* __restrict__ dpk, int32_t* err) {
  int flags = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rays;
       r += (int64_t)gridDim.x * blockDim.x) {
    // non-empty packets of this ray, ordered by first-sample index
    int ord[VR_MAX_REGIONS];
    int key[VR_MAX_REGIONS];
    int n = 0;
    for (int k = 0; k < n_regions; ++k) {
      const int kf = pk_key(pk, (int64_t)k * n_rays + r);
      if (kf == INT32_MAX) continue;
      int j = n++;
      while (j > 0 && key[j - 1] > kf) {  // insertion sort, ties impossible
        key[j] = key[j - 1];
        ord[j] = ord[j - 1];
        --j;
      }
      key[j] = kf;
      ord[j] = k;
    }
    double P = 1.0, C[3] = {0.0, 0.0, 0.0}, A = 0.0, D = 0.0, L = 0.0;
    double sP[VR_MAX_REGIONS], sA[VR_MAX_REGIONS], sD[VR_MAX_REGIONS];
    for (int s = 0; s < n; ++s) {
      const Pk p = load_pk(pk, (int64_t)ord[s] * n_rays + r);
      if (!(isfinite(p.T) && isfinite(p.C[0]) && isfinite(p.C[1]) && isfinite(p.C[2]) &&
            isfinite(p.A) && isfinite(p.D) && isfinite(p.L)))
        flags |= VR_FLAG_NONFINITE;
      sP[s] = P;
      sA[s] = A;
      sD[s] = D;
      L += P * P * p.L + 2.0 * P * (p.D * A - p.A * D);
      C[0] += P * p.C[0];
      C[1] += P * p.C[1];
      C[2] += P * p.C[2];
      A += P * p.A;
      D += P * p.D;
      P *= p.T;
    }
    if (L < 0.0) {
      if (L < -1e-12) flags |= VR_FLAG_NEG_LOSS;
      L = 0.0;
    }
    const double te = ray_te[r];
    const double bg[3] = {bg0, bg1, bg2};
    double pix[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) pix[c] = C[c] + P * bg[c];
#pragma unroll
    for (int c = 0; c < 3; ++c)
      out[c * n_rays + r] = clip_bg ? (float)fmin(fmax(pix[c], 0.0), 1.0) : (float)C[c];
    out[3 * n_rays + r] = (float)A;
    out[4 * n_rays + r] = (float)(D + A * te);
    out[5 * n_rays + r] = (float)P;
    out[6 * n_rays + r] = (float)L;
    if (TRAIN) {
      double gC[3], loss = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double d = pix[c] - (double)targets[3 * r + c];
        loss += d * d;
        gC[c] = 2.0 * d;
      }
      loss += (double)lambda_dist * L;
      ray_loss[r] = loss;
      const double gL = lambda_dist;
      // reverse sweep of the fold
      double bP = gC[0] * bg[0] + gC[1] * bg[1] + gC[2] * bg[2];  // adjoint of final P
      double bAc = 0.0, bDc = 0.0;
      for (int k = 0; k < own_cnt; ++k) {
        // zero the adjoints of owned regions first (empty / absent segments)
        const int64_t idx = (int64_t)k * n_rays + r;
        dpk[2 * idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        dpk[2 * idx + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      for (int s = n - 1; s >= 0; --s) {
        const Pk p = load_pk(pk, (int64_t)ord[s] * n_rays + r);
        const double Ps = sP[s], As = sA[s], Ds = sD[s];
        const int kk = ord[s] - own_lo;
        if (kk >= 0 && kk < own_cnt) {
          const int64_t idx = (int64_t)kk * n_rays + r;
          const double dT = bP * Ps;
          const double dA = bAc * Ps + gL * 2.0 * Ps * (-Ds);
          const double dD = bDc * Ps + gL * 2.0 * Ps * As;
          const double dL = gL * Ps * Ps;
          dpk[2 * idx] = make_float4((float)dT, (float)(gC[0] * Ps), (float)(gC[1] * Ps),
                                     (float)(gC[2] * Ps));
          dpk[2 * idx + 1] = make_float4((float)dA, (float)dD, (float)dL, 0.f);
        }
        // adjoint of the state before segment s
        const double nbP = bP * p.T + gC[0] * p.C[0] + gC[1] * p.C[1] + gC[2] * p.C[2] +
                           bAc * p.A + bDc * p.D +
                           gL * (2.0 * Ps * p.L + 2.0 * (p.D * As - p.A * Ds));
        const double nbA = bAc + gL * 2.0 * Ps * p.D;
        const double nbD = bDc - gL * 2.0 * Ps * p.A;
        bP = nbP;
        bAc = nbA;
        bDc = nbD;
      }
    }
  }
  if (flags) atomicOr(err, flags);
}

// ---- deterministic float64 sum ---------------------------------------------------------
constexpr int SUM_BLOCKS = VR_SUM_PARTIALS;
constexpr int SUM_THREADS = 256;

__global__ void k_sum_partial(const double* __restrict__ x, int64_t n, double* partial) {
  __shared__ double sh[SUM_THREADS];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)SUM_THREADS + threadIdx.x; i < n;
       i += (int64_t)SUM_BLOCKS * SUM_THREADS)
    acc += x[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = SUM_THREADS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_sum_final(const double* partial, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < SUM_BLOCKS; ++i) acc += partial[i];
    out[0] = acc;
  }
}

// ---- Adam ------------------------------------------------------------------------------
__global__ void k_adam(float4* __restrict__ p, const float4* __restrict__ g, float4* __restrict__ m,
                       float4* __restrict__ v, int64_t n4, float lr, float b1, float b2, float eps,
                       float bc1, float bc2, const int32_t* __restrict__ err) {
  if (err && *err) return;  // the step flagged an error: no update (vr_capi.h)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = p[i], gg = g[i], mm = m[i], vv = v[i];
    float* pa = &pp.x;
    float* ga = &gg.x;
    float* ma = &mm.x;
    float* va = &vv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ma[k] = b1 * ma[k] + (1.f - b1) * ga[k];
      va[k] = b2 * va[k] + (1.f - b2) * ga[k] * ga[k];
      pa[k] -= lr * (ma[k] / bc1) / (sqrtf(va[k] / bc2) + eps);
    }
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
  }
}

__global__ void k_adam_tail(float* p, const float* g, float* m, float* v, int64_t lo, int64_t n,
                            float lr, float b1, float b2, float eps, float bc1, float bc2,
                            const int32_t* __restrict__ err) {
  if (err && *err) return;
  for (int64_t i = lo + threadIdx.x; i < n; i += blockDim.x) {
    m[i] = b1 * m[i] + (1.f - b1) * g[i];
    v[i] = b2 * v[i] + (1.f - b2) * g[i] * g[i];
    p[i] -= lr * (m[i] / bc1) / (sqrtf(v[i] / bc2) + eps);
  }
}

__global__ void k_cast_f16(const float* __restrict__ src, __half* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2half_rn(src[i]);
}


// ---- lane-serial K4 (segwalk.cuh): K consecutive samples per lane ------------------------
// Per sample, the reference's own arithmetic (composite_samples quadrature.py:152-154):
// alpha = 1 - exp(-sigma delta), keep = 1 - alpha — one exp per sample.
constexpr int K4_LANE = 4;  // samples per lane (a chunk is 128 samples)

struct K4In {
  double a[K4_LANE], b[K4_LANE];
  float4 v[K4_LANE];
};

__device__ __forceinline__ void k4_load(K4In& in, const double* __restrict__ t0,
                                        const double* __restrict__ t1,
                                        const float4* __restrict__ sr, int64_t s0, int cnt) {
  // zero, then predicated loads straight into the registers (no select that would wait
  // for the loads here: they are consumed one chunk later)
#pragma unroll
  for (int k = 0; k < K4_LANE; ++k) {
    in.a[k] = in.b[k] = 0.0;
    in.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int k = 0; k < K4_LANE; ++k) {
    if (k < cnt) {
      in.a[k] = __ldg(t0 + s0 + k);
      in.b[k] = __ldg(t1 + s0 + k);
      in.v[k] = __ldg(sr + s0 + k);
    }
  }
}

__device__ __forceinline__ void keep_alpha(double sigma, double dlt, double& keep,
                                           double& alpha) {
  alpha = 1.0 - exp(-(sigma * dlt));
  keep = 1.0 - alpha;
}

__device__ __forceinline__ void k4_emit(float4* __restrict__ packets, double* __restrict__ seg_tot,
                                        const int32_t* __restrict__ seg_first, int64_t seg,
                                        const Comp& c) {
  packets[2 * seg] = make_float4((float)c.T, (float)c.C0, (float)c.C1, (float)c.C2);
  packets[2 * seg + 1] =
      make_float4((float)c.A, (float)c.D, (float)c.L, order_bits(seg_first[seg]));
  if (seg_tot) {  // float64 totals for the backward
    double* st = seg_tot + SEG_TOT * seg;
    st[0] = c.T;
    st[1] = c.C0;
    st[2] = c.C1;
    st[3] = c.C2;
    st[4] = c.A;
    st[5] = c.D;
    st[6] = c.L;
  }
}

// TMA staging (tma.cuh): per warp two chunk buffers {t0, t1: 65 rows of two float64 from
// the even sample at or below the chunk's first, sig_rgb [128] float4}, one mbarrier each
constexpr int K4_CHUNK = 32 * K4_LANE;
constexpr int K4_PAIRS = K4_CHUNK / 2 + 1;
constexpr uint32_t K4_TB = (K4_PAIRS * 16 + 127) / 128 * 128;  // one t buffer, 128-aligned
constexpr uint32_t K4_BUF = 2 * K4_TB + K4_CHUNK * 16;
constexpr uint32_t K4_TMA_SMEM = SEG_WARPS * 2 * K4_BUF + 128;  // + alignment slack
struct K4Maps {
  CUtensorMap t0, t1, sr;
};

// lane 0: the chunk at sample `base` into buffer b of this warp
__device__ __forceinline__ void k4_issue(uint8_t* wbuf, uint64_t* bars, int b, int64_t base,
                                         const K4Maps& maps) {
  uint8_t* dst = wbuf + b * K4_BUF;
  tma::fence_proxy_async();
  tma::expect_tx(&bars[b], 2 * K4_PAIRS * 16 + K4_CHUNK * 16);
  tma::load_2d(dst, &maps.t0, 0, (int32_t)(base >> 1), &bars[b]);
  tma::load_2d(dst + K4_TB, &maps.t1, 0, (int32_t)(base >> 1), &bars[b]);
  tma::load_2d(dst + 2 * K4_TB, &maps.sr, 0, (int32_t)base, &bars[b]);
}

__device__ __forceinline__ void k4_from_smem(K4In& in, const uint8_t* buf, int lane, int cnt,
                                             int64_t base) {
  const double* a = reinterpret_cast<const double*>(buf) + (base & 1);
  const double* b = reinterpret_cast<const double*>(buf + K4_TB) + (base & 1);
  const float4* v = reinterpret_cast<const float4*>(buf + 2 * K4_TB);
#pragma unroll
  for (int k = 0; k < K4_LANE; ++k) {
    const bool ok = k < cnt;
    in.a[k] = ok ? a[K4_LANE * lane + k] : 0.0;
    in.b[k] = ok ? b[K4_LANE * lane + k] : 0.0;
    in.v[k] = ok ? v[K4_LANE * lane + k] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

template <bool TMA>
__global__ void __launch_bounds__(SEG_WARPS * 32, 2)  // (3 blocks: spills, 5.9 -> 8.2 ms)
    k_segment_fwd_ls(const double* __restrict__ t0, const double* __restrict__ t1,
                     const float4* __restrict__ sr, const int64_t* __restrict__ off,
                     const int32_t* __restrict__ seg_first, const double* __restrict__ ray_te,
                     int64_t n_rays, int64_t n_segs, float4* __restrict__ packets,
                     double* __restrict__ seg_tot, const __grid_constant__ K4Maps maps) {
  __shared__ int64_t s_off_all[SEG_WARPS][33];
  __shared__ double s_te_all[SEG_WARPS][32];
  __shared__ uint64_t s_bar[SEG_WARPS][2];
  extern __shared__ __align__(128) uint8_t k4_dyn[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t* O = s_off_all[wid];
  double* TE = s_te_all[wid];
  // TMA destinations 128-byte aligned (the dynamic region follows the static arrays)
  uint8_t* dyn = k4_dyn + ((128 - (tma::smem_addr(k4_dyn) & 127)) & 127);
  uint8_t* wbuf = dyn + wid * 2 * K4_BUF;
  uint64_t* bars = s_bar[wid];
  uint32_t cc = 0;  // this warp's chunks so far: buffer cc & 1, its (cc >> 1)-th use
  if (TMA) {
    if (tma::elect_one()) {
      tma::mbar_init(&bars[0], 1);
      tma::mbar_init(&bars[1], 1);
      tma::fence_init();
    }
    __syncwarp();
  }
  const int64_t n_groups = ceil_div(n_segs, 32);
  const bool narrow = n_segs < INT32_MAX;
  const int64_t gstep = (int64_t)gridDim.x * SEG_WARPS;
  // TMA: the next group's offsets and entry depths are loaded into registers while this
  // group is walked, and its first chunk's copies are issued with this group's last chunk,
  // so a group starts without a memory round trip
  GroupPrefetch pf;
  double te_n = 0.0;
  bool first_issued = false;
  if (TMA) {
    const int64_t g0 = (int64_t)blockIdx.x * SEG_WARPS + wid;
    pf.load(off, g0, n_groups, n_segs, lane);
    te_n = lane < pf.nseg ? __ldg(ray_te + seg_ray(pf.seg0 + lane, n_rays, narrow)) : 0.0;
  }
  for (int64_t grp = (int64_t)blockIdx.x * SEG_WARPS + wid; grp < n_groups; grp += gstep) {
    const int64_t seg0 = grp * 32;
    const int nseg = (int)min((int64_t)32, n_segs - seg0);
    __syncwarp();  // the previous group's readers are done with O / TE
    if (TMA) {
      pf.stage(O, lane);
      TE[lane] = te_n;
      __syncwarp();
      pf.load(off, grp + gstep, n_groups, n_segs, lane);
      te_n = lane < pf.nseg ? __ldg(ray_te + seg_ray(pf.seg0 + lane, n_rays, narrow)) : 0.0;
    } else {
      stage_offsets(off, seg0, nseg, lane, O);
      TE[lane] = lane < nseg ? ray_te[seg_ray(seg0 + lane, n_rays, narrow)] : 0.0;
      __syncwarp();
    }
    const int64_t s_beg = O[0], s_end = O[nseg];
    if (lane < nseg && O[lane] == O[lane + 1]) {  // empty segment: identity packet
      packets[2 * (seg0 + lane)] = make_float4(1.f, 0.f, 0.f, 0.f);
      packets[2 * (seg0 + lane) + 1] = make_float4(0.f, 0.f, 0.f, order_bits(INT32_MAX));
    }
    Comp carry = comp_id();
    K4In nxt;
    if (TMA) {
      if (!first_issued && s_beg < s_end && tma::elect_one())
        k4_issue(wbuf, bars, cc & 1, s_beg, maps);
      first_issued = false;
    } else {
      const LaneSpan sp = lane_span<K4_LANE>(O, nseg, s_beg, s_end, lane);
      k4_load(nxt, t0, t1, sr, sp.s0, sp.cnt);
    }
    for (int64_t base = s_beg; base < s_end; base += K4_CHUNK) {
      const LaneSpan sp = lane_span<K4_LANE>(O, nseg, base, s_end, lane);
      K4In in;
      if (TMA) {  // the next chunk's copies (or the next group's first), then this chunk's
        if (base + K4_CHUNK < s_end) {
          if (tma::elect_one()) k4_issue(wbuf, bars, (cc + 1) & 1, base + K4_CHUNK, maps);
        } else if (pf.nseg > 0) {
          const int64_t nb = __shfl_sync(0xffffffffu, pf.o, 0);
          const int64_t ne = pf.nseg < 32 ? __shfl_sync(0xffffffffu, pf.o, pf.nseg)
                                          : __shfl_sync(0xffffffffu, pf.o32, 0);
          if (nb < ne) {
            if (tma::elect_one()) k4_issue(wbuf, bars, (cc + 1) & 1, nb, maps);
            first_issued = true;
          }
        }
        tma::wait(&bars[cc & 1], (cc >> 1) & 1);
        k4_from_smem(in, wbuf + (cc & 1) * K4_BUF, lane, sp.cnt, base);
        __syncwarp();  // every lane has read the buffer before it is refilled
        ++cc;
      } else {
        in = nxt;
        // next chunk's inputs (loads only; used one chunk later)
        const LaneSpan sn = lane_span<K4_LANE>(O, nseg, base + K4_CHUNK, s_end, lane);
        k4_load(nxt, t0, t1, sr, sn.s0, sn.cnt);
      }
      Comp head = comp_id(), cur = comp_id();
      bool head_done = false;
      int seg = sp.sf;
      // the lane's exps first (independent: ILP), then the serial fold
      double kp[K4_LANE], al[K4_LANE];
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k)
        keep_alpha((double)in.v[k].x, in.b[k] - in.a[k], kp[k], al[k]);
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        if (k < sp.cnt) {
          const int64_t s = sp.s0 + k;
          while (s >= O[seg + 1]) {  // the segment ended inside this lane
            if (!head_done) {
              head = cur;
              head_done = true;
            } else if (O[seg] < O[seg + 1]) {  // (empty segments have their identity)
              k4_emit(packets, seg_tot, seg_first, seg0 + seg, cur);
            }
            ++seg;
            cur = comp_id();
          }
          comp_push(cur, kp[k], al[k], in.v[k], sample_mid(in.a[k], in.b[k]) - TE[seg]);
        }
      }
      const bool closed = sp.cnt > 0 && O[seg + 1] == sp.s0 + sp.cnt;
      const bool single = !head_done;  // one segment piece in this lane
      if (single) head = cur;
      else if (closed) k4_emit(packets, seg_tot, seg_first, seg0 + seg, cur);
      // the piece open at the lane's end enters the cross-lane scan; a piece that started
      // in an earlier lane (or chunk) continues its predecessors'
      Comp e = cur;
      bool f = !(single && sp.open_left);
      if (sp.cnt == 0) {
        e = comp_id();
        f = false;
      }
      if (lane == 0 && sp.open_left && single) {
        e = comp_cat(carry, e);
        f = true;
      }
      const Comp S = lane_seg_scan(e, f, lane, comp_cat, comp_shfl_up);
      Comp X = comp_shfl_up(S, 1);
      if (lane == 0) X = carry;
      // the head segment closes in this lane: prefix from the lanes (chunks) before
      if (sp.cnt > 0 && (!single || closed))
        k4_emit(packets, seg_tot, seg_first, seg0 + sp.sf, sp.open_left ? comp_cat(X, head) : head);
      carry = comp_shfl(S, 31);
    }
  }
}

// T only (the proposal fields' segment transmittance): the same walk and fold order as
// k_segment_fwd_ls, so T[seg] equals the full packet's T bit for bit.
__global__ void __launch_bounds__(SEG_WARPS * 32)
    k_segment_T_ls(const double* __restrict__ t0, const double* __restrict__ t1,
                   const float4* __restrict__ sr, const int64_t* __restrict__ off,
                   int64_t n_segs, float* __restrict__ T_out) {
  __shared__ int64_t s_off_all[SEG_WARPS][33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t* O = s_off_all[wid];
  const float* sigma = reinterpret_cast<const float*>(sr);
  const int64_t n_groups = ceil_div(n_segs, 32);
  auto mul = [](double a, double b) { return a * b; };
  auto up = [](double a, int o) { return __shfl_up_sync(0xffffffffu, a, o); };
  const int64_t gstep = (int64_t)gridDim.x * SEG_WARPS;
  GroupPrefetch pf;
  pf.load(off, (int64_t)blockIdx.x * SEG_WARPS + wid, n_groups, n_segs, lane);
  for (int64_t grp = (int64_t)blockIdx.x * SEG_WARPS + wid; grp < n_groups; grp += gstep) {
    const int64_t seg0 = grp * 32;
    const int nseg = (int)min((int64_t)32, n_segs - seg0);
    __syncwarp();
    pf.stage(O, lane);
    pf.load(off, grp + gstep, n_groups, n_segs, lane);
    const int64_t s_beg = O[0], s_end = O[nseg];
    if (lane < nseg && O[lane] == O[lane + 1]) T_out[seg0 + lane] = 1.f;
    double carry = 1.0;
    for (int64_t base = s_beg; base < s_end; base += 32 * K4_LANE) {
      const LaneSpan sp = lane_span<K4_LANE>(O, nseg, base, s_end, lane);
      double a[K4_LANE], b[K4_LANE];
      float sg[K4_LANE];
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        a[k] = b[k] = 0.0;
        sg[k] = 0.f;
      }
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        if (k < sp.cnt) {
          a[k] = __ldg(t0 + sp.s0 + k);
          b[k] = __ldg(t1 + sp.s0 + k);
          sg[k] = __ldg(sigma + 4 * (sp.s0 + k));
        }
      }
      double head = 1.0, cur = 1.0;
      bool head_done = false;
      int seg = sp.sf;
      double kp[K4_LANE];
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        double al;
        keep_alpha((double)sg[k], b[k] - a[k], kp[k], al);
      }
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        if (k < sp.cnt) {
          const int64_t s = sp.s0 + k;
          while (s >= O[seg + 1]) {
            if (!head_done) {
              head = cur;
              head_done = true;
            } else if (O[seg] < O[seg + 1]) {
              T_out[seg0 + seg] = (float)cur;
            }
            ++seg;
            cur = 1.0;
          }
          cur *= kp[k];
        }
      }
      const bool closed = sp.cnt > 0 && O[seg + 1] == sp.s0 + sp.cnt;
      const bool single = !head_done;
      if (single) head = cur;
      else if (closed) T_out[seg0 + seg] = (float)cur;
      double e = cur;
      bool f = !(single && sp.open_left);
      if (sp.cnt == 0) {
        e = 1.0;
        f = false;
      }
      if (lane == 0 && sp.open_left && single) {
        e = carry * e;
        f = true;
      }
      const double S = lane_seg_scan(e, f, lane, mul, up);
      double X = __shfl_up_sync(0xffffffffu, S, 1);
      if (lane == 0) X = carry;
      if (sp.cnt > 0 && (!single || closed))
        T_out[seg0 + sp.sf] = (float)(sp.open_left ? X * head : head);
      carry = __shfl_sync(0xffffffffu, S, 31);
    }
  }
}

// Backward from the forward's float64 segment totals.  Per sample j of a segment with
// packet adjoints (bT, bC, bA, bD, bL):
//   v_j = bC.c_j + bA + bD m_j + bL g_j,  g_j = 2 (m_j a_<j - d_<j + d_>j - m_j a_>j)
//   dL/ds_j = -bT T + T_{j+1} v_j - (V - sum_{i<=j} w_i v_i),  V = sum_i w_i v_i
// Walk 1 folds the prefix state (T, A, D) per lane piece; a cross-lane scan gives each
// lane's incoming prefix; walk 2 forms the per-sample terms and the lane pieces' sums of
// w v; a second cross-lane scan gives their incoming sums; walk 3 writes the gradients.
struct K4Seg {
  float bC0, bC1, bC2, bA, bD, bL;
  double te, A, Dt, V, bTT;
};

__global__ void __launch_bounds__(SEG_WARPS * 32, 2)
    k_segment_bwd_ls(const double* __restrict__ t0, const double* __restrict__ t1,
                     const float4* __restrict__ sr, const int64_t* __restrict__ off,
                     const double* __restrict__ ray_te, int64_t n_rays, int64_t n_segs,
                     const float4* __restrict__ dpk, const double* __restrict__ seg_tot,
                     float4* __restrict__ dsr) {
  __shared__ int64_t s_off_all[SEG_WARPS][33];
  __shared__ K4Seg s_seg_all[SEG_WARPS][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t* O = s_off_all[wid];
  K4Seg* SG = s_seg_all[wid];
  const int64_t n_groups = ceil_div(n_segs, 32);
  auto add = [](double a, double b) { return a + b; };
  auto up = [](double a, int o) { return __shfl_up_sync(0xffffffffu, a, o); };
  const bool narrow = n_segs < INT32_MAX;
  for (int64_t grp = (int64_t)blockIdx.x * SEG_WARPS + wid; grp < n_groups;
       grp += (int64_t)gridDim.x * SEG_WARPS) {
    const int64_t seg0 = grp * 32;
    const int nseg = (int)min((int64_t)32, n_segs - seg0);
    __syncwarp();
    stage_offsets(off, seg0, nseg, lane, O);
    const int64_t s_beg = O[0], s_end = O[nseg];
    if (s_beg == s_end) continue;
    if (lane < nseg && O[lane] < O[lane + 1]) {
      const int64_t my = seg0 + lane;
      const float4 g0 = dpk[2 * my], g1 = dpk[2 * my + 1];
      const double* st = seg_tot + SEG_TOT * my;
      const double Tn = st[0], c0 = st[1], c1 = st[2], c2 = st[3], a = st[4], d = st[5],
                   l = st[6];
      K4Seg q;
      q.bC0 = g0.y;
      q.bC1 = g0.z;
      q.bC2 = g0.w;
      q.bA = g1.x;
      q.bD = g1.y;
      q.bL = g1.z;
      q.te = ray_te[seg_ray(my, n_rays, narrow)];
      q.A = a;
      q.Dt = d;
      q.V = (double)g0.y * c0 + (double)g0.z * c1 + (double)g0.w * c2 + (double)g1.x * a +
            (double)g1.y * d + 2.0 * (double)g1.z * l;
      q.bTT = (double)g0.x * Tn;
      SG[lane] = q;
    }
    __syncwarp();
    Pre pcarry = pre_id();
    double ucarry = 0.0;
    K4In nxt;
    {
      const LaneSpan sp = lane_span<K4_LANE>(O, nseg, s_beg, s_end, lane);
      k4_load(nxt, t0, t1, sr, sp.s0, sp.cnt);
    }
    for (int64_t base = s_beg; base < s_end; base += 32 * K4_LANE) {
      const LaneSpan sp = lane_span<K4_LANE>(O, nseg, base, s_end, lane);
      const K4In in = nxt;
      {
        const LaneSpan sn = lane_span<K4_LANE>(O, nseg, base + 32 * K4_LANE, s_end, lane);
        k4_load(nxt, t0, t1, sr, sn.s0, sn.cnt);
      }
      double keep[K4_LANE], alpha[K4_LANE];
      int sid[K4_LANE];
      // walk 1: prefix state of the lane's pieces
      Pre cur = pre_id();
      int seg = sp.sf;
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        keep[k] = 1.0;
        alpha[k] = 0.0;
        sid[k] = seg;
        if (k < sp.cnt) {
          const int64_t s = sp.s0 + k;
          while (s >= O[seg + 1]) {
            ++seg;
            cur = pre_id();
          }
          sid[k] = seg;
          // (in the fold, not ahead of it: the backward spills with the exps hoisted)
          keep_alpha((double)in.v[k].x, in.b[k] - in.a[k], keep[k], alpha[k]);
          const double m = sample_mid(in.a[k], in.b[k]) - SG[seg].te;
          const double w = cur.T * alpha[k];
          cur.A += w;
          cur.D += w * m;
          cur.T *= keep[k];
        }
      }
      const bool single = seg == sp.sf;
      Pre e = cur;
      bool f = !(single && sp.open_left);
      if (sp.cnt == 0) {
        e = pre_id();
        f = false;
      }
      if (lane == 0 && sp.open_left && single) {
        e = pre_cat(pcarry, e);
        f = true;
      }
      const Pre S = lane_seg_scan(e, f, lane, pre_cat, pre_shfl_up);
      Pre X = pre_shfl_up(S, 1);
      if (lane == 0) X = pcarry;
      pcarry = pre_shfl(S, 31);
      // walk 2: per-sample terms, lane-local running sums of w v per piece
      double r[K4_LANE], ul[K4_LANE], wk[K4_LANE];
      Pre q = sp.open_left ? X : pre_id();
      double u = 0.0;
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        r[k] = ul[k] = wk[k] = 0.0;
        if (k < sp.cnt) {
          if (k > 0 && sid[k] != sid[k - 1]) {
            q = pre_id();
            u = 0.0;
          }
          const K4Seg& g = SG[sid[k]];
          const double m = sample_mid(in.a[k], in.b[k]) - g.te;
          const double w = q.T * alpha[k];
          const double a_incl = q.A + w, d_incl = q.D + w * m;
          const double gk = 2.0 * (m * q.A - q.D + (g.Dt - d_incl) - m * (g.A - a_incl));
          const double v = (double)g.bC0 * in.v[k].y + (double)g.bC1 * in.v[k].z +
                           (double)g.bC2 * in.v[k].w + (double)g.bA + (double)g.bD * m +
                           (double)g.bL * gk;
          const double Tn = q.T * keep[k];
          u += w * v;
          ul[k] = u;
          r[k] = -g.bTT + Tn * v - g.V;
          wk[k] = w;
          q.T = Tn;
          q.A = a_incl;
          q.D = d_incl;
        }
      }
      double eu = u;
      bool fu = !(single && sp.open_left);
      if (sp.cnt == 0) {
        eu = 0.0;
        fu = false;
      }
      if (lane == 0 && sp.open_left && single) {
        eu = ucarry + eu;
        fu = true;
      }
      const double SU = lane_seg_scan(eu, fu, lane, add, up);
      double XU = __shfl_up_sync(0xffffffffu, SU, 1);
      if (lane == 0) XU = ucarry;
      ucarry = __shfl_sync(0xffffffffu, SU, 31);
      // walk 3: dL/dsigma_j = delta_j dL/ds_j, dL/dc_j = w_j bC
#pragma unroll
      for (int k = 0; k < K4_LANE; ++k) {
        if (k < sp.cnt) {
          const bool in_head = sid[k] == sp.sf && sp.open_left;
          const double ds = r[k] + (in_head ? XU : 0.0) + ul[k];
          const K4Seg& g = SG[sid[k]];
          const double dlt = in.b[k] - in.a[k];
          __stcs(dsr + sp.s0 + k, make_float4((float)(ds * dlt), (float)(wk[k] * g.bC0),
                                             (float)(wk[k] * g.bC1), (float)(wk[k] * g.bC2)));
        }
      }
    }
  }
}

// K4 kernels: lane-serial walks (default) or the per-sample grouped scans (VR_K4_WALK=grp,
// kept for A/B measurement and as the backward without forward totals)
// tensor maps of the walks' inputs (n_samples: the arrays' length; 0 = unknown, no TMA);
// VR_K4_TMA=0 keeps the per-lane loads
static bool k4_maps(K4Maps& m, const double* t0, const double* t1, const float* sr,
                    int64_t n_samples) {
  static const bool on = [] {
    const char* e = getenv("VR_K4_TMA");
    return !(e && strcmp(e, "0") == 0);
  }();
  memset(&m, 0, sizeof(m));
  if (!on || n_samples <= 0 || n_samples > INT32_MAX) return false;
  return tma::encode_pairs(&m.t0, t0, (uint64_t)n_samples, K4_PAIRS) &&
         tma::encode_pairs(&m.t1, t1, (uint64_t)n_samples, K4_PAIRS) &&
         tma::encode_rows(&m.sr, sr, (uint64_t)n_samples, 4, K4_CHUNK);
}
static PacketSrc pk_source(const float* pk, const float* extra, const float* rec,
                           const int32_t* index, int width) {
  PacketSrc s;
  s.pk = reinterpret_cast<const float4*>(pk);
  s.extra = extra;
  s.rec = rec;
  s.index = index;
  s.width = width;
  return s;
}
static bool k4_lane_serial() {
  static const bool ls = [] {
    const char* e = getenv("VR_K4_WALK");
    return !(e && strcmp(e, "grp") == 0);
  }();
  return ls;
}

}  // namespace vr

using namespace vr;

extern "C" int vr_segment_fwd(const double* t0, const double* t1, const float* sr,
                              const int64_t* off, const int32_t* seg_first, const double* ray_te,
                              int64_t n_rays, int32_t region_cnt, float* packets,
                              double* seg_totals, int32_t* err, int64_t n_samples,
                              void* stream) {
  (void)err;
  if (n_rays < 0 || region_cnt < 1 || region_cnt > VR_MAX_REGIONS) {
    set_error("vr_segment_fwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n_segs = n_rays * region_cnt;
  if (n_segs == 0) return VR_OK;
  K4Maps maps;
  const bool use_tma = k4_lane_serial() && k4_maps(maps, t0, t1, sr, n_samples);
  const int grid = grid_for(ceil_div(n_segs, 32 * SEG_WARPS), 1, 8);
  if (use_tma) {
    cudaFuncSetAttribute(k_segment_fwd_ls<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)K4_TMA_SMEM);
    k_segment_fwd_ls<true><<<grid, SEG_WARPS * 32, K4_TMA_SMEM, (cudaStream_t)stream>>>(
        t0, t1, reinterpret_cast<const float4*>(sr), off, seg_first, ray_te, n_rays, n_segs,
        reinterpret_cast<float4*>(packets), seg_totals, maps);
  } else if (k4_lane_serial())
    k_segment_fwd_ls<false><<<grid, SEG_WARPS * 32, 0, (cudaStream_t)stream>>>(
        t0, t1, reinterpret_cast<const float4*>(sr), off, seg_first, ray_te, n_rays, n_segs,
        reinterpret_cast<float4*>(packets), seg_totals, maps);
  else
    k_segment_fwd_grp<<<grid_for(ceil_div(n_segs, 32 * SEG_WARPS), 1, 8), SEG_WARPS * 32, 0,
                        (cudaStream_t)stream>>>(t0, t1, reinterpret_cast<const float4*>(sr), off,
                                                seg_first, ray_te, n_rays, n_segs,
                                                reinterpret_cast<float4*>(packets), seg_totals);
  return check_launch("vr_segment_fwd");
}

extern "C" int vr_segment_transmittance(const double* t0, const double* t1, const float* sr,
                                        const int64_t* off, int64_t n_rays, int32_t region_cnt,
                                        float* T_out, void* stream) {
  if (n_rays < 0 || region_cnt < 1 || region_cnt > VR_MAX_REGIONS || !T_out) {
    set_error("vr_segment_transmittance: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n_segs = n_rays * region_cnt;
  if (n_segs == 0) return VR_OK;
  if (k4_lane_serial())
    k_segment_T_ls<<<grid_for(ceil_div(n_segs, 32 * SEG_WARPS), 1, 8), SEG_WARPS * 32, 0,
                     (cudaStream_t)stream>>>(t0, t1, reinterpret_cast<const float4*>(sr), off,
                                             n_segs, T_out);
  else
    k_segment_T_grp<<<grid_for(ceil_div(n_segs, 32 * SEG_WARPS), 1, 8), SEG_WARPS * 32, 0,
                      (cudaStream_t)stream>>>(t0, t1, reinterpret_cast<const float4*>(sr), off,
                                              n_segs, T_out);
  return check_launch("vr_segment_transmittance");
}

extern "C" int vr_segment_bwd(const double* t0, const double* t1, const float* sr,
                              const int64_t* off, const double* ray_te, int64_t n_rays,
                              int32_t region_cnt, const float* dpk, const double* seg_totals,
                              float* dsr, void* stream) {
  if (n_rays < 0 || region_cnt < 1 || region_cnt > VR_MAX_REGIONS) {
    set_error("vr_segment_bwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n_segs = n_rays * region_cnt;
  if (n_segs == 0) return VR_OK;
  if (k4_lane_serial() && seg_totals)
    k_segment_bwd_ls<<<grid_for(ceil_div(n_segs, 32 * SEG_WARPS), 1, 8), SEG_WARPS * 32, 0,
                       (cudaStream_t)stream>>>(t0, t1, reinterpret_cast<const float4*>(sr), off,
                                               ray_te, n_rays, n_segs,
                                               reinterpret_cast<const float4*>(dpk), seg_totals,
                                               reinterpret_cast<float4*>(dsr));
  else
    k_segment_bwd_grp<<<grid_for(ceil_div(n_segs, 32 * SEG_WARPS), 1, 8), SEG_WARPS * 32, 0,
                        (cudaStream_t)stream>>>(t0, t1, reinterpret_cast<const float4*>(sr), off,
                                                ray_te, n_rays, n_segs,
                                                reinterpret_cast<const float4*>(dpk), seg_totals,
                                                reinterpret_cast<float4*>(dsr));
  return check_launch("vr_segment_bwd");
}

extern "C" int vr_global_fwd(const float* pk, int32_t n_regions, int64_t n_rays,
                             const double* ray_te, const float* bg, int32_t clip_bg, float* out,
                             int32_t* err, void* stream) {
  if (n_regions < 1 || n_regions > VR_MAX_REGIONS || n_rays < 0 || !bg || !err) {
    set_error("vr_global_fwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  k_global<false><<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(
      pk_source(pk, nullptr, nullptr, nullptr, 0), n_regions, n_rays, ray_te, bg[0], bg[1],
      bg[2], clip_bg, nullptr, 0.f, 0, 0, out, nullptr, nullptr, err);
  return check_launch("vr_global_fwd");
}

extern "C" int vr_global_train(const float* pk, int32_t n_regions, int64_t n_rays,
                               const double* ray_te, const float* bg, const float* targets,
                               float lambda_dist, int32_t own_lo, int32_t own_cnt, float* out,
                               double* ray_loss, float* dpk, int32_t* err, void* stream) {
  if (n_regions < 1 || n_regions > VR_MAX_REGIONS || n_rays < 0 || !bg || !err || own_lo < 0 ||
      own_cnt < 1 || own_lo + own_cnt > n_regions) {
    set_error("vr_global_train: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  k_global<true><<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(
      pk_source(pk, nullptr, nullptr, nullptr, 0), n_regions, n_rays, ray_te, bg[0], bg[1],
      bg[2], 0, targets, lambda_dist, own_lo, own_cnt, out, ray_loss,
      reinterpret_cast<float4*>(dpk), err);
  return check_launch("vr_global_train");
}

extern "C" int vr_global_fwd_records(const float* recv, int32_t width, const int32_t* index,
                                     int32_t n_regions, int64_t n_rays, const double* ray_te,
                                     const float* bg, int32_t clip_bg, float* out, int32_t* err,
                                     void* stream) {
  if (n_regions < 1 || n_regions > VR_MAX_REGIONS || n_rays < 0 || !bg || !err ||
      (n_rays > 0 && (!recv || !index)) || (width != 9 && width != 10)) {
    set_error("vr_global_fwd_records: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  k_global<false><<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(
      pk_source(nullptr, nullptr, recv, index, width), n_regions, n_rays, ray_te, bg[0], bg[1],
      bg[2], clip_bg, nullptr, 0.f, 0, 0, out, nullptr, nullptr, err);
  return check_launch("vr_global_fwd_records");
}

extern "C" int vr_global_train_records(const float* recv, int32_t width, const int32_t* index,
                                       int32_t n_regions, int64_t n_rays, const double* ray_te,
                                       const float* bg, const float* targets, float lambda_dist,
                                       int32_t own_lo, int32_t own_cnt, float* out,
                                       double* ray_loss, float* dpk, int32_t* err, void* stream) {
  if (n_regions < 1 || n_regions > VR_MAX_REGIONS || n_rays < 0 || !bg || !err || own_lo < 0 ||
      own_cnt < 1 || own_lo + own_cnt > n_regions || (n_rays > 0 && (!recv || !index)) ||
      (width != 9 && width != 10)) {
    set_error("vr_global_train_records: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  k_global<true><<<grid_for(n_rays, 128), 128, 0, (cudaStream_t)stream>>>(
      pk_source(nullptr, nullptr, recv, index, width), n_regions, n_rays, ray_te, bg[0], bg[1],
      bg[2], 0, targets, lambda_dist, own_lo, own_cnt, out, ray_loss,
      reinterpret_cast<float4*>(dpk), err);
  return check_launch("vr_global_train_records");
}

// ---- sample-broadcast protocol: region-major <-> ray-major sample order ---------------
// Segment (k, r) occupies [off[k*R + r], off[k*R + r + 1]) in the region-major layout and
// [ray_off[r] + seg_first[k*R + r], ...) in the ray-major one (seg_first = index along the
// ray of the segment's first sample, so a ray's segments land in t order).  Warp per
// segment, lanes copy consecutive elements of ELEM bytes.
template <typename T>
__global__ void k_segment_permute(const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ seg_first,
                                  const int64_t* __restrict__ ray_off, int64_t n_rays,
                                  int64_t n_segs, const T* __restrict__ src, T* __restrict__ dst,
                                  int to_ray_major) {
  const int lane = threadIdx.x & 31;
  for (int64_t sg = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sg < n_segs;
       sg += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t b = off[sg], e = off[sg + 1];
    if (b == e) continue;
    const int64_t rm = ray_off[sg % n_rays] + seg_first[sg];
    for (int64_t j = lane; j < e - b; j += 32) {
      if (to_ray_major)
        dst[rm + j] = src[b + j];
      else
        dst[b + j] = src[rm + j];
    }
  }
}

extern "C" int vr_segment_permute(const int64_t* off, const int32_t* seg_first,
                                  const int64_t* ray_off, int64_t n_rays, int32_t n_regions,
                                  const void* src, void* dst, int32_t elem_bytes,
                                  int32_t to_ray_major, void* stream) {
  if (n_rays < 0 || n_regions < 1 || n_regions > VR_MAX_REGIONS ||
      (elem_bytes != 4 && elem_bytes != 8 && elem_bytes != 16)) {
    set_error("vr_segment_permute: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const int64_t n_segs = n_rays * n_regions;
  if (n_segs == 0) return VR_OK;
  const int grid = grid_for(ceil_div(n_segs, 8), 1, 16);
  cudaStream_t s = (cudaStream_t)stream;
  if (elem_bytes == 4)
    k_segment_permute<<<grid, 256, 0, s>>>(off, seg_first, ray_off, n_rays, n_segs,
                                           (const float*)src, (float*)dst, to_ray_major);
  else if (elem_bytes == 8)
    k_segment_permute<<<grid, 256, 0, s>>>(off, seg_first, ray_off, n_rays, n_segs,
                                           (const double*)src, (double*)dst, to_ray_major);
  else
    k_segment_permute<<<grid, 256, 0, s>>>(off, seg_first, ray_off, n_rays, n_segs,
                                           (const float4*)src, (float4*)dst, to_ray_major);
  return check_launch("vr_segment_permute");
}

// ---- sparse packet exchange ---------------------------------------------------------
// Only the packets of non-empty segments travel (a ray crosses ~3 of c3's 8 regions and
// ~1.6 of c4's): record = {global slab index (int32 bits), 8 packet floats[, proposal T]};
// row 0 of a rank's buffer holds its record count.  The receiver fills the dense
// [K][R][8] slab with identity packets (what K4 writes for an empty segment) and
// scatters the records, so K5 reads bit-identical slabs on every rank.
__global__ void k_packets_pack(const float4* __restrict__ pk, const float* __restrict__ extra,
                               const int32_t* __restrict__ counts, int64_t n_segs,
                               int64_t n_rays, int region_lo, int width, float* out, int64_t cap,
                               int32_t* n_out, int32_t* err) {
  const int lane = threadIdx.x & 31;
  int flags = 0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n_segs;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t seg = base + lane;
    const bool live = seg < n_segs && counts[seg] > 0;
    const unsigned m = __ballot_sync(0xffffffffu, live);
    if (!m) continue;
    int32_t slot0 = 0;
    if (lane == 0) slot0 = atomicAdd(n_out, __popc(m));
    slot0 = __shfl_sync(0xffffffffu, slot0, 0);
    if (live) {
      const int64_t slot = 1 + slot0 + __popc(m & ((1u << lane) - 1u));
      if (slot > cap) {
        flags |= VR_FLAG_OVERFLOW;
      } else {
        float* rec = out + slot * width;
        const int64_t gidx = (int64_t)region_lo * n_rays + seg;
        const float4 a = pk[2 * seg], b = pk[2 * seg + 1];
        rec[0] = __int_as_float((int32_t)gidx);
        rec[1] = a.x; rec[2] = a.y; rec[3] = a.z; rec[4] = a.w;
        rec[5] = b.x; rec[6] = b.y; rec[7] = b.z; rec[8] = b.w;
        if (extra) rec[9] = extra[seg];
      }
    }
  }
  flags = (int)__reduce_or_sync(0xffffffffu, (unsigned)flags);
  if (flags && lane == 0) atomicOr(err, flags);
}

__global__ void k_packets_header(const int32_t* n_out, float* out) {
  out[0] = __int_as_float(*n_out);
}

__global__ void k_packets_identity(float4* __restrict__ slab, float* __restrict__ extra_slab,
                                   int64_t n_segs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_segs;
       i += (int64_t)gridDim.x * blockDim.x) {
    slab[2 * i] = make_float4(1.f, 0.f, 0.f, 0.f);
    slab[2 * i + 1] = make_float4(0.f, 0.f, 0.f, order_bits(INT32_MAX));
    if (extra_slab) extra_slab[i] = 1.f;
  }
}

__global__ void k_packets_unpack(const float* __restrict__ recv, int world, int64_t rows,
                                 int width, int64_t n_segs, float4* __restrict__ slab,
                                 float* __restrict__ extra_slab, int32_t* err) {
  int flags = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)world * rows;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rk = t / rows, i = t - rk * rows;
    const float* buf = recv + rk * rows * width;
    const int32_t n = __float_as_int(buf[0]);
    if (i == 0 || i > n) continue;
    if (n >= rows) {
      flags |= VR_FLAG_OVERFLOW;
      continue;
    }
    const float* rec = buf + i * width;
    const int64_t g = (int64_t)__float_as_int(rec[0]);
    if (g < 0 || g >= n_segs) {
      flags |= VR_FLAG_OVERFLOW;
      continue;
    }
    slab[2 * g] = make_float4(rec[1], rec[2], rec[3], rec[4]);
    slab[2 * g + 1] = make_float4(rec[5], rec[6], rec[7], rec[8]);
    if (extra_slab) extra_slab[g] = rec[9];
  }
  if (flags) atomicOr(err, flags);
}

extern "C" int vr_packets_pack(const float* packets, const float* extra, const int32_t* counts,
                               int64_t n_rays, int32_t region_lo, int32_t region_cnt, float* out,
                               int64_t capacity, int32_t* count_dev, int32_t* err,
                               void* stream) {
  if (n_rays < 0 || region_lo < 0 || region_cnt < 1 || capacity < 0 || !out || !count_dev ||
      !err || (int64_t)(region_lo + region_cnt) * n_rays > INT32_MAX) {
    set_error("vr_packets_pack: bad argument");
    return VR_ERR_BAD_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n_segs = n_rays * region_cnt;
  cudaMemsetAsync(count_dev, 0, sizeof(int32_t), s);
  if (n_segs > 0)
    k_packets_pack<<<grid_for(n_segs, 256), 256, 0, s>>>(
        (const float4*)packets, extra, counts, n_segs, n_rays, region_lo, extra ? 10 : 9, out,
        capacity, count_dev, err);
  k_packets_header<<<1, 1, 0, s>>>(count_dev, out);
  return check_launch("vr_packets_pack");
}

extern "C" int vr_packets_unpack(const float* recv, int32_t world, int64_t rows, int32_t width,
                                 int64_t n_rays, int32_t n_regions, float* slab,
                                 float* extra_slab, int32_t* err, void* stream) {
  if (world < 1 || rows < 1 || (width != 9 && width != 10) || (width == 10) != !!extra_slab ||
      n_rays < 0 || n_regions < 1 || n_regions > VR_MAX_REGIONS || !slab || !err) {
    set_error("vr_packets_unpack: bad argument");
    return VR_ERR_BAD_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n_segs = n_rays * n_regions;
  if (n_segs == 0) return VR_OK;
  k_packets_identity<<<grid_for(n_segs, 256), 256, 0, s>>>((float4*)slab, extra_slab, n_segs);
  k_packets_unpack<<<grid_for((int64_t)world * rows, 256), 256, 0, s>>>(
      recv, world, rows, width, n_segs, (float4*)slab, extra_slab, err);
  return check_launch("vr_packets_unpack");
}

// index[g] = the record slot (rank * rows + i) of segment g; -1 (memset) for empty segments
__global__ void k_packets_index(const float* __restrict__ recv, int world, int64_t rows,
                                int width, int64_t n_segs, int32_t* __restrict__ index,
                                int32_t* err) {
  int flags = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)world * rows;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rk = t / rows, i = t - rk * rows;
    const float* buf = recv + rk * rows * width;
    const int32_t n = __float_as_int(buf[0]);
    if (i == 0 || i > n) continue;
    if (n >= rows) {
      flags |= VR_FLAG_OVERFLOW;
      continue;
    }
    const int64_t g = (int64_t)__float_as_int(buf[i * width]);
    if (g < 0 || g >= n_segs) {
      flags |= VR_FLAG_OVERFLOW;
      continue;
    }
    index[g] = (int32_t)t;
  }
  if (flags) atomicOr(err, flags);
}

extern "C" int vr_packets_index(const float* recv, int32_t world, int64_t rows, int32_t width,
                                int64_t n_rays, int32_t n_regions, int32_t* index, int32_t* err,
                                void* stream) {
  if (world < 1 || rows < 1 || (width != 9 && width != 10) || n_rays < 0 || n_regions < 1 ||
      n_regions > VR_MAX_REGIONS || !index || !err || (int64_t)world * rows > INT32_MAX) {
    set_error("vr_packets_index: bad argument");
    return VR_ERR_BAD_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n_segs = n_rays * n_regions;
  if (n_segs == 0) return VR_OK;
  cudaMemsetAsync(index, 0xFF, (size_t)n_segs * sizeof(int32_t), s);
  k_packets_index<<<grid_for((int64_t)world * rows, 256), 256, 0, s>>>(recv, world, rows, width,
                                                                       n_segs, index, err);
  return check_launch("vr_packets_index");
}

extern "C" int vr_sum_f64(const double* x, int64_t n, double* out, double* ws, void* stream) {
  if (n < 0 || !out || !ws) {
    set_error("vr_sum_f64: bad argument");
    return VR_ERR_BAD_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  k_sum_partial<<<SUM_BLOCKS, SUM_THREADS, 0, s>>>(x, n, ws);
  k_sum_final<<<1, 32, 0, s>>>(ws, out);
  return check_launch("vr_sum_f64");
}

extern "C" int vr_adam_step(float* p, const float* g, float* m, float* v, int64_t n, float lr,
                            float b1, float b2, float eps, int32_t step, const int32_t* err,
                            void* stream) {
  if (n < 0 || step < 1) {
    set_error("vr_adam_step: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  const float bc1 = 1.f - powf(b1, (float)step), bc2 = 1.f - powf(b2, (float)step);
  const bool aligned = ((uintptr_t)p | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v) % 16 == 0;
  const int64_t n4 = aligned ? n / 4 : 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (n4)
    k_adam<<<grid_for(n4, 256), 256, 0, s>>>((float4*)p, (const float4*)g, (float4*)m,
                                             (float4*)v, n4, lr, b1, b2, eps, bc1, bc2, err);
  if (4 * n4 < n)
    k_adam_tail<<<1, 256, 0, s>>>(p, g, m, v, 4 * n4, n, lr, b1, b2, eps, bc1, bc2, err);
  return check_launch("vr_adam_step");
}

extern "C" int vr_cast_f32_f16(const float* src, void* dst, int64_t n, void* stream) {
  if (n < 0) {
    set_error("vr_cast_f32_f16: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_cast_f16<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, (__half*)dst, n);
  return check_launch("vr_cast_f32_f16");
}
