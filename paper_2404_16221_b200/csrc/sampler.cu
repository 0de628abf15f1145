// K1 — warp-per-ray ray/region intersection and per-segment sample generation.
//
// One warp owns one ray.  Lanes intersect the leaf boxes in parallel (lane per box),
// compact and sort the cut distances in shared memory, then walk the global dt
// grid 32 bins at a time (lane per bin), split each bin at the cuts, locate every
// sub-bin's midpoint and write it into its region's segment.  All geometry is
// float64 with explicit round-to-nearest intrinsics so the bin edges, midpoints
// and tile ids are bit-identical to the reference:
//   generate_samples    quadrature.py:66-88
//   split_at_planes     quadrature.py:91-114
//   tile_cut_distances  partitioner.py:195-206
//   locate_many         partitioner.py:177-192
//   participants        distsim.py:415-419
// Regions are contiguous along a ray (each leaf is an intersection of half-spaces
// whose predicates are monotone in t), so a sample's slot inside its segment is
// (index along the ray) - (index of the segment's first sample).
//
// Multi-rank: a rank owning a block of regions only walks the bins that can hold its own
// samples.  Rays missing the (slightly inflated) bounding box of its regions are skipped
// after the root slab test; for the others, the bins before the box are only counted (no
// owner lookup), so every sample keeps its global index along the ray and the result is
// bit-identical to sampling all regions and keeping the own ones.  (Callers asking for
// ray_part / ray_total — the reference's CommStats — get the full walk.)
//
// One walk instead of two (vr_sample_stage + vr_sample_compact): the count pass also
// writes every own piece into a staging buffer, in a slot range each ray reserves from
// its block's slice before walking (at most one piece per walked bin plus one per cut);
// after the scan of the counts a warp-per-ray copy moves the segments to their
// region-major slots.  The staging traffic (16 B written + 16 B read per sample) is a
// fraction of the second fp64 walk it replaces.  A block whose slice is too small reports
// it and the caller runs the fill pass instead.
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "common.cuh"

namespace vr {

constexpr int K1_WARPS = 4;
// 64 registers, 32 resident warps per SM (c3 one-walk stage: 72 registers 2.33 ms, 64
// 2.09, 48 2.49, 40 2.88 — fewer spill to the stack)
constexpr int K1_MIN_BLOCKS = 8;

struct K1Smem {
  VrTree tree;
  double cand[K1_WARPS][2 * VR_MAX_REGIONS];
  double cut[K1_WARPS][2 * VR_MAX_REGIONS];
  int candf[K1_WARPS][2 * VR_MAX_REGIONS];
  int cnt[K1_WARPS][VR_MAX_REGIONS];
  int first[K1_WARPS][VR_MAX_REGIONS];
  int64_t off[K1_WARPS][VR_MAX_REGIONS];
  int64_t end[K1_WARPS][VR_MAX_REGIONS];
  double own_mn[3], own_mx[3];  // inflated bounding box of the rank's regions
  unsigned long long stage_top; // staging slots reserved by this block
};

// Multi-rank prefilter, thread per ray: rays that miss the rank's inflated region box get
// their (empty) count-pass outputs here; the others are appended to ray_list for the
// warp-per-ray walk, which on a rank owning 1 of 8 regions then skips ~60 % of the warps.
__global__ void __launch_bounds__(256)
    k_sample_prefilter(const VrTree tree, const double* __restrict__ rays, int64_t stride,
                       int64_t n_rays, int region_lo, int region_cnt, int32_t* counts,
                       int32_t* seg_first, double* ray_te, int32_t* ray_list) {
  __shared__ double own_mn[3], own_mx[3];
  if (threadIdx.x < 3) {  // the same inflated box as k_sample<RESTRICT>
    const int a = threadIdx.x;
    double mn = INFINITY, mx = -INFINITY;
    for (int k = region_lo; k < region_lo + region_cnt; ++k) {
      mn = fmin(mn, tree.leaf_mn[k][a]);
      mx = fmax(mx, tree.leaf_mx[k][a]);
    }
    const double pad = 1e-9 * (1.0 + fmax(fabs(mn), fabs(mx)));
    own_mn[a] = mn - pad;
    own_mx[a] = mx + pad;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n_rays;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = base + lane;
    bool own = false;
    if (r < n_rays) {
      const RayD ray = load_ray(rays, stride, r);
      double te, tx, ta, tb;
      const bool hit = ray_box(ray, tree.root_mn, tree.root_mx, te, tx);
      own = ray_box(ray, own_mn, own_mx, ta, tb);
      if (!own) {
        for (int kk = 0; kk < region_cnt; ++kk) {
          const int64_t idx = (int64_t)kk * n_rays + r;
          counts[idx] = 0;
          seg_first[idx] = INT32_MAX;
        }
        ray_te[r] = hit ? te : 0.0;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, own);
    if (m) {
      int slot = 0;
      if (lane == 0) slot = atomicAdd(ray_list, __popc(m));
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (own) ray_list[1 + slot + __popc(m & ((1u << lane) - 1u))] = (int32_t)r;
    }
  }
}

// STAGE (count pass only): also write the own pieces to st0/st1 — block b owns slots
// [b * slice, (b + 1) * slice); sslot[r] + (index along the ray) is a piece's slot.
// stage_info[0] += slots reserved, stage_info[1] = max over blocks (the slice needed).
// the occupancy bit of a point in leaf g's grid (VrOccupancy in vr_capi.h)
__device__ __forceinline__ bool occupied(const VrOccupancy& occ, const VrTree& t, int g,
                                         const double p[3]) {
  const int G = occ.res;
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double u = ddiv(dsub(p[a], t.leaf_mn[g][a]), dsub(t.leaf_mx[g][a], t.leaf_mn[g][a]));
    const double x = fmin(fmax(floor(dmul(u, (double)G)), 0.0), (double)(G - 1));
    c[a] = (int)x;
  }
  const int64_t words = ((int64_t)G * G * G + 31) / 32;
  const int64_t idx = c[0] + (int64_t)G * (c[1] + (int64_t)G * c[2]);
  return (__ldg(occ.bits + (int64_t)g * words + (idx >> 5)) >> (idx & 31)) & 1u;
}

template <bool FILL, bool RESTRICT, bool STAGE>
__global__ void __launch_bounds__(K1_WARPS * 32, K1_MIN_BLOCKS)
    k_sample(const VrTree tree_param, const VrOccupancy occ, const double* __restrict__ rays,
             int64_t stride,
             int64_t n_rays, double dt, int region_lo, int region_cnt, int32_t* counts,
             int32_t* seg_first, double* ray_te, uint32_t* ray_part, int32_t* ray_total,
             const int64_t* __restrict__ offsets, double* t0o, double* t1o, int32_t* rido,
             int64_t capacity, int32_t* err, double* st0, double* st1, int64_t* sslot,
             int64_t slice, unsigned long long* stage_info,
             const int32_t* __restrict__ ray_list) {
  static_assert(!(FILL && STAGE), "staging is part of the count pass");
  __shared__ K1Smem sm;
  if (STAGE && threadIdx.x == 0) sm.stage_top = 0;
  {
    const uint64_t* src = reinterpret_cast<const uint64_t*>(&tree_param);
    uint64_t* dst = reinterpret_cast<uint64_t*>(&sm.tree);
    for (int i = threadIdx.x; i < (int)(sizeof(VrTree) / 8); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const VrTree& tree = sm.tree;
  constexpr bool restrict_own = RESTRICT;  // host: no ray_part / ray_total, not all regions
  if (RESTRICT && threadIdx.x < 3) {  // bounding box of the own regions, inflated far beyond rounding
    const int a = threadIdx.x;
    double mn = INFINITY, mx = -INFINITY;
    for (int k = region_lo; k < region_lo + region_cnt; ++k) {
      mn = fmin(mn, tree.leaf_mn[k][a]);
      mx = fmax(mx, tree.leaf_mx[k][a]);
    }
    const double pad = 1e-9 * (1.0 + fmax(fabs(mn), fabs(mx)));
    sm.own_mn[a] = mn - pad;
    sm.own_mx[a] = mx + pad;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int n_leaves = tree.n_leaves;
  // occupancy: a sample's index along the ray counts kept samples only, so the bins
  // before the own regions must be walked (their occupancy decides the indices)
  const bool use_occ = occ.bits != nullptr && occ.res > 0;
  double* cand = sm.cand[warp];
  double* cut = sm.cut[warp];
  int flags = 0;

  // ray_list (RESTRICT): [0] = n, then the rays k_sample_prefilter found to reach the own
  // box (the others' outputs are written there)
  const int64_t n_work = ray_list ? (int64_t)ray_list[0] : n_rays;
  for (int64_t i = (int64_t)blockIdx.x * K1_WARPS + warp; i < n_work;
       i += (int64_t)gridDim.x * K1_WARPS) {
    const int64_t r = ray_list ? (int64_t)ray_list[1 + i] : i;
    const RayD ray = load_ray(rays, stride, r);
    double te, tx;
    const bool hit = ray_box(ray, tree.root_mn, tree.root_mx, te, tx);
    double ta = te, tb = tx;  // t range that can hold own samples
    const bool own_hit = !restrict_own || ray_box(ray, sm.own_mn, sm.own_mx, ta, tb);
    if (!own_hit) {  // no own sample on this ray
      if (!FILL) {
        if (lane < region_cnt) {
          const int64_t idx = (int64_t)lane * n_rays + r;
          counts[idx] = 0;
          seg_first[idx] = INT32_MAX;
        }
        if (lane == 0) ray_te[r] = hit ? te : 0.0;
      }
      continue;
    }

    // --- leaf boxes: participation mask and candidate cut distances --------------
    uint32_t part = 0;
    int ncand = 0;
    for (int j0 = 0; j0 < n_leaves; j0 += 32) {
      const int j = j0 + lane;
      double a = 0.0, b = 0.0;
      bool h = false;
      if (j < n_leaves) h = ray_box(ray, tree.leaf_mn[j], tree.leaf_mx[j], a, b);
      part |= __ballot_sync(0xffffffffu, h) << j0;
      const bool ca = hit && h && te < a && a < tx;
      const bool cb = hit && h && te < b && b < tx;
      const unsigned ma = __ballot_sync(0xffffffffu, ca);
      const unsigned mb = __ballot_sync(0xffffffffu, cb);
      const unsigned below = (1u << lane) - 1u;
      if (ca) cand[ncand + __popc(ma & below)] = a;
      if (cb) cand[ncand + __popc(ma) + __popc(mb & below)] = b;
      ncand += __popc(ma) + __popc(mb);
    }
    __syncwarp();

    // --- sort + dedup the cuts (Python set semantics, sorted) ---------------------
    int* candf = sm.candf[warp];
    for (int i = lane; i < ncand; i += 32) {
      const double v = cand[i];
      int f = 1;
      for (int k = 0; k < i; ++k)
        if (cand[k] == v) f = 0;
      candf[i] = f;
    }
    __syncwarp();
    int ncut = 0;
    for (int i = 0; i < ncand; ++i) ncut += candf[i];
    for (int i = lane; i < ncand; i += 32) {
      if (candf[i]) {
        const double v = cand[i];
        int rank = 0;
        for (int k = 0; k < ncand; ++k) rank += (candf[k] && cand[k] < v) ? 1 : 0;
        cut[rank] = v;
      }
    }
    // per-ray region counters
    if (lane < region_cnt) {
      sm.cnt[warp][lane] = 0;
      sm.first[warp][lane] = INT32_MAX;
      if (FILL) {
        const int64_t idx = (int64_t)lane * n_rays + r;
        sm.first[warp][lane] = seg_first[idx];
        sm.off[warp][lane] = offsets[idx];
        sm.end[warp][lane] = offsets[idx + 1];
      }
    }
    __syncwarp();

    int total = 0;
    const double span = hit ? dsub(tx, te) : 0.0;
    if (hit && span > VR_SLIVER) {
      // --- global grid (quadrature.py:79-88) ---------------------------------------
      const double q = ddiv(span, dt);
      if (!(q < 1.0e9)) {
        flags |= VR_FLAG_OVERFLOW;
      } else {
        const int64_t n = (int64_t)floor(q);
        const double e_n = dadd(te, dmul((double)n, dt));
        const int64_t nb = (dsub(tx, e_n) > VR_SLIVER) ? n + 1 : n;  // append tx / replace
        // bin k: edges (t0, t1), its inner cuts cut[i0 .. i1) and its piece count
        auto bin_pieces = [&](int64_t k, int64_t k_end, double& t0, double& t1, int& i0,
                              int& i1) {
          int ne = 0;
          t0 = t1 = 0.0;
          i0 = i1 = 0;
          if (k < k_end) {
            t0 = (k == nb) ? tx : dadd(te, dmul((double)k, dt));
            t1 = (k + 1 == nb) ? tx : dadd(te, dmul((double)(k + 1), dt));
            if (dsub(t1, t0) > VR_SLIVER) {
              // inner cuts strictly inside (t0, t1)  (quadrature.py:106)
              while (i0 < ncut && !(cut[i0] > t0)) ++i0;
              i1 = i0;
              while (i1 < ncut && cut[i1] < t1) ++i1;
              double a = t0;
              for (int s = i0; s <= i1; ++s) {
                const double b = (s < i1) ? cut[s] : t1;
                if (dsub(b, a) > VR_SLIVER) ++ne;
                a = b;
              }
            }
          }
          return ne;
        };
        // bins that can hold own samples (conservative); earlier bins are only counted
        int64_t k_begin = 0, k_end = nb;
        if (restrict_own) {
          if (!use_occ) k_begin = max((int64_t)0, (int64_t)floor(ddiv(dsub(ta, te), dt)) - 1);
          k_end = min(nb, (int64_t)floor(ddiv(dsub(tb, te), dt)) + 2);
        }
        // pieces before bin k_begin: every bin is longer than a sliver, so it holds one
        // piece plus (pieces - 1) extra where cuts fall strictly inside it — count those
        // bins only (lane per cut, the bin's first inner cut does it), O(cuts) not O(bins)
        int carry = 0;
        // staging: reserve one slot per walked bin plus one per cut
        int64_t stage_base = -1;
        int64_t stage_n = 0;
        if (STAGE) {
          stage_n = (k_end > k_begin ? k_end - k_begin : 0) + ncut;
          unsigned long long b = 0;
          if (lane == 0) b = atomicAdd(&sm.stage_top, (unsigned long long)stage_n);
          b = __shfl_sync(0xffffffffu, b, 0);
          if ((int64_t)b + stage_n <= slice) stage_base = (int64_t)blockIdx.x * slice + (int64_t)b;
        }
        if (k_begin > 0) {
          const double e_begin = (k_begin >= nb) ? tx : dadd(te, dmul((double)k_begin, dt));
          int extra = 0;
          for (int s = lane; s < ncut; s += 32) {
            const double c = cut[s];
            if (!(c < e_begin)) continue;
            auto edge = [&](int64_t k) { return (k >= nb) ? tx : dadd(te, dmul((double)k, dt)); };
            int64_t k = (int64_t)floor(ddiv(dsub(c, te), dt));
            k = max((int64_t)0, min(k, nb - 1));
            while (k > 0 && edge(k) > c) --k;
            while (k + 1 < nb && !(edge(k + 1) > c)) ++k;  // edge(k) <= c < edge(k + 1)
            if (!(edge(k) < c)) continue;                    // on an edge: no split
            if (s > 0 && cut[s - 1] > edge(k)) continue;     // not the bin's first inner cut
            double t0, t1;
            int i0, i1;
            extra += bin_pieces(k, nb, t0, t1, i0, i1) - 1;
          }
          carry = (int)k_begin + __reduce_add_sync(0xffffffffu, extra);
        }
        const int carry_begin = carry;
        if (STAGE && lane == 0) sslot[r] = stage_base >= 0 ? stage_base - carry_begin : INT64_MIN / 2;
        for (int64_t c0 = k_begin; c0 < k_end; c0 += 32) {
          const int64_t k = c0 + lane;
          double t0, t1;
          int i0, i1;
          const int ne = bin_pieces(k, k_end, t0, t1, i0, i1);
          int nk = ne;  // kept pieces
          if (use_occ && ne > 0) {
            nk = 0;
            double a = t0;
            for (int s = i0; s <= i1; ++s) {
              const double b = (s < i1) ? cut[s] : t1;
              if (dsub(b, a) > VR_SLIVER) {
                double p[3];
                point_at(ray, sample_mid(a, b), p);
                bool oob;
                const int g = locate_point(tree, p, oob);
                nk += occupied(occ, tree, g, p) ? 1 : 0;
              }
              a = b;
            }
          }
          const int incl = warp_incl_sum_i(nk, lane);
          int gidx = carry + incl - nk;
          carry += __shfl_sync(0xffffffffu, incl, 31);
          if (ne > 0) {
            double a = t0;
            for (int s = i0; s <= i1; ++s) {
              const double b = (s < i1) ? cut[s] : t1;
              if (dsub(b, a) > VR_SLIVER) {
                const double m = sample_mid(a, b);
                double p[3];
                point_at(ray, m, p);
                bool oob;
                const int g = locate_point(tree, p, oob);
                if (oob) flags |= VR_FLAG_OOB;
                if (use_occ && !occupied(occ, tree, g, p)) {  // empty space: skipped
                  a = b;
                  continue;
                }
                const int kk = g - region_lo;
                if (kk >= 0 && kk < region_cnt) {
                  if (!FILL) {
                    atomicAdd(&sm.cnt[warp][kk], 1);
                    atomicMin(&sm.first[warp][kk], gidx);
                    if (STAGE && stage_base >= 0) {
                      const int64_t j = (int64_t)(gidx - carry_begin);
                      if (j < stage_n) {
                        st0[stage_base + j] = a;
                        st1[stage_base + j] = b;
                      } else {
                        flags |= VR_FLAG_OVERFLOW;  // cannot happen: one piece per bin + cut
                      }
                    }
                  } else {
                    const int64_t pos = sm.off[warp][kk] + (int64_t)(gidx - sm.first[warp][kk]);
                    if (pos >= sm.off[warp][kk] && pos < sm.end[warp][kk] && pos < capacity) {
                      t0o[pos] = a;
                      t1o[pos] = b;
                      rido[pos] = (int32_t)r;
                    } else {
                      flags |= VR_FLAG_OVERFLOW;
                    }
                  }
                }
                ++gidx;
              }
              a = b;
            }
          }
        }
        total = carry;
      }
    }
    __syncwarp();
    if (!FILL) {
      if (lane < region_cnt) {
        const int64_t idx = (int64_t)lane * n_rays + r;
        const int c = sm.cnt[warp][lane];
        counts[idx] = c;
        seg_first[idx] = c ? sm.first[warp][lane] : INT32_MAX;
      }
      if (lane == 0) {
        ray_te[r] = hit ? te : 0.0;
        if (ray_part) ray_part[r] = part;
        if (ray_total) ray_total[r] = total;
      }
    }
    __syncwarp();
  }
  flags = (int)__reduce_or_sync(0xffffffffu, (unsigned)flags);
  if (flags && lane == 0) atomicOr(err, flags);
  if (STAGE) {
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(&stage_info[0], sm.stage_top);
      atomicMax(&stage_info[1], sm.stage_top);
    }
  }
}

// Staged pieces -> region-major slots: warp per ray.  A ray's staged samples are ordered
// along the ray and each own segment is a contiguous run of them, so the lanes walk the
// staged range 32 samples at a time and look up each sample's segment among the ray's
// non-empty ones (lane kk holds segment kk's first index, count and output offset).
// Rays with more than 32 own regions take the region loop below.
__global__ void __launch_bounds__(256)
    k_sample_compact(int64_t n_rays, int region_cnt, const int32_t* __restrict__ counts,
                     const int32_t* __restrict__ seg_first, const int64_t* __restrict__ offsets,
                     const int64_t* __restrict__ sslot, const double* __restrict__ st0,
                     const double* __restrict__ st1, double* t0o, double* t1o, int32_t* rido,
                     int64_t capacity, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int flags = 0;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rays; r += warps) {
    for (int k0 = 0; k0 < region_cnt; k0 += 32) {
      const int kk = k0 + lane;
      const int64_t idx = (int64_t)kk * n_rays + r;
      const int c = kk < region_cnt ? counts[idx] : 0;
      const unsigned live = __ballot_sync(0xffffffffu, c > 0);
      if (!live) continue;
      const int64_t base = sslot[r];
      if (base <= INT64_MIN / 4) {  // the ray was not staged (base itself may be negative)
        flags |= VR_FLAG_OVERFLOW;
        break;
      }
      int first = INT32_MAX, last = 0;
      int64_t dst = 0;
      if (c > 0) {
        first = seg_first[idx];
        last = first + c;
        dst = offsets[idx];
      }
      const int g_lo = __reduce_min_sync(0xffffffffu, (unsigned)first);
      const int g_hi = (int)__reduce_max_sync(0xffffffffu, (unsigned)last);
      for (int g0 = g_lo; g0 < g_hi; g0 += 32) {
        const int g = g0 + lane;
        int64_t d = -1;
        for (unsigned m = live; m; m &= m - 1) {
          const int l = __ffs(m) - 1;
          const int f = __shfl_sync(0xffffffffu, first, l);
          const int e = __shfl_sync(0xffffffffu, last, l);
          const int64_t o = __shfl_sync(0xffffffffu, dst, l);
          if (g >= f && g < e) d = o + (g - f);
        }
        if (d >= 0) {
          if (d < capacity) {
            t0o[d] = st0[base + g];
            t1o[d] = st1[base + g];
            rido[d] = (int32_t)r;
          } else {
            flags |= VR_FLAG_OVERFLOW;
          }
        }
      }
    }
  }
  flags = (int)__reduce_or_sync(0xffffffffu, (unsigned)flags);
  if (flags && lane == 0) atomicOr(err, flags);
}

__global__ void k_locate(const VrTree tree, const double* __restrict__ pts, int64_t n,
                         int32_t* tile, int32_t* err) {
  int flags = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    bool oob;
    const int g = locate_point(tree, p, oob);
    tile[i] = oob ? -1 : g;
    if (oob) flags |= VR_FLAG_OOB;
  }
  if (flags) atomicOr(err, flags);
}

struct ToI64 {
  __host__ __device__ int64_t operator()(int32_t v) const { return (int64_t)v; }
};

__global__ void k_scan_tail(const int32_t* counts, int64_t n, int64_t* offsets) {
  if (n == 0) {
    offsets[0] = 0;
  } else {
    offsets[n] = offsets[n - 1] + (int64_t)counts[n - 1];
  }
}

static bool valid_occ(const VrOccupancy* o) {
  return !o || o->res == 0 || (o->res > 0 && o->res <= 1024 && o->bits);
}

static VrOccupancy occ_or_none(const VrOccupancy* o) {
  VrOccupancy v;
  v.bits = (o && o->res > 0) ? o->bits : nullptr;
  v.res = (o && o->bits) ? o->res : 0;
  v.pad_ = 0;
  return v;
}

static bool valid_tree(const VrTree* t) {
  return t && t->n_leaves >= 1 && t->n_leaves <= VR_MAX_REGIONS && t->n_nodes >= 0 &&
         t->n_nodes < VR_MAX_REGIONS && (t->n_nodes == 0 ? t->n_leaves == 1 : true);
}

}  // namespace vr

using namespace vr;

extern "C" int vr_sample_count(const VrTree* tree, const double* rays, int64_t stride,
                               int64_t n_rays, double dt, int32_t region_lo, int32_t region_cnt,
                               int32_t* counts, int32_t* seg_first, double* ray_te,
                               uint32_t* ray_part, int32_t* ray_total,
                               const VrOccupancy* occ, int32_t* err, void* stream) {
  if (!valid_tree(tree) || !(dt > 0.0) || region_lo < 0 || region_cnt < 1 ||
      region_lo + region_cnt > tree->n_leaves || n_rays < 0 || !err || !valid_occ(occ)) {
    set_error("vr_sample_count: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const VrOccupancy oc = occ_or_none(occ);
  if (n_rays == 0) return VR_OK;
  const int grid = grid_for(ceil_div(n_rays, K1_WARPS), 1, 16);
  const bool restrict_own = !ray_part && !ray_total &&
                            !(region_lo == 0 && region_cnt == tree->n_leaves);
  if (restrict_own)
    k_sample<false, true, false><<<grid, K1_WARPS * 32, 0, (cudaStream_t)stream>>>(
        *tree, oc, rays, stride, n_rays, dt, region_lo, region_cnt, counts, seg_first, ray_te,
        ray_part, ray_total, nullptr, nullptr, nullptr, nullptr, 0, err, nullptr, nullptr,
        nullptr, 0, nullptr, nullptr);
  else
    k_sample<false, false, false><<<grid, K1_WARPS * 32, 0, (cudaStream_t)stream>>>(
        *tree, oc, rays, stride, n_rays, dt, region_lo, region_cnt, counts, seg_first, ray_te,
        ray_part, ray_total, nullptr, nullptr, nullptr, nullptr, 0, err, nullptr, nullptr,
        nullptr, 0, nullptr, nullptr);
  return check_launch("vr_sample_count");
}

extern "C" int64_t vr_sample_stage_blocks(int64_t n_rays) {
  return n_rays > 0 ? grid_for(ceil_div(n_rays, K1_WARPS), 1, 16) : 0;
}

extern "C" int vr_sample_stage(const VrTree* tree, const double* rays, int64_t stride,
                               int64_t n_rays, double dt, int32_t region_lo, int32_t region_cnt,
                               int32_t* counts, int32_t* seg_first, double* ray_te,
                               uint32_t* ray_part, int32_t* ray_total, double* st0, double* st1,
                               int64_t stage_capacity, int64_t* sslot, uint64_t* stage_info,
                               int32_t* ray_list, const VrOccupancy* occ, int32_t* err,
                               void* stream) {
  if (!valid_tree(tree) || !(dt > 0.0) || region_lo < 0 || region_cnt < 1 ||
      region_lo + region_cnt > tree->n_leaves || n_rays < 0 || !err || !stage_info ||
      stage_capacity < 0 || (n_rays > 0 && (!st0 || !st1 || !sslot)) || !valid_occ(occ)) {
    set_error("vr_sample_stage: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const VrOccupancy oc = occ_or_none(occ);
  if (n_rays == 0) return VR_OK;
  const int grid = (int)vr_sample_stage_blocks(n_rays);
  const int64_t slice = stage_capacity / grid;
  const bool restrict_own = !ray_part && !ray_total &&
                            !(region_lo == 0 && region_cnt == tree->n_leaves);
  auto* info = reinterpret_cast<unsigned long long*>(stage_info);
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t* list = nullptr;
  if (restrict_own && ray_list) {
    cudaMemsetAsync(ray_list, 0, sizeof(int32_t), s);
    k_sample_prefilter<<<grid_for(n_rays, 256), 256, 0, s>>>(
        *tree, rays, stride, n_rays, region_lo, region_cnt, counts, seg_first, ray_te, ray_list);
    list = ray_list;
  }
  if (restrict_own)
    k_sample<false, true, true><<<grid, K1_WARPS * 32, 0, s>>>(
        *tree, oc, rays, stride, n_rays, dt, region_lo, region_cnt, counts, seg_first, ray_te,
        ray_part, ray_total, nullptr, nullptr, nullptr, nullptr, 0, err, st0, st1, sslot, slice,
        info, list);
  else
    k_sample<false, false, true><<<grid, K1_WARPS * 32, 0, s>>>(
        *tree, oc, rays, stride, n_rays, dt, region_lo, region_cnt, counts, seg_first, ray_te,
        ray_part, ray_total, nullptr, nullptr, nullptr, nullptr, 0, err, st0, st1, sslot, slice,
        info, nullptr);
  return check_launch("vr_sample_stage");
}

extern "C" int vr_sample_compact(int64_t n_rays, int32_t region_cnt, const int32_t* counts,
                                 const int32_t* seg_first, const int64_t* offsets,
                                 const int64_t* sslot, const double* st0, const double* st1,
                                 double* t0, double* t1, int32_t* ray_id, int64_t capacity,
                                 int32_t* err, void* stream) {
  if (n_rays < 0 || region_cnt < 1 || !err) {
    set_error("vr_sample_compact: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n_rays == 0) return VR_OK;
  k_sample_compact<<<grid_for(n_rays, 8), 256, 0, (cudaStream_t)stream>>>(
      n_rays, region_cnt, counts, seg_first, offsets, sslot, st0, st1, t0, t1, ray_id, capacity,
      err);
  return check_launch("vr_sample_compact");
}

extern "C" int vr_sample_fill(const VrTree* tree, const double* rays, int64_t stride,
                              int64_t n_rays, double dt, int32_t region_lo, int32_t region_cnt,
                              const int64_t* offsets, const int32_t* seg_first, double* t0,
                              double* t1, int32_t* ray_id, int64_t capacity,
                              const VrOccupancy* occ, int32_t* err, void* stream) {
  if (!valid_tree(tree) || !(dt > 0.0) || region_lo < 0 || region_cnt < 1 ||
      region_lo + region_cnt > tree->n_leaves || n_rays < 0 || !err || !valid_occ(occ)) {
    set_error("vr_sample_fill: bad argument");
    return VR_ERR_BAD_ARG;
  }
  const VrOccupancy oc = occ_or_none(occ);
  if (n_rays == 0) return VR_OK;
  const int grid = grid_for(ceil_div(n_rays, K1_WARPS), 1, 16);
  // the fill walks the same bins as the count (restricted unless all regions are owned;
  // the counts of a restricted count pass are exactly the full walk's)
  if (!(region_lo == 0 && region_cnt == tree->n_leaves))
    k_sample<true, true, false><<<grid, K1_WARPS * 32, 0, (cudaStream_t)stream>>>(
        *tree, oc, rays, stride, n_rays, dt, region_lo, region_cnt, nullptr,
        const_cast<int32_t*>(seg_first), nullptr, nullptr, nullptr, offsets, t0, t1, ray_id,
        capacity, err, nullptr, nullptr, nullptr, 0, nullptr, nullptr);
  else
    k_sample<true, false, false><<<grid, K1_WARPS * 32, 0, (cudaStream_t)stream>>>(
        *tree, oc, rays, stride, n_rays, dt, region_lo, region_cnt, nullptr,
        const_cast<int32_t*>(seg_first), nullptr, nullptr, nullptr, offsets, t0, t1, ray_id,
        capacity, err, nullptr, nullptr, nullptr, 0, nullptr, nullptr);
  return check_launch("vr_sample_fill");
}

extern "C" int vr_locate(const VrTree* tree, const double* pts, int64_t n, int32_t* tile,
                         int32_t* err, void* stream) {
  if (!valid_tree(tree) || n < 0 || !err) {
    set_error("vr_locate: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_locate<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*tree, pts, n, tile, err);
  return check_launch("vr_locate");
}

extern "C" size_t vr_scan_workspace_bytes(int64_t n) {
  size_t bytes = 0;
  cub::TransformInputIterator<int64_t, ToI64, const int32_t*> it(nullptr, ToI64());
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (int64_t*)nullptr, n > 0 ? n : 1);
  return bytes + 256;
}

extern "C" int vr_scan_offsets(const int32_t* counts, int64_t n, int64_t* offsets, void* ws,
                               size_t ws_bytes, void* stream) {
  if (n < 0 || !offsets) {
    set_error("vr_scan_offsets: bad argument");
    return VR_ERR_BAD_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (n > 0) {
    size_t need = 0;
    cub::TransformInputIterator<int64_t, ToI64, const int32_t*> it(counts, ToI64());
    cub::DeviceScan::ExclusiveSum(nullptr, need, it, offsets, n, s);
    if (need > ws_bytes) {
      set_error("vr_scan_offsets: workspace too small");
      return VR_ERR_BAD_ARG;
    }
    if (cub::DeviceScan::ExclusiveSum(ws, need, it, offsets, n, s) != cudaSuccess) {
      set_error("vr_scan_offsets: cub scan failed");
      return VR_ERR_CUDA;
    }
  }
  k_scan_tail<<<1, 1, 0, s>>>(counts, n, offsets);
  return check_launch("vr_scan_offsets");
}
