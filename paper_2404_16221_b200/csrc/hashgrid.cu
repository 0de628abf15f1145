// K2 — per-region multiresolution hash-grid encoding (Instant-NGP).
//
// There is no reference implementation; the spec below is
// restated bit-for-bit in oracle/hashmlp_oracle.py:
//   u   = float32((p - box_mn) / (box_mx - box_mn))          float64 ops, one cast
//   pos = u * scale_l + 0.5f        (two float32 roundings, no FMA)
//   g   = clamp(floor(pos), 0, res_l - 2),  f = pos - g
//   corner c = (cx, cy, cz):  idx = dense_l ? x + res*(y + res*z)
//                                           : (x ^ y*2654435761 ^ z*805459861) & (T-1)
//   w_c = (wx * wy) * wz,  feat_l = sum_{c even} w_c t_c + sum_{c odd} w_c t_c   (F = 2,
//   float32, each half summed in increasing c from 0, no FMA; t_c = table[offset_l + idx_c])
// Encodings are written level-major enc[l][n] as half2 so both the gather kernel
// and the MLP read them coalesced.  Gathers and the backward's float2 atomics run in lane
// pairs (two lanes per sample, one per x side of the cell: gather_half / scatter_half in
// hashgrid.cuh); the coarsest dense level's atomics go through per-warp replicas
// (RepPlan).
// The production training path fuses both directions into the tensor-core MLP kernels
// (mlp_tc.cu); these standalone kernels serve inference-only callers and the tests.
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "hashgrid.cuh"

namespace vr {

constexpr int HASH_THREADS = 256;

// Lane pairs: a warp covers 16 samples per step; lane 2j+p gathers half p of sample j's
// corners (gather_half), the partner's half arrives by one shuffle.
__global__ void __launch_bounds__(HASH_THREADS)
    k_hash_fwd(const VrHashGridDesc g, const float2* __restrict__ table,
               const double* __restrict__ rays, int64_t stride, const double* __restrict__ t0,
               const double* __restrict__ t1, const int32_t* __restrict__ rid, int64_t n,
               __half2* __restrict__ enc, float* __restrict__ pos) {
  const BoxInv bi = box_inv(g);
  const int lane = threadIdx.x & 31, p = lane & 1;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s0 = warp0 * 16; s0 < n; s0 += n_warps * 16) {
    const int64_t i = s0 + (lane >> 1);
    const bool valid = i < n;
    float u[3] = {0.f, 0.f, 0.f};
    if (valid && p == 0) norm_pos(g, bi, rays, stride, t0, t1, rid, i, u);
#pragma unroll
    for (int a = 0; a < 3; ++a) u[a] = __shfl_sync(0xffffffffu, u[a], lane & ~1);
    if (pos && valid && p == 1) {
      pos[i] = u[0];
      pos[n + i] = u[1];
      pos[2 * n + i] = u[2];
    }
#pragma unroll 2
    for (int l = 0; l < g.n_levels; ++l) {
      float2 h = make_float2(0.f, 0.f);
      if (valid) h = gather_half(g, l, table + g.offset[l], u, p);
      const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, h.x, 1),
                                   __shfl_xor_sync(0xffffffffu, h.y, 1));
      if (valid && p == 0)
        enc[(int64_t)l * n + i] = __floats2half2_rn(__fadd_rn(h.x, o.x), __fadd_rn(h.y, o.y));
    }
  }
}

__global__ void __launch_bounds__(HASH_THREADS)
    k_hash_bwd(const VrHashGridDesc g, const RepPlan plan, const double* __restrict__ rays,
               int64_t stride, const double* __restrict__ t0, const double* __restrict__ t1,
               const int32_t* __restrict__ rid, int64_t n, const float2* __restrict__ denc,
               float2* __restrict__ grad, float2* __restrict__ ws) {
  const BoxInv bi = box_inv(g);
  const int gwarp = blockIdx.x * (HASH_THREADS / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31, p = lane & 1;  // lane pairs (scatter_half)
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s0 = warp0 * 16; s0 < n; s0 += n_warps * 16) {
    const int64_t i = s0 + (lane >> 1);
    const bool valid = i < n;
    float u[3] = {0.f, 0.f, 0.f};
    if (valid && p == 0) norm_pos(g, bi, rays, stride, t0, t1, rid, i, u);
#pragma unroll
    for (int a = 0; a < 3; ++a) u[a] = __shfl_sync(0xffffffffu, u[a], lane & ~1);
    if (!valid) continue;
#pragma unroll 2
    for (int l = 0; l < g.n_levels; ++l) {
      const float2 d = denc[(int64_t)l * n + i];
      if (d.x != 0.f || d.y != 0.f) scatter_half(g, plan, l, u, d, p, gwarp, grad, ws);
    }
  }
}

// ---- level-major variants (tables larger than L2) ---------------------------------------
// With T = 2^22 a region's table is ~0.5 GB: per-sample loops over all 16 levels turn every
// corner access into a DRAM sector read-modify-write.  Level-major kernels walk the
// samples once per level pass: a persistent grid claims (pass, chunk) work items from a
// counter in increasing order, so every block has claimed its last item of pass p before
// any block starts pass p + 1 (ordered by construction — not by the block scheduler's
// dispatch order — and without the drain between passes that one launch per pass costs:
// c4 325.0 vs 311.7 ms measured for per-pass launches vs one launch): only one level's
// slice (<= 32 MB) is live, it stays in L2, and the
// DRAM traffic becomes the streaming of u / enc / d(enc) (16 B per sample and level).
// The normalised positions are computed once (k_hash_pos) and reused by the backward;
// the streamed pos / enc / d(enc) use evict-first accesses so they do not push the live
// table slice out of L2.
__global__ void __launch_bounds__(HASH_THREADS)
    k_hash_pos(const VrHashGridDesc g, const double* __restrict__ rays, int64_t stride,
               const double* __restrict__ t0, const double* __restrict__ t1,
               const int32_t* __restrict__ rid, int64_t n, float* __restrict__ pos) {
  const BoxInv bi = box_inv(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float u[3];
    norm_pos(g, bi, rays, stride, t0, t1, rid, i, u);
    pos[i] = u[0];
    pos[n + i] = u[1];
    pos[2 * n + i] = u[2];
  }
}

// Passes group consecutive levels (pass p = levels [first[p], first[p+1])): the
// small coarse levels share one pass, so their atomics are diluted among several levels'
// (one coarse level alone would put every SM's atomics on a few thousand addresses).
struct LmPasses {
  int32_t n;
  int32_t first[VR_MAX_LEVELS + 1];
};

constexpr int64_t LM_CHUNK = 4096;  // samples per work item
constexpr int SU = 4;               // scatter: warp steps (16 samples each) per iteration

// the block's next work item (block-uniform); item = pass * chunks + chunk
__device__ __forceinline__ int64_t lm_claim(unsigned long long* ctr) {
  __shared__ long long item;
  __syncthreads();  // the previous item is consumed by every thread
  if (threadIdx.x == 0) item = (long long)atomicAdd(ctr, 1ull);
  __syncthreads();
  return item;
}

__global__ void __launch_bounds__(HASH_THREADS, 6)  // 40 regs: c5 57.0 -> 55.2 ms
    k_hash_fwd_lm(const VrHashGridDesc g, const LmPasses passes, const float2* __restrict__ table,
                  const float* __restrict__ pos, int64_t n, __half2* __restrict__ enc,
                  unsigned long long* ctr) {
  const int lane = threadIdx.x & 31, p = lane & 1;  // lane pairs as in k_hash_fwd
  const int warp = threadIdx.x >> 5, n_warps = blockDim.x >> 5;
  const int64_t chunks = ceil_div(n, LM_CHUNK);
  for (int64_t item = lm_claim(ctr); item < passes.n * chunks; item = lm_claim(ctr)) {
  const int pass = (int)(item / chunks);
  const int l0 = passes.first[pass], l1 = passes.first[pass + 1];
  const int64_t c0 = (item - pass * chunks) * LM_CHUNK, c1 = min(n, c0 + LM_CHUNK);
  for (int64_t s0 = c0 + warp * 16; s0 < c1; s0 += n_warps * 16) {
    const int64_t i = s0 + (lane >> 1);
    const bool valid = i < c1;
    float u[3] = {0.f, 0.f, 0.f};
    if (valid) {
      u[0] = __ldcs(pos + i);
      u[1] = __ldcs(pos + n + i);
      u[2] = __ldcs(pos + 2 * n + i);
    }
    for (int l = l0; l < l1; ++l) {
      float2 h = make_float2(0.f, 0.f);
      if (valid) h = gather_half(g, l, table + g.offset[l], u, p);
      const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, h.x, 1),
                                   __shfl_xor_sync(0xffffffffu, h.y, 1));
      if (valid && p == 0)
        __stcs(enc + (int64_t)l * n + i,
               __floats2half2_rn(__fadd_rn(h.x, o.x), __fadd_rn(h.y, o.y)));
    }
  }
  }
}

// rows (optional, vr_active_rows): scatter only the samples rows[0, m), m = *n_rows, whose
// d(enc) the MLP backward wrote at compact positions (denc[l][j] belongs to sample rows[j]);
// positions are read at the sample index.
// 4 resident blocks (64 registers): the scatter is load-latency bound, warps matter more
// than registers (c4 serial scatter 20.2 -> 16.1 ms against the unconstrained 89 registers)
__global__ void __launch_bounds__(HASH_THREADS, 4)
    k_hash_bwd_lm(const VrHashGridDesc g, const RepPlan plan, const LmPasses passes,
                  const float* __restrict__ pos, int64_t n, const float2* __restrict__ denc,
                  float2* __restrict__ grad, float2* __restrict__ ws, unsigned long long* ctr,
                  const int32_t* __restrict__ rows, const int32_t* __restrict__ n_rows) {
  const int gwarp = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31, p = lane & 1;  // lane pairs (scatter_half)
  const int warp = threadIdx.x >> 5, n_warps = blockDim.x >> 5;
  const int64_t m = rows ? (int64_t)__ldg(n_rows) : n;
  const int64_t chunks = ceil_div(m, LM_CHUNK);
  for (int64_t item = lm_claim(ctr); item < passes.n * chunks; item = lm_claim(ctr)) {
    const int pass = (int)(item / chunks);
    const int l0 = passes.first[pass], l1 = passes.first[pass + 1];
    const int64_t c0 = (item - pass * chunks) * LM_CHUNK, c1 = min(m, c0 + LM_CHUNK);
    // SU warp steps of 16 samples per iteration, every load issued before the atomics that
    // depend on it and the next level's d(enc) loaded while this level's atomics issue
    // (ncu, c4 steady state: one step per iteration left 75 % of the warps' cycles waiting
    // on the d(enc) / position loads — the scatter was latency-bound, not L2-atomic bound)
    for (int64_t s0 = c0 + warp * 16 * SU; s0 < c1; s0 += n_warps * 16 * SU) {
      int64_t jj[SU];
      float u[SU][3];
#pragma unroll
      for (int k = 0; k < SU; ++k) {
        jj[k] = s0 + 16 * k + (lane >> 1);
        int64_t i = 0;
        if (jj[k] < c1) {
          i = rows ? (int64_t)__ldg(rows + jj[k]) : jj[k];
          if (!VR_CHECK(i >= 0 && i < n)) i = 0;
        }
        u[k][0] = jj[k] < c1 ? __ldcs(pos + i) : 0.f;
        u[k][1] = jj[k] < c1 ? __ldcs(pos + n + i) : 0.f;
        u[k][2] = jj[k] < c1 ? __ldcs(pos + 2 * n + i) : 0.f;
      }
      float2 dc[SU];
#pragma unroll
      for (int k = 0; k < SU; ++k)
        dc[k] = jj[k] < c1 ? __ldcs(denc + (int64_t)l0 * n + jj[k]) : make_float2(0.f, 0.f);
      for (int l = l0; l < l1; ++l) {
        float2 dn[SU];
#pragma unroll
        for (int k = 0; k < SU; ++k)
          dn[k] = (l + 1 < l1 && jj[k] < c1) ? __ldcs(denc + (int64_t)(l + 1) * n + jj[k])
                                             : make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < SU; ++k)
          if (dc[k].x != 0.f || dc[k].y != 0.f) {
            const float uk[3] = {u[k][0], u[k][1], u[k][2]};
            scatter_half(g, plan, l, uk, dc[k], p, gwarp, grad, ws);
          }
#pragma unroll
        for (int k = 0; k < SU; ++k) dc[k] = dn[k];
      }
    }
  }
}

// greedy: consecutive levels share a pass while their slices total <= 48 MB (the streamed
// positions are re-read once per pass, the live slices must stay in L2; measured on c4/c5:
// 64 MB passes — two 32 MB hashed levels — thrash L2, c5 97 -> 111 ms)
static LmPasses lm_passes(const VrHashGridDesc* g) {
  LmPasses p;
  memset(&p, 0, sizeof(p));
  const int64_t budget = (int64_t)48 << 20;
  int64_t bytes = 0;
  for (int l = 0; l < g->n_levels; ++l) {
    const int64_t b = (g->offset[l + 1] - g->offset[l]) * (int64_t)sizeof(float2);
    if (l == 0 || bytes + b > budget) {
      p.first[p.n++] = l;
      bytes = 0;
    }
    bytes += b;
  }
  p.first[p.n] = g->n_levels;
  return p;
}

// grad[level l entry e] += sum_r ws[l][r][e]; the replicas are zeroed for the next use
__global__ void k_hash_rep_reduce(const VrHashGridDesc g, const RepPlan plan,
                                  float2* __restrict__ grad, float2* __restrict__ ws,
                                  int64_t total) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = t;
    int l = 0;
    while (l < plan.n_rep - 1 && e >= g.offset[l + 1] - g.offset[l]) {
      e -= g.offset[l + 1] - g.offset[l];
      ++l;
    }
    const int64_t size_l = g.offset[l + 1] - g.offset[l];
    float2* w = ws + plan.off[l] + e;
    float2 acc = make_float2(0.f, 0.f);
    // the replicas' loads unrolled (independent), the sum in replica order as before
#pragma unroll 8
    for (int r = 0; r < plan.R[l]; ++r) {
      const float2 v = w[r * size_l];
      acc.x += v.x;
      acc.y += v.y;
      w[r * size_l] = make_float2(0.f, 0.f);
    }
    float2* gp = grad + g.offset[l] + e;
    gp->x += acc.x;
    gp->y += acc.y;
  }
}

RepPlan hash_rep_plan(const VrHashGridDesc* g, int64_t* ws_entries, int64_t* red_entries) {
  RepPlan p;
  memset(&p, 0, sizeof(p));
  int64_t off = 0, red = 0;
  for (int l = 0; l < g->n_levels; ++l) {
    const int64_t size_l = g->offset[l + 1] - g->offset[l];
    // measured on c3 (scripts/bench_hash.py): only the coarsest level (17^3 entries) is
    // contention-bound; replicating the 24^3 / 32^3 levels costs more than it saves
    if (!g->dense[l] || size_l > 8192) break;
    const int R = 64;
    p.R[l] = R;
    p.off[l] = off;
    off += (int64_t)R * size_l;
    red += size_l;
    p.n_rep = l + 1;
  }
  *ws_entries = off;
  *red_entries = red;
  return p;
}

int hash_rep_reduce(const VrHashGridDesc* g, const RepPlan& plan, int64_t red, float* grad,
                    void* ws, void* stream) {
  if (plan.n_rep == 0) return VR_OK;
  k_hash_rep_reduce<<<grid_for(red, 256, 4), 256, 0, (cudaStream_t)stream>>>(
      *g, plan, reinterpret_cast<float2*>(grad), reinterpret_cast<float2*>(ws), red);
  return check_launch("hash_rep_reduce");
}

__global__ void k_hash_idx(const VrHashGridDesc g, const double* __restrict__ rays, int64_t stride,
                           const double* __restrict__ t0, const double* __restrict__ t1,
                           const int32_t* __restrict__ rid, int64_t n, int32_t* __restrict__ out) {
  const BoxInv bi = box_inv(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float u[3];
    norm_pos(g, bi, rays, stride, t0, t1, rid, i, u);
    for (int l = 0; l < g.n_levels; ++l) {
      Corners c;
      level_corners(g, l, u, c);
#pragma unroll
      for (int k = 0; k < 8; ++k) out[((int64_t)l * n + i) * 8 + k] = (int32_t)c.idx[k];
    }
  }
}

bool valid_grid(const VrHashGridDesc* g) {
  if (!g || g->n_levels < 1 || g->n_levels > VR_MAX_LEVELS || g->log2_T < 1 || g->log2_T > 28)
    return false;
  for (int l = 0; l < g->n_levels; ++l)
    if (g->res[l] < 2) return false;
  return true;
}

}  // namespace vr

using namespace vr;

extern "C" int vr_hash_fwd(const VrHashGridDesc* g, const float* table, const double* rays,
                           int64_t stride, const double* t0, const double* t1, const int32_t* rid,
                           int64_t n, void* enc, float* pos, void* stream) {
  if (!valid_grid(g) || n < 0) {
    set_error("vr_hash_fwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_hash_fwd<<<grid_for(2 * n, HASH_THREADS, 8), HASH_THREADS, 0, (cudaStream_t)stream>>>(
      *g, reinterpret_cast<const float2*>(table), rays, stride, t0, t1, rid, n,
      reinterpret_cast<__half2*>(enc), pos);
  return check_launch("vr_hash_fwd");
}

extern "C" size_t vr_hash_bwd_workspace_bytes(const VrHashGridDesc* g) {
  if (!valid_grid(g)) return 0;
  int64_t ws = 0, red = 0;
  hash_rep_plan(g, &ws, &red);
  return (size_t)ws * sizeof(float2);
}

extern "C" int vr_hash_bwd(const VrHashGridDesc* g, const double* rays, int64_t stride,
                           const double* t0, const double* t1, const int32_t* rid, int64_t n,
                           const float* denc, float* grad, void* ws, size_t ws_bytes,
                           void* stream) {
  if (!valid_grid(g) || n < 0) {
    set_error("vr_hash_bwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  int64_t ws_entries = 0, red = 0;
  RepPlan plan = hash_rep_plan(g, &ws_entries, &red);
  if (!ws || ws_bytes < (size_t)ws_entries * sizeof(float2)) plan.n_rep = 0;  // plain atomics
  k_hash_bwd<<<grid_for(2 * n, HASH_THREADS, 8), HASH_THREADS, 0, (cudaStream_t)stream>>>(
      *g, plan, rays, stride, t0, t1, rid, n, reinterpret_cast<const float2*>(denc),
      reinterpret_cast<float2*>(grad), reinterpret_cast<float2*>(ws));
  const int rc = check_launch("vr_hash_bwd");
  if (rc != VR_OK) return rc;
  return hash_rep_reduce(g, plan, red, grad, ws, stream);
}

extern "C" int vr_hash_indices(const VrHashGridDesc* g, const double* rays, int64_t stride,
                               const double* t0, const double* t1, const int32_t* rid, int64_t n,
                               int32_t* out, void* stream) {
  if (!valid_grid(g) || n < 0) {
    set_error("vr_hash_indices: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_hash_idx<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(*g, rays, stride, t0, t1, rid,
                                                                   n, out);
  return check_launch("vr_hash_indices");
}

extern "C" int vr_hash_positions(const VrHashGridDesc* g, const double* rays, int64_t stride,
                                 const double* t0, const double* t1, const int32_t* rid,
                                 int64_t n, float* pos, void* stream) {
  if (!valid_grid(g) || n < 0 || (n > 0 && !pos)) {
    set_error("vr_hash_positions: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_hash_pos<<<grid_for(n, HASH_THREADS, 8), HASH_THREADS, 0, (cudaStream_t)stream>>>(
      *g, rays, stride, t0, t1, rid, n, pos);
  return check_launch("vr_hash_positions");
}

// persistent grid of the ordered level-major kernels: the SMs' resident blocks
template <class K>
static int lm_blocks(K kernel, int threads, int64_t items) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess ||
      per_sm < 1)
    per_sm = 4;
  const int64_t b = (int64_t)VR_NUM_SMS * per_sm;
  return (int)(items < b ? (items > 0 ? items : 1) : b);
}

// a work counter zeroed on the stream: slot k of a ring allocated once per device (calls
// in flight at the same time — on different streams — take different slots)
static unsigned long long* lm_counter(cudaStream_t s) {
  constexpr int SLOTS = 4096;
  static unsigned long long* ring[64] = {};
  static std::atomic<unsigned> next{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!ring[dev]) {
    void* p = nullptr;
    if (cudaMalloc(&p, SLOTS * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    ring[dev] = reinterpret_cast<unsigned long long*>(p);
  }
  unsigned long long* c = ring[dev] + (next.fetch_add(1) % SLOTS);
  cudaMemsetAsync(c, 0, sizeof(unsigned long long), s);
  return c;
}

extern "C" int vr_hash_lm_passes(const VrHashGridDesc* g) {
  return valid_grid(g) ? lm_passes(g).n : 0;
}

extern "C" int vr_hash_fwd_lm(const VrHashGridDesc* g, const float* table, const float* pos,
                              int64_t n, void* enc, void* stream) {
  if (!valid_grid(g) || n < 0 || (n > 0 && (!table || !pos || !enc))) {
    set_error("vr_hash_fwd_lm: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  const LmPasses passes = lm_passes(g);
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* ctr = lm_counter(s);
  if (!ctr) {
    set_error("vr_hash_fwd_lm: work counter allocation failed");
    return VR_ERR_CUDA;
  }
  const int blocks = lm_blocks(k_hash_fwd_lm, HASH_THREADS, passes.n * ceil_div(n, LM_CHUNK));
  k_hash_fwd_lm<<<blocks, HASH_THREADS, 0, s>>>(*g, passes, reinterpret_cast<const float2*>(table),
                                               pos, n, reinterpret_cast<__half2*>(enc), ctr);
  return check_launch("vr_hash_fwd_lm");
}

extern "C" int vr_hash_scatter(const VrHashGridDesc* g, const float* pos, int64_t n,
                               const float* denc, float* grad, void* ws, size_t ws_bytes,
                               int32_t level_major, int32_t max_blocks, const int32_t* rows,
                               const int32_t* n_rows, void* stream) {
  if (!valid_grid(g) || n < 0 || max_blocks < 0 || (n > 0 && (!pos || !denc || !grad)) ||
      (!rows != !n_rows)) {
    set_error("vr_hash_scatter: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  int64_t ws_entries = 0, red = 0;
  RepPlan plan = hash_rep_plan(g, &ws_entries, &red);
  if (!ws || ws_bytes < (size_t)ws_entries * sizeof(float2)) plan.n_rep = 0;
  LmPasses passes;
  if (level_major) {
    passes = lm_passes(g);
  } else {  // one pass over all levels: sample order
    memset(&passes, 0, sizeof(passes));
    passes.n = 1;
    passes.first[1] = g->n_levels;
  }
  cudaStream_t s = (cudaStream_t)stream;
  auto kern = k_hash_bwd_lm;
  int threads = HASH_THREADS;
  int blocks = lm_blocks(kern, HASH_THREADS, passes.n * ceil_div(n, LM_CHUNK));
  if (max_blocks > 0) {  // co-resident with another kernel: a few small blocks
    threads = 128;
    blocks = max_blocks;
  }
  unsigned long long* ctr = lm_counter(s);
  if (!ctr) {
    set_error("vr_hash_scatter: work counter allocation failed");
    return VR_ERR_CUDA;
  }
  kern<<<blocks, threads, 0, s>>>(*g, plan, passes, pos, n,
                                           reinterpret_cast<const float2*>(denc),
                                           reinterpret_cast<float2*>(grad),
                                           reinterpret_cast<float2*>(ws), ctr, rows, n_rows);
  const int rc = check_launch("vr_hash_scatter");
  if (rc != VR_OK) return rc;
  return hash_rep_reduce(g, plan, red, grad, ws, stream);
}

extern "C" int vr_hash_bwd_lm(const VrHashGridDesc* g, const float* pos, int64_t n,
                              const float* denc, float* grad, void* ws, size_t ws_bytes,
                              void* stream) {
  return vr_hash_scatter(g, pos, n, denc, grad, ws, ws_bytes, 1, 0, nullptr, nullptr, stream);
}
