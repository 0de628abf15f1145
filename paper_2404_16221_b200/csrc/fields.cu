// Field plugins evaluated at bin midpoints (quadrature.fill_samples, quadrature.py:117-128).
//
// The analytic fields and the voxel grid are the reference's own test fields
// (field.py:88-240); they let the whole GPU path be checked end to end against the
// unmodified reference.  Evaluation is float64 (these are parity fields, not the
// performance path) and each sample is evaluated only by the region that owns it,
// which is exactly MaskedField/tile_mask semantics (field.py:243-273): the owner
// sees the base field, nobody else receives the sample.
#include "common.cuh"

namespace vr {

struct Sample {
  double p[3];
};

__device__ __forceinline__ void sample_point(const double* __restrict__ rays, int64_t stride,
                                             const double* __restrict__ t0,
                                             const double* __restrict__ t1,
                                             const int32_t* __restrict__ rid, int64_t i,
                                             double p[3]) {
  const int64_t r = checked_ray(rid[i], stride);
  const double m = sample_mid(t0[i], t1[i]);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    p[a] = dadd(__ldg(rays + a * stride + r), dmul(m, __ldg(rays + (3 + a) * stride + r)));
}

// GaussianBlobs.sigma_many/rgb_many (field.py:97-114) for one child
__device__ void eval_blobs(const VrAnalyticField& f, int lo, int cnt, const double p[3],
                           double& sigma, double rgb[3]) {
  double tot = 0.0, w[3] = {0.0, 0.0, 0.0}, mean[3] = {0.0, 0.0, 0.0};
  for (int b = lo; b < lo + cnt; ++b) {
    const VrBlob& bl = f.blobs[b];
    const double dx = p[0] - bl.center[0], dy = p[1] - bl.center[1], dz = p[2] - bl.center[2];
    const double d2 = dx * dx + dy * dy + dz * dz;
    const double s = bl.amplitude * exp(-0.5 * d2 / (bl.scale * bl.scale));
    tot += s;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      w[c] += s * bl.color[c];
      mean[c] += bl.color[c];
    }
  }
  sigma = tot;
#pragma unroll
  for (int c = 0; c < 3; ++c) rgb[c] = tot > 0.0 ? w[c] / tot : mean[c] / (double)cnt;
}

__global__ void k_field_analytic(const VrAnalyticField f, const double* __restrict__ rays,
                                 int64_t stride, const double* __restrict__ t0,
                                 const double* __restrict__ t1, const int32_t* __restrict__ rid,
                                 int64_t n, float4* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p[3];
    sample_point(rays, stride, t0, t1, rid, i, p);
    double sig_tot = 0.0, wsum[3] = {0.0, 0.0, 0.0}, mean[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < f.n_children; ++c) {
      double s, rgb[3];
      if (f.child_kind[c] == 0) {
        eval_blobs(f, f.child_blob_lo[c], f.child_blob_cnt[c], p, s, rgb);
      } else {
        const bool in = p[0] >= f.box_mn[c][0] && p[1] >= f.box_mn[c][1] &&
                        p[2] >= f.box_mn[c][2] && p[0] <= f.box_mx[c][0] &&
                        p[1] <= f.box_mx[c][1] && p[2] <= f.box_mx[c][2];
        s = in ? f.box_density[c] : 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) rgb[k] = in ? f.box_color[c][k] : 0.0;
      }
      sig_tot += s;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        wsum[k] += s * rgb[k];
        mean[k] += rgb[k];
      }
    }
    double rgb[3];
    if (f.n_children == 1) {
      // a plain field: its own colour rule already applied
#pragma unroll
      for (int k = 0; k < 3; ++k) rgb[k] = mean[k];
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k)
        rgb[k] = sig_tot > 0.0 ? wsum[k] / sig_tot : mean[k] / (double)f.n_children;
    }
    out[i] = make_float4((float)sig_tot, (float)rgb[0], (float)rgb[1], (float)rgb[2]);
  }
}

// ---- VoxelGrid (field.py:137-209) -------------------------------------------------------
struct VoxStencil {
  int i0[3], i1[3];
  double f[3];
};

__device__ __forceinline__ bool voxel_stencil(const VrVoxelDesc& g, const double p[3],
                                              VoxStencil& st, int near_idx[3]) {
  const bool in = p[0] >= g.box_mn[0] && p[1] >= g.box_mn[1] && p[2] >= g.box_mn[2] &&
                  p[0] <= g.box_mx[0] && p[1] <= g.box_mx[1] && p[2] <= g.box_mx[2];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double cell = (g.box_mx[a] - g.box_mn[a]) / (double)g.res[a];
    double u = (p[a] - g.box_mn[a]) / cell;
    int nidx = (int)floor(u);
    near_idx[a] = min(max(nidx, 0), g.res[a] - 1);
    u = u - 0.5;
    int i0 = (int)floor(u);
    i0 = min(max(i0, 0), max(g.res[a] - 2, 0));
    st.i0[a] = i0;
    st.i1[a] = min(i0 + 1, g.res[a] - 1);
    st.f[a] = fmin(fmax(u - (double)i0, 0.0), 1.0);
  }
  return in;
}

// F64: float64 outputs sig64[n], rgb64[n][3] (the finite-difference probe) instead of
// the training path's float4 (sigma, rgb)
template <bool F64>
__global__ void k_voxel_fwd(const VrVoxelDesc g, const double* __restrict__ dens,
                            const double* __restrict__ cols, const double* __restrict__ rays,
                            int64_t stride, const double* __restrict__ t0,
                            const double* __restrict__ t1, const int32_t* __restrict__ rid,
                            int64_t n, float4* __restrict__ out, double* __restrict__ sig64,
                            double* __restrict__ rgb64) {
  const int ny = g.res[1], nz = g.res[2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p[3];
    sample_point(rays, stride, t0, t1, rid, i, p);
    VoxStencil st;
    int nidx[3];
    if (!voxel_stencil(g, p, st, nidx)) {
      if (F64) {
        sig64[i] = 0.0;
        rgb64[3 * i] = rgb64[3 * i + 1] = rgb64[3 * i + 2] = 0.0;
      } else {
        out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      continue;
    }
    double sig = 0.0, rgb[3] = {0.0, 0.0, 0.0};
    if (!g.trilinear) {
      const int64_t v = ((int64_t)nidx[0] * ny + nidx[1]) * nz + nidx[2];
      sig = dens[v];
#pragma unroll
      for (int k = 0; k < 3; ++k) rgb[k] = cols[3 * v + k];
    } else {
#pragma unroll
      for (int cx = 0; cx < 2; ++cx)
#pragma unroll
        for (int cy = 0; cy < 2; ++cy)
#pragma unroll
          for (int cz = 0; cz < 2; ++cz) {
            const double wx = cx ? st.f[0] : 1.0 - st.f[0];
            const double wy = cy ? st.f[1] : 1.0 - st.f[1];
            const double wz = cz ? st.f[2] : 1.0 - st.f[2];
            const double w = wx * wy * wz;
            const int64_t v = ((int64_t)(cx ? st.i1[0] : st.i0[0]) * ny +
                               (cy ? st.i1[1] : st.i0[1])) * nz + (cz ? st.i1[2] : st.i0[2]);
            sig += dens[v] * w;
#pragma unroll
            for (int k = 0; k < 3; ++k) rgb[k] += cols[3 * v + k] * w;
          }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) rgb[k] = fmin(fmax(rgb[k], 0.0), 1.0);
    if (F64) {
      sig64[i] = sig;
#pragma unroll
      for (int k = 0; k < 3; ++k) rgb64[3 * i + k] = rgb[k];
    } else {
      out[i] = make_float4((float)sig, (float)rgb[0], (float)rgb[1], (float)rgb[2]);
    }
  }
}

__global__ void k_voxel_bwd(const VrVoxelDesc g, const double* __restrict__ rays, int64_t stride,
                            const double* __restrict__ t0, const double* __restrict__ t1,
                            const int32_t* __restrict__ rid, int64_t n,
                            const float4* __restrict__ dsr, double* __restrict__ gdens) {
  const int ny = g.res[1], nz = g.res[2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ds = (double)dsr[i].x;
    if (ds == 0.0) continue;
    double p[3];
    sample_point(rays, stride, t0, t1, rid, i, p);
    VoxStencil st;
    int nidx[3];
    if (!voxel_stencil(g, p, st, nidx)) continue;
    if (!g.trilinear) {
      atomicAdd(gdens + ((int64_t)nidx[0] * ny + nidx[1]) * nz + nidx[2], ds);
      continue;
    }
#pragma unroll
    for (int cx = 0; cx < 2; ++cx)
#pragma unroll
      for (int cy = 0; cy < 2; ++cy)
#pragma unroll
        for (int cz = 0; cz < 2; ++cz) {
          const double w = (cx ? st.f[0] : 1.0 - st.f[0]) * (cy ? st.f[1] : 1.0 - st.f[1]) *
                           (cz ? st.f[2] : 1.0 - st.f[2]);
          const int64_t v = ((int64_t)(cx ? st.i1[0] : st.i0[0]) * ny +
                             (cy ? st.i1[1] : st.i0[1])) * nz + (cz ? st.i1[2] : st.i0[2]);
          atomicAdd(gdens + v, w * ds);
        }
  }
}

}  // namespace vr

using namespace vr;

extern "C" int vr_field_analytic_fwd(const VrAnalyticField* f, const double* rays, int64_t stride,
                                     const double* t0, const double* t1, const int32_t* rid,
                                     int64_t n, float* out, void* stream) {
  if (!f || f->n_children < 1 || f->n_children > VR_MAX_CHILDREN || f->n_blobs < 0 ||
      f->n_blobs > VR_MAX_BLOBS || n < 0) {
    set_error("vr_field_analytic_fwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_field_analytic<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      *f, rays, stride, t0, t1, rid, n, reinterpret_cast<float4*>(out));
  return check_launch("vr_field_analytic_fwd");
}

extern "C" int vr_voxel_fwd(const VrVoxelDesc* g, const double* dens, const double* cols,
                            const double* rays, int64_t stride, const double* t0,
                            const double* t1, const int32_t* rid, int64_t n, float* out,
                            void* stream) {
  if (!g || g->res[0] < 1 || g->res[1] < 1 || g->res[2] < 1 || n < 0) {
    set_error("vr_voxel_fwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_voxel_fwd<false><<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      *g, dens, cols, rays, stride, t0, t1, rid, n, reinterpret_cast<float4*>(out), nullptr,
      nullptr);
  return check_launch("vr_voxel_fwd");
}

extern "C" int vr_voxel_fwd_f64(const VrVoxelDesc* g, const double* dens, const double* cols,
                                const double* rays, int64_t stride, const double* t0,
                                const double* t1, const int32_t* rid, int64_t n, double* sigma,
                                double* rgb, void* stream) {
  if (!g || g->res[0] < 1 || g->res[1] < 1 || g->res[2] < 1 || n < 0 ||
      (n > 0 && (!sigma || !rgb))) {
    set_error("vr_voxel_fwd_f64: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_voxel_fwd<true><<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      *g, dens, cols, rays, stride, t0, t1, rid, n, nullptr, sigma, rgb);
  return check_launch("vr_voxel_fwd_f64");
}

extern "C" int vr_voxel_bwd(const VrVoxelDesc* g, const double* rays, int64_t stride,
                            const double* t0, const double* t1, const int32_t* rid, int64_t n,
                            const float* dsr, double* gdens, void* stream) {
  if (!g || g->res[0] < 1 || g->res[1] < 1 || g->res[2] < 1 || n < 0) {
    set_error("vr_voxel_bwd: bad argument");
    return VR_ERR_BAD_ARG;
  }
  if (n == 0) return VR_OK;
  k_voxel_bwd<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      *g, rays, stride, t0, t1, rid, n, reinterpret_cast<const float4*>(dsr), gdens);
  return check_launch("vr_voxel_bwd");
}
