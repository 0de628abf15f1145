/*
 * vr_capi.h — C ABI of the B200-native NeRF-XL ray-march / composite hot path.
 *
 * This is the drop-in boundary.  The reference (`volray`, pure Python) has no
 * FFI; every entry point below replaces one reference function or call site on
 * the tile-protocol path `distsim._run_ray` (reference pkg/src/volray/distsim.py:395-454).
 * The Python host package `paper_2404_16221_b200` binds these with ctypes and
 * mirrors the reference's Python API on top.
 *
 * Conventions:
 *  - every pointer argument named *_dev / device arrays is a caller-owned DEVICE
 *    pointer; descriptor structs (VrTree, VrAnalyticField, ...) are HOST pointers
 *    copied by value into the kernel launch;
 *  - every call is asynchronous on the caller's stream (`stream` = cudaStream_t
 *    passed as void*), returns VR_OK or a VR_ERR_* status for argument/launch
 *    errors, and never synchronises;
 *  - data-dependent failures (non-finite packets, negative composed loss, points
 *    outside the root box, capacity overflow) are OR-ed into a caller-owned device
 *    int32 flag word `err_dev`; the host reads it at its own sync point and maps
 *    bits to the reference's exceptions (VR_FLAG_* below);
 *  - rays are SoA float64, layout [8][ray_stride]: ox, oy, oz, dx, dy, dz, t_near, t_far
 *    (reference Ray, geometry.py:70-106);
 *  - samples of one rank are region-major: region kk (0..region_cnt-1) owns the
 *    contiguous range [offsets[kk*n_rays], offsets[(kk+1)*n_rays]); inside it the
 *    segment of ray r is [offsets[kk*n_rays + r], offsets[kk*n_rays + r + 1]).
 *  - a packet (reference TilePayload, distsim.py:154-180) is 8 float32:
 *    {T, Cr, Cg, Cb, A, D', L, order}; D' is depth relative to the ray's root-box
 *    entry t (ray_te), `order` holds the int32 bits of the segment's first sample
 *    index along the ray (exact replacement of order_t, distsim.py:378); an empty
 *    segment is the identity packet {1,0,0,0,0,0,0, INT32_MAX}.
 */
#ifndef VR_CAPI_H
#define VR_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VR_ABI_VERSION 1
#define VR_MAX_REGIONS 32
#define VR_MAX_BLOBS 32
#define VR_MAX_CHILDREN 8
#define VR_MAX_LEVELS 16
#define VR_PACKET_FLOATS 8
#define VR_OUT_FIELDS 7 /* r, g, b, alpha, depth, transmittance, distortion */

/* status codes */
#define VR_OK 0
#define VR_ERR_BAD_ARG 1
#define VR_ERR_CUDA 2
#define VR_ERR_UNSUPPORTED 3

/* device error-flag bits (err_dev) */
#define VR_FLAG_NONFINITE 1      /* segrender.NonFiniteInputError, segrender.py:124-127   */
#define VR_FLAG_NEG_LOSS 2       /* segrender.NegativeLossError, segrender.py:137-141     */
#define VR_FLAG_OOB 4            /* partitioner.OutOfBoundsError, partitioner.py:179-180  */
#define VR_FLAG_OVERFLOW 8       /* capacity / bin-count overflow (no reference analogue) */
#define VR_FLAG_TOO_MANY_SEGS 16 /* > VR_MAX_REGIONS non-empty segments on one ray        */
#define VR_FLAG_GRAD_OVERFLOW 32 /* a scaled MLP gradient not representable in fp16      */

/* Partition tree (reference PartitionTree/SplitNode/LeafNode, partitioner.py:51-80).
 * Internal nodes are indexed 0..n_nodes-1 with node 0 the root; a child index
 * c >= 0 is a node, c < 0 is leaf (-c - 1).  n_nodes == 0 means a single leaf. */
typedef struct VrTree {
  double root_mn[3];
  double root_mx[3];
  double leaf_mn[VR_MAX_REGIONS][3];
  double leaf_mx[VR_MAX_REGIONS][3];
  double node_plane[VR_MAX_REGIONS];
  int32_t node_axis[VR_MAX_REGIONS];
  int32_t node_low[VR_MAX_REGIONS];
  int32_t node_high[VR_MAX_REGIONS];
  int32_t n_leaves;
  int32_t n_nodes;
} VrTree;

/* Occupancy grid (the paper's per-region empty-space skipping,
 * PAPER.md:296; the reference has none): one res^3 bitfield per leaf, over
 * the leaf's own box.  bits[k * words + (c >> 5)] bit (c & 31), words = ceil(res^3 / 32),
 * c = cx + res (cy + res cz), c_a = clamp(floor(((p_a - mn_a) / (mx_a - mn_a)) * res), 0,
 * res - 1) in float64 without FMA (bit-exact in the oracle).  K1 keeps a sub-bin only
 * when the bit of its midpoint in its owner's grid is set; kept samples are indexed
 * consecutively along the ray (segments stay contiguous runs of kept samples).  bits ==
 * NULL or res == 0: every sample is kept. */
typedef struct VrOccupancy {
  const uint32_t* bits;
  int32_t res;
  int32_t pad_;
} VrOccupancy;

/* Analytic test field: a SumField (field.py:212-240) of up to VR_MAX_CHILDREN
 * children, each GaussianBlobs (field.py:88-114) or ConstantBox (field.py:117-134).
 * A plain (non-sum) field is a one-child sum; both give identical results. */
typedef struct VrBlob {
  double center[3];
  double amplitude;
  double scale;
  double color[3];
} VrBlob;

typedef struct VrAnalyticField {
  int32_t n_children;
  int32_t n_blobs;
  int32_t child_kind[VR_MAX_CHILDREN]; /* 0 = gaussian_blobs, 1 = constant_box */
  int32_t child_blob_lo[VR_MAX_CHILDREN];
  int32_t child_blob_cnt[VR_MAX_CHILDREN];
  double box_mn[VR_MAX_CHILDREN][3];
  double box_mx[VR_MAX_CHILDREN][3];
  double box_density[VR_MAX_CHILDREN];
  double box_color[VR_MAX_CHILDREN][3];
  VrBlob blobs[VR_MAX_BLOBS];
} VrAnalyticField;

/* VoxelGrid (field.py:137-209): cell-centred, clamped trilinear or nearest. */
typedef struct VrVoxelDesc {
  double box_mn[3];
  double box_mx[3];
  int32_t res[3];
  int32_t trilinear;
} VrVoxelDesc;

/* Multiresolution hash grid (Instant-NGP, named at PAPER.md:386-388; no reference
 * code — restated in oracle/hashmlp_oracle.py).  Positions are normalised with
 * u = (p - box_mn) / (box_mx - box_mn) in float64, then cast to float32. */
typedef struct VrHashGridDesc {
  int32_t n_levels;
  int32_t log2_T;
  float scale[VR_MAX_LEVELS];
  int32_t res[VR_MAX_LEVELS];
  int32_t dense[VR_MAX_LEVELS];
  int64_t offset[VR_MAX_LEVELS + 1]; /* in table entries (float2) */
  double box_mn[3];
  double box_mx[3];
} VrHashGridDesc;

/* ---- meta ------------------------------------------------------------------ */
int vr_abi_version(void);
/* 1 when tensor maps can be encoded (the driver's cuTensorMapEncodeTiled is reachable):
 * the K4 walks then stage their inputs by TMA. */
int vr_tma_available(void);
/* sizes of the descriptor structs, for host-side layout checks: out[0..4] =
 * sizeof(VrTree), sizeof(VrAnalyticField), sizeof(VrVoxelDesc), sizeof(VrHashGridDesc),
 * sizeof(VrBlob). */
int vr_struct_sizes(int64_t* out5);
const char* vr_last_error(void);
/* Checked builds (-DVR_CHECKED): device range checks at the hot global accesses (a
 * sample's ray index, hash-table entries per level) that skip a bad access and count it;
 * returns the failures since the last call and clears them (synchronises the device).
 * Release builds return -1. */
int vr_check_failures(void);
int vr_device_sync(void);

/* ---- K1: ray/region intersection + sampling ------------------------------------
 * Replaces generate_samples (quadrature.py:66-88), tile_cut_distances
 * (partitioner.py:195-206), split_at_planes (quadrature.py:91-114), locate_many
 * (partitioner.py:177-192) and the bin assignment of _run_ray (distsim.py:406-425).
 * Count pass: per owned region kk and ray r, the number of samples, and the index
 * of its first sample along the ray (INT32_MAX if none).  ray_te[r] = root-box
 * entry t (0 on a miss); ray_part[r] = bitmask of leaves whose box the ray hits
 * (distsim.py:415-419 participants); ray_total[r] = samples over ALL regions. */
int vr_sample_count(const VrTree* tree, const double* rays_dev, int64_t ray_stride,
                    int64_t n_rays, double dt, int32_t region_lo, int32_t region_cnt,
                    int32_t* counts_dev, int32_t* seg_first_dev, double* ray_te_dev,
                    uint32_t* ray_part_dev, int32_t* ray_total_dev, const VrOccupancy* occ,
                    int32_t* err_dev, void* stream);
/* occ (may be NULL) in every K1 entry point: the occupancy grid (VrOccupancy above) —
 * with it, counts / indices / samples are those of the kept (occupied) sub-bins. */
/* exclusive scan of n int32 counts into n+1 int64 offsets (offsets[n] = total) */
size_t vr_scan_workspace_bytes(int64_t n);
int vr_scan_offsets(const int32_t* counts_dev, int64_t n, int64_t* offsets_dev,
                    void* workspace_dev, size_t workspace_bytes, void* stream);
/* Fill pass: writes each owned sample's bin edges t0/t1 (float64, bit-exact with
 * the reference) and its ray index into the slots given by offsets. */
/* capacity: entries of t0/t1/ray_id; samples at positions >= capacity are dropped and
 * raise VR_FLAG_OVERFLOW (an asynchronous fill into a buffer sized before the count is
 * known; the caller compares the total with the capacity). */
int vr_sample_fill(const VrTree* tree, const double* rays_dev, int64_t ray_stride,
                   int64_t n_rays, double dt, int32_t region_lo, int32_t region_cnt,
                   const int64_t* offsets_dev, const int32_t* seg_first_dev, double* t0_dev,
                   double* t1_dev, int32_t* ray_id_dev, int64_t capacity,
                   const VrOccupancy* occ, int32_t* err_dev, void* stream);
/* One walk instead of count + fill (the same generate_samples quadrature.py:66-88 /
 * split_at_planes :91-114 / locate_many partitioner.py:177-192 replacement as the pair
 * above, for _prepare_samples distsim.py:369-373 + the assignment :406-425):
 * vr_sample_stage is vr_sample_count that also writes
 * every own sample's t0/t1 into staging buffers st0/st1 (stage_capacity entries, split in
 * vr_sample_stage_blocks(n_rays) equal slices, one per CTA; a ray reserves one slot per
 * walked bin plus one per cut); sslot_dev[r] locates the ray's staged samples.
 * stage_info_dev (2 x uint64, zeroed by the caller) receives [0] += slots reserved and
 * [1] = max slots one CTA needed: if [1] > stage_capacity / vr_sample_stage_blocks(n_rays)
 * the staging is incomplete and the caller runs vr_sample_fill (the counts are exact
 * either way).  After vr_scan_offsets, vr_sample_compact moves the staged samples to their
 * slots (the same t0/t1/ray_id vr_sample_fill writes, bit for bit).  ray_list_dev
 * (optional, n_rays + 1 int32 of scratch): with a region block smaller than the tree, a
 * thread-per-ray prefilter first settles the rays that miss the block's box, and the
 * warp-per-ray walk only visits the others. */
int64_t vr_sample_stage_blocks(int64_t n_rays);
int vr_sample_stage(const VrTree* tree, const double* rays_dev, int64_t ray_stride,
                    int64_t n_rays, double dt, int32_t region_lo, int32_t region_cnt,
                    int32_t* counts_dev, int32_t* seg_first_dev, double* ray_te_dev,
                    uint32_t* ray_part_dev, int32_t* ray_total_dev, double* st0_dev,
                    double* st1_dev, int64_t stage_capacity, int64_t* sslot_dev,
                    uint64_t* stage_info_dev, int32_t* ray_list_dev, const VrOccupancy* occ,
                    int32_t* err_dev, void* stream);
int vr_sample_compact(int64_t n_rays, int32_t region_cnt, const int32_t* counts_dev,
                      const int32_t* seg_first_dev, const int64_t* offsets_dev,
                      const int64_t* sslot_dev, const double* st0_dev, const double* st1_dev,
                      double* t0_dev, double* t1_dev, int32_t* ray_id_dev, int64_t capacity,
                      int32_t* err_dev, void* stream);
/* Owner lookup of arbitrary points (locate_many, partitioner.py:177-192). */
int vr_locate(const VrTree* tree, const double* pts_dev /*[n][3]*/, int64_t n,
              int32_t* tile_dev, int32_t* err_dev, void* stream);

/* ---- fields (the Field plugin seam, field.py:46-59 / fill_samples quadrature.py:117-128)
 * All evaluate at bin midpoints m = 0.5 (t0 + t1), p = o + m d (float64) and write
 * sig_rgb[i] = {sigma, r, g, b} (float32). */
int vr_field_analytic_fwd(const VrAnalyticField* f, const double* rays_dev, int64_t ray_stride,
                          const double* t0_dev, const double* t1_dev, const int32_t* ray_id_dev,
                          int64_t n, float* sig_rgb_dev, void* stream);
int vr_voxel_fwd(const VrVoxelDesc* g, const double* densities_dev, const double* colors_dev,
                 const double* rays_dev, int64_t ray_stride, const double* t0_dev,
                 const double* t1_dev, const int32_t* ray_id_dev, int64_t n, float* sig_rgb_dev,
                 void* stream);
/* d(loss)/d(densities) scatter-add (float64 atomics); colours are not parameters. */
int vr_voxel_bwd(const VrVoxelDesc* g, const double* rays_dev, int64_t ray_stride,
                 const double* t0_dev, const double* t1_dev, const int32_t* ray_id_dev, int64_t n,
                 const float* dsig_rgb_dev, double* grad_densities_dev, void* stream);
/* The same lookup with float64 outputs sigma_dev[n], rgb_dev[n][3] (the finite-difference
 * probe, DistributedLossProbe segrender.py:146-251, which needs float64 packets). */
int vr_voxel_fwd_f64(const VrVoxelDesc* g, const double* densities_dev,
                     const double* colors_dev, const double* rays_dev, int64_t ray_stride,
                     const double* t0_dev, const double* t1_dev, const int32_t* ray_id_dev,
                     int64_t n, double* sigma_dev, double* rgb_dev, void* stream);

/* ---- occupancy grid maintenance (csrc/occupancy.cu; the grid itself: VrOccupancy) ----
 * vr_occupancy_points: one jittered point per cell of the box's res^3 grid, written as
 * zero-length rays (rays_dev [8][res^3] float64: origin = the point, dir = +x, t = [0, 1);
 * evaluate with t0 = t1 = 0); jitter u_a = (lowbias32(seed * 0x9E3779B9 + 3 c + a) >> 8) *
 * 2^-24, point = mn + ((cell + u) / res) (mx - mn).  vr_occupancy_update: per cell, density
 * EMA d = max(decay d, sigma) from the field's output at those points (sig_rgb_dev [res^3]
 * float4), bit = d > threshold into bits_dev (ceil(res^3 / 32) words of one leaf). */
int vr_occupancy_points(const double* box_mn3, const double* box_mx3, int32_t res, uint32_t seed,
                        double* rays_dev, void* stream);
int vr_occupancy_update(const float* sig_rgb_dev, int32_t res, float decay, float threshold,
                        float* density_dev, uint32_t* bits_dev, void* stream);

/* ---- float64 segment API (aggregate_segment / compose_render / compose_distortion,
 * segrender.py:71-142) — for float64 callers (the reference's hand cases, the FD probe);
 * the training path's float32 packets are K4 / K5 below.  Round-to-nearest, no FMA, the
 * reference's operation order.  vr_segment_aggregate_f64: one segment per [seg_off[s],
 * seg_off[s+1]) of the float64 bins (t0, t1, sigma, rgb[n][3]), out[s] = {T, C[3], A, D,
 * L, order_t} (order_t = first bin's t0, +inf when empty).  vr_compose_f64: per ray its
 * n_segs[r] packets seg[r][k] = {T, C[3], A, D, L} in (order_t, tile) order -> out[r] =
 * {C[3], A, D, T, L}; VR_FLAG_NONFINITE / VR_FLAG_NEG_LOSS in err_dev (may be NULL). */
int vr_segment_aggregate_f64(const double* t0_dev, const double* t1_dev, const double* sigma_dev,
                             const double* rgb_dev, const int64_t* seg_off_dev, int64_t n_segs,
                             double* out_dev, void* stream);
int vr_compose_f64(const double* seg_dev, const int32_t* n_segs_dev, int32_t max_segs,
                   int64_t n_rays, double* out_dev, int32_t* err_dev, void* stream);

/* ---- K2: hash-grid encoding ---------------------------------------------------- */
/* enc layout: [n_levels][n] half2 (level-major, coalesced on samples).  pos_dev (may be
 * NULL) receives the normalised positions [3][n] float32 for the fused backward. */
int vr_hash_fwd(const VrHashGridDesc* g, const float* table_dev, const double* rays_dev,
                int64_t ray_stride, const double* t0_dev, const double* t1_dev,
                const int32_t* ray_id_dev, int64_t n, void* enc_dev, float* pos_dev,
                void* stream);
/* denc layout: [n_levels][n] float2; grad_table float2 scatter-add.  workspace: zero-
 * initialised device buffer of vr_hash_bwd_workspace_bytes() (left zeroed on return)
 * holding per-warp replicas of the small dense levels, whose atomics would otherwise
 * serialise on a few thousand addresses; NULL = plain atomics everywhere. */
size_t vr_hash_bwd_workspace_bytes(const VrHashGridDesc* g);
int vr_hash_bwd(const VrHashGridDesc* g, const double* rays_dev, int64_t ray_stride,
                const double* t0_dev, const double* t1_dev, const int32_t* ray_id_dev, int64_t n,
                const float* denc_dev, float* grad_table_dev, void* workspace_dev,
                size_t workspace_bytes, void* stream);
/* Level-major variants for tables larger than L2 (T = 2^22: ~0.5 GB per region): the
 * samples are walked once per level so only one level's slice is live in L2.
 * vr_hash_positions writes the normalised positions pos[3][n] float32 (computed exactly
 * as inside vr_hash_fwd); vr_hash_fwd_lm / vr_hash_bwd_lm then produce the same enc and
 * the same gradient sums as vr_hash_fwd / vr_hash_bwd (same replica workspace). */
int vr_hash_positions(const VrHashGridDesc* g, const double* rays_dev, int64_t ray_stride,
                      const double* t0_dev, const double* t1_dev, const int32_t* ray_id_dev,
                      int64_t n, float* pos_dev, void* stream);
/* number of level passes of the level-major kernels for g (one launch walks them in order
 * through a work counter) */
int vr_hash_lm_passes(const VrHashGridDesc* g);
int vr_hash_fwd_lm(const VrHashGridDesc* g, const float* table_dev, const float* pos_dev,
                   int64_t n, void* enc_dev, void* stream);
int vr_hash_bwd_lm(const VrHashGridDesc* g, const float* pos_dev, int64_t n,
                   const float* denc_dev, float* grad_table_dev, void* workspace_dev,
                   size_t workspace_bytes, void* stream);
/* General scatter from stored positions: level_major = 0 walks all levels per sample
 * (tables that fit L2), 1 as vr_hash_bwd_lm.  max_blocks > 0 launches that many 128-thread
 * blocks per pass, sized to run concurrently with the tensor-core MLP backward of the next
 * region on another stream (dedicated scatter warps next to the MLP's CTAs). */
int vr_hash_scatter(const VrHashGridDesc* g, const float* pos_dev, int64_t n,
                    const float* denc_dev, float* grad_table_dev, void* workspace_dev,
                    size_t workspace_bytes, int32_t level_major, int32_t max_blocks,
                    const int32_t* rows_dev, const int32_t* n_rows_dev, void* stream);
/* debug/parity: the 8 corner indices per (level, sample): idx[l][n][8] int32 */
int vr_hash_indices(const VrHashGridDesc* g, const double* rays_dev, int64_t ray_stride,
                    const double* t0_dev, const double* t1_dev, const int32_t* ray_id_dev,
                    int64_t n, int32_t* idx_dev, void* stream);

/* ---- K3: density + colour MLP ---------------------------------------------------
 * weights_dev: packed fp16 [W1d 64x32 | W2d 16x64 | W1c 64x32 | W2c 64x64 | W3c 16x64]
 * (row = output neuron, K-major); see VR_MLP_* offsets.  grad_dev: same packing, f32. */
#define VR_MLP_W1D 0
#define VR_MLP_W2D (VR_MLP_W1D + 64 * 32)
#define VR_MLP_W1C (VR_MLP_W2D + 16 * 64)
#define VR_MLP_W2C (VR_MLP_W1C + 64 * 32)
#define VR_MLP_W3C (VR_MLP_W2C + 64 * 64)
#define VR_MLP_NPARAMS (VR_MLP_W3C + 16 * 64)
int vr_mlp_fwd(const void* weights_dev, const void* enc_dev, const double* rays_dev,
               int64_t ray_stride, const int32_t* ray_id_dev, int64_t n, float* sig_rgb_dev,
               void* stream);
int vr_mlp_bwd(const void* weights_dev, const void* enc_dev, const double* rays_dev,
               int64_t ray_stride, const int32_t* ray_id_dev, int64_t n,
               const float* dsig_rgb_dev, float* grad_weights_dev, float* denc_dev,
               void* stream);
/* Same MLP on the 5th-gen tensor cores (tcgen05.mma kind::f16, TMEM accumulators,
 * persistent 128-sample tiles).  The production path; vr_mlp_fwd / vr_mlp_bwd are the
 * CUDA-core reference kernels it is tested against.  The backward raises
 * VR_FLAG_GRAD_OVERFLOW in err_dev if a result is not finite (a scaled gradient operand
 * overflowed fp16, or a non-finite upstream gradient): checked on d(enc) and the flushed
 * weight gradients, not per operand. */
int vr_mlp_fwd_tc(const void* weights_dev, const void* enc_dev, const double* rays_dev,
                  int64_t ray_stride, const int32_t* ray_id_dev, int64_t n, float* sig_rgb_dev,
                  void* stream);
/* max_ctas: 0 = the persistent grid (2 CTAs per SM); fewer leave SMs to a kernel running
 * beside it (the split backward's side-stream scatter: 1.25 CTAs per SM measured best).
 * sig_rgb_dev (may be NULL): the forward's output for these samples; with it each CTA
 * scales its gradients by a power of two so that the fp16 hi + lo split of the upstream
 * gradients keeps full precision (without it: 2^-24 absolute precision, ~4e-5 relative
 * at the typical |dL/dsigma| ~ 1e-3), and unscales d(enc) and the weight gradients. */
int vr_mlp_bwd_tc(const void* weights_dev, const void* enc_dev, const double* rays_dev,
                  int64_t ray_stride, const int32_t* ray_id_dev, int64_t n,
                  const float* dsig_rgb_dev, const float* sig_rgb_dev, float* grad_weights_dev,
                  float* denc_dev, int32_t* err_dev, int32_t max_ctas,
                  const int32_t* rows_dev, const int32_t* n_rows_dev, void* stream);

/* Density branch only (proposal fields of the interlevel loss, whose colour head is never
 * read): out[i] = {sigma, 0, 0, 0}; the backward reads dL/dsigma (dsig_rgb[i].x), writes
 * d(enc) and accumulates the W1d / W2d gradients only. */
int vr_mlp_fwd_tc_density(const void* weights_dev, const void* enc_dev, int64_t n,
                          float* sig_rgb_dev, void* stream);
int vr_mlp_bwd_tc_density(const void* weights_dev, const void* enc_dev, const double* rays_dev,
                          int64_t ray_stride, const int32_t* ray_id_dev, int64_t n,
                          const float* dsig_rgb_dev, const float* sig_rgb_dev,
                          float* grad_weights_dev, float* denc_dev, int32_t* err_dev,
                          int32_t max_ctas, const int32_t* rows_dev, const int32_t* n_rows_dev,
                          void* stream);

/* ---- K2 + K3 fused (production training path) ------------------------------------
 * Forward: the tensor-core MLP kernel computes each row's hash encoding itself (no
 * encoding round trip through HBM before the MLP) and, if enc_out != NULL, writes it
 * (level-major half2) for the backward.  Backward: the MLP backward scatters the
 * hash-grid gradients straight from its last epilogue (no d(enc) round trip);
 * workspace as for vr_hash_bwd; pos_dev (may be NULL: recomputed from the rays) are the
 * normalised positions written by vr_hash_fwd / vr_hash_positions for these samples. */
int vr_field_fwd_tc(const VrHashGridDesc* g, const float* table_dev, const void* weights_dev,
                    const double* rays_dev, int64_t ray_stride, const double* t0_dev,
                    const double* t1_dev, const int32_t* ray_id_dev, int64_t n, void* enc_out_dev,
                    float* sig_rgb_dev, void* stream);
int vr_field_bwd_tc(const VrHashGridDesc* g, const void* weights_dev, const void* enc_dev,
                    const double* rays_dev, int64_t ray_stride, const double* t0_dev,
                    const double* t1_dev, const int32_t* ray_id_dev, int64_t n,
                    const float* dsig_rgb_dev, const float* sig_rgb_dev, float* grad_weights_dev,
                    float* grad_table_dev, void* workspace_dev, size_t workspace_bytes,
                    int32_t* err_dev, const float* pos_dev, const int32_t* rows_dev,
                    const int32_t* n_rows_dev, void* stream);

/* ---- Active rows of a backward (sparse backward) ---------------------------------
 * Samples whose upstream gradient dsig_rgb[i] (float4) is exactly zero contribute exactly
 * zero to every parameter gradient (d(enc) = 0, no weight-gradient term), and behind an
 * opaque surface most do (transmittance underflows to 0 in float32).  vr_active_rows
 * writes the indices of the others, in increasing order, to rows_dev[0, m) and m to
 * *n_rows_dev (device memory: no host sync).  NaN / inf upstream values count as active
 * (the kernels downstream flag them).  Workspace: vr_active_rows_workspace_bytes(n).
 * The backward kernels above take (rows_dev, n_rows_dev) — both NULL = every sample —
 * and then cut their 128-row tiles from the list; vr_mlp_bwd_tc* write d(enc) at the
 * compact position j of sample rows[j] (denc[l][j], row stride still n), and
 * vr_hash_scatter reads it there with the position of sample rows[j]. */
size_t vr_active_rows_workspace_bytes(int64_t n);
int vr_active_rows(const float* dsig_rgb_dev, int64_t n, int32_t* rows_dev, int32_t* n_rows_dev,
                   void* workspace_dev, size_t workspace_bytes, void* stream);

/* ---- K4: per-segment front-to-back composite (composite_samples quadrature.py:141-165,
 * aggregate_segment segrender.py:71-90, process_inbox distsim.py:318-329) ------------- */
/* n_samples: the number of samples in t0 / t1 / sig_rgb, or 0: with it the walk stages each
 * chunk's inputs into shared memory by TMA (cp.async.bulk.tensor) — t0 and t1 must then be
 * allocated with an even number (>= n_samples) of elements, 16-byte aligned, since the
 * copies read 16-byte pairs; with 0 every lane loads its own samples.
 * seg_totals_dev (optional, [region_cnt * n_rays][7] float64): each non-empty segment's
 * totals {T, C[3], A, D, L} before the float32 rounding of its packet, for
 * vr_segment_bwd (which otherwise recomputes them in a first sweep). */
int vr_segment_fwd(const double* t0_dev, const double* t1_dev, const float* sig_rgb_dev,
                   const int64_t* offsets_dev, const int32_t* seg_first_dev,
                   const double* ray_te_dev, int64_t n_rays, int32_t region_cnt,
                   float* packets_dev, double* seg_totals_dev, int32_t* err_dev,
                   int64_t n_samples, void* stream);
/* Sample-broadcast protocol (distsim.py:311-316, _compose_samples distsim.py:385-392):
 * move per-sample elements (4, 8 or 16 bytes) between the region-major K1 layout and a
 * ray-major layout (ray_off = exclusive scan of per-ray totals, a ray's segments in t
 * order via seg_first), so vr_segment_fwd/bwd with region_cnt = 1 composite whole rays. */
int vr_segment_permute(const int64_t* offsets_dev, const int32_t* seg_first_dev,
                       const int64_t* ray_offsets_dev, int64_t n_rays, int32_t n_regions,
                       const void* src_dev, void* dst_dev, int32_t elem_bytes,
                       int32_t to_ray_major, void* stream);
/* Sparse packet exchange (the transit of TilePayloads, distsim.py:333-344 / :435-446:
 * only participating segments travel).  vr_packets_pack writes the packets of this
 * rank's non-empty segments (counts > 0) as records {global slab index (int32 bits), 8
 * packet floats[, extra]} into rows 1..n of out [capacity + 1][width] (width 9, or 10
 * with extra = per-segment proposal transmittance [region_cnt][n_rays]); row 0 holds n
 * (int32 bits); count_dev receives n; n > capacity raises VR_FLAG_OVERFLOW.
 * vr_packets_unpack takes world such buffers back to back ([world][rows][width]), fills
 * slab [n_regions][n_rays][8] with identity packets (and extra_slab with 1) and scatters
 * every record: the same slab the dense all-gather of vr_segment_fwd outputs gives. */
int vr_packets_pack(const float* packets_dev, const float* extra_dev, const int32_t* counts_dev,
                    int64_t n_rays, int32_t region_lo, int32_t region_cnt, float* out_dev,
                    int64_t capacity, int32_t* count_dev, int32_t* err_dev, void* stream);
int vr_packets_unpack(const float* recv_dev, int32_t world, int64_t rows, int32_t width,
                      int64_t n_rays, int32_t n_regions, float* slab_dev, float* extra_slab_dev,
                      int32_t* err_dev, void* stream);
/* Instead of a dense slab: index_dev [n_regions][n_rays] int32 = the slot
 * (rank * rows + i) of segment (k, r)'s record in recv_dev, -1 for an empty segment — 4 B
 * per segment instead of the slab's 32 B write and read.  The *_records variants of K5 and
 * the interlevel prefix read the packets through it (bit-identical results). */
int vr_packets_index(const float* recv_dev, int32_t world, int64_t rows, int32_t width,
                     int64_t n_rays, int32_t n_regions, int32_t* index_dev, int32_t* err_dev,
                     void* stream);
/* analytic backward: dpackets [region_cnt][n_rays][8] = adjoints of {T,C,A,D',L};
 * writes dsig_rgb[i] = {dL/dsigma, dL/dr, dL/dg, dL/db}. */
/* transmittance only (the T of composite_samples quadrature.py:141-165 per run):
 * T_dev[seg] = the T of vr_segment_fwd's packet (1 for an empty segment),
 * [region_cnt][n_rays] float32 — the proposal fields' packets (interlevel) */
int vr_segment_transmittance(const double* t0_dev, const double* t1_dev,
                             const float* sig_rgb_dev, const int64_t* offsets_dev,
                             int64_t n_rays, int32_t region_cnt, float* T_dev, void* stream);
int vr_segment_bwd(const double* t0_dev, const double* t1_dev, const float* sig_rgb_dev,
                   const int64_t* offsets_dev, const double* ray_te_dev, int64_t n_rays,
                   int32_t region_cnt, const float* dpackets_dev,
                   const double* seg_totals_dev /* from vr_segment_fwd, or NULL */,
                   float* dsig_rgb_dev, void* stream);

/* ---- K5: global composite (compose_render segrender.py:93-110, compose_distortion
 * segrender.py:113-142, _compose_tile distsim.py:376-382) --------------------------
 * packets: all regions' slab [n_regions][n_rays][8].  out: [7][n_rays] float32
 * (r, g, b, alpha, depth, T, L); clip_bg != 0 writes clip(C + T*bg, 0, 1) into r,g,b
 * (render_image distsim.py:531), else the raw composed colour. */
int vr_global_fwd(const float* packets_dev, int32_t n_regions, int64_t n_rays,
                  const double* ray_te_dev, const float* background3, int32_t clip_bg,
                  float* out_dev, int32_t* err_dev, void* stream);
/* training: loss_r = |C + T*bg - target|^2 + lambda * L (segrender.py:198-207);
 * writes ray_loss[r] (float64) and the packet adjoints of regions
 * [own_lo, own_lo + own_cnt) into dpackets [own_cnt][n_rays][8]. */
int vr_global_train(const float* packets_dev, int32_t n_regions, int64_t n_rays,
                    const double* ray_te_dev, const float* background3,
                    const float* targets_dev /*[n_rays][3]*/, float lambda_dist, int32_t own_lo,
                    int32_t own_cnt, float* out_dev, double* ray_loss_dev, float* dpackets_dev,
                    int32_t* err_dev, void* stream);
/* the same two, reading the exchanged records through vr_packets_index's index */
int vr_global_fwd_records(const float* recv_dev, int32_t width, const int32_t* index_dev,
                          int32_t n_regions, int64_t n_rays, const double* ray_te_dev,
                          const float* background3, int32_t clip_bg, float* out_dev,
                          int32_t* err_dev, void* stream);
int vr_global_train_records(const float* recv_dev, int32_t width, const int32_t* index_dev,
                            int32_t n_regions, int64_t n_rays, const double* ray_te_dev,
                            const float* background3, const float* targets_dev,
                            float lambda_dist, int32_t own_lo, int32_t own_cnt, float* out_dev,
                            double* ray_loss_dev, float* dpackets_dev, int32_t* err_dev,
                            void* stream);
/* ---- interlevel (proposal) loss — no reference code (spec in
 * csrc/interlevel.cu and oracle/grad_oracle.py).  vr_prefix_train: NeRF and proposal
 * transmittance in front of each owned segment, prefix [own_cnt][n_rays][2] float32,
 * from the exchanged packets and the exchanged proposal transmittances prop_T
 * [n_regions][n_rays].  vr_interlevel: per-segment loss (float64 [region_cnt][n_rays])
 * and d(loss)/d(proposal sigma) into dsig_prop[i].x (float4, other lanes zero).
 * dsig_prop_dev is also the kernel's scratch (its first sweep parks a double2 in each
 * sample's 16-byte slot, the second overwrites it with the float4 result): it must be
 * 16-byte aligned and must not alias sig_rgb_dev or sig_prop_dev (VR_ERR_BAD_ARG). */
int vr_prefix_train(const float* packets_dev, const float* prop_T_dev, int32_t n_regions,
                    int64_t n_rays, int32_t own_lo, int32_t own_cnt, float* prefix_dev,
                    void* stream);
/* the same from width-10 records (the proposal T in field 9) through vr_packets_index */
int vr_prefix_train_records(const float* recv_dev, const int32_t* index_dev, int32_t n_regions,
                            int64_t n_rays, int32_t own_lo, int32_t own_cnt, float* prefix_dev,
                            void* stream);
int vr_interlevel(const double* t0_dev, const double* t1_dev, const float* sig_rgb_dev,
                  const float* sig_prop_dev, const int64_t* offsets_dev, const float* prefix_dev,
                  int64_t n_rays, int32_t region_cnt, float lambda_interlevel, float eps,
                  double* seg_loss_dev, float* dsig_prop_dev, void* stream);

/* deterministic float64 sum (fixed reduction tree) — the probe's loss total
 * (segrender.py:198-207 sums per-ray terms); ws_dev: VR_SUM_PARTIALS doubles of
 * caller-owned scratch (stream-ordered like every buffer here) */
#define VR_SUM_PARTIALS 296
int vr_sum_f64(const double* x_dev, int64_t n, double* out_dev, double* ws_dev, void* stream);

/* ---- optimiser ------------------------------------------------ */
/* Adam (torch.optim.Adam semantics, no weight decay).  err_dev (may be NULL): the step's
 * device error word; when it is non-zero at the time the kernel runs (an earlier kernel
 * of the step flagged a non-finite packet, a negative distortion or an overflow) the
 * update is skipped, so a poisoned gradient never reaches the parameters or the moments
 * (segrender.py:124-141 raises before the value is used). */
int vr_adam_step(float* param_dev, const float* grad_dev, float* m_dev, float* v_dev, int64_t n,
                 float lr, float beta1, float beta2, float eps, int32_t step,
                 const int32_t* err_dev, void* stream);
/* fp32 master -> fp16 copy (MLP weights) */
int vr_cast_f32_f16(const float* src_dev, void* dst_dev, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VR_CAPI_H */
