"""Per-region field plugins (the reference's Field seam, field.py:46-59).

Value types mirror the reference's analytic scene fields (field.py:72-240) so a
reference scene description maps one-to-one onto a GPU field.  Each ``*Region``
class is the device-resident instance one region (tile) owns — the analogue of
``tile_mask(field, leaf.box, root_box)`` handed to a worker by ``spawn``
(distsim.py:358-364): the region only ever evaluates the samples it owns, which is
exactly MaskedField's half-open ownership (field.py:243-273).

``HashGridMLP`` is the NeRF-XL per-region model (Instant-NGP hash grid + density /
colour MLPs); it has no reference code and is specified in
``csrc/hashgrid.cu``, ``csrc/mlp.cu`` and restated in ``oracle/hashmlp_oracle.py``.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from .geometry import Aabb, vec3


def _rgb(c) -> np.ndarray:
    c = vec3(c)
    if np.any(c < 0.0) or np.any(c > 1.0):
        raise ValueError(f"color components must be in [0,1], got {c}")
    return c


# ---- value types (reference field.py) -------------------------------------------------

@dataclass(frozen=True)
class GaussianBlob:
    center: np.ndarray
    amplitude: float
    scale: float
    color: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "center", vec3(self.center))
        object.__setattr__(self, "color", _rgb(self.color))
        if self.amplitude < 0.0:
            raise ValueError("blob amplitude must be >= 0")
        if self.scale <= 0.0:
            raise ValueError("blob scale must be > 0")


@dataclass(frozen=True)
class GaussianBlobs:
    blobs: tuple

    def __post_init__(self):
        object.__setattr__(self, "blobs", tuple(self.blobs))


@dataclass(frozen=True)
class ConstantBox:
    box: Aabb
    density: float
    color: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "color", _rgb(self.color))
        if self.density < 0.0:
            raise ValueError("density must be >= 0")


@dataclass(frozen=True)
class VoxelGrid:
    box: Aabb
    densities: np.ndarray
    colors: np.ndarray
    interpolation: str = "trilinear"

    def __post_init__(self):
        d = np.asarray(self.densities, dtype=np.float64)
        c = np.asarray(self.colors, dtype=np.float64)
        if d.ndim != 3 or c.shape != d.shape + (3,):
            raise ValueError("densities (nx,ny,nz) and colors (nx,ny,nz,3) expected")
        if np.any(d < 0.0) or not np.all(np.isfinite(d)):
            raise ValueError("densities must be finite and >= 0")
        if self.interpolation not in ("nearest", "trilinear"):
            raise ValueError(f"unknown interpolation {self.interpolation!r}")
        object.__setattr__(self, "densities", d)
        object.__setattr__(self, "colors", c)

    @property
    def resolution(self):
        return self.densities.shape

    def voxel_center(self, index) -> np.ndarray:
        cell = self.box.size / np.array(self.resolution, dtype=np.float64)
        return self.box.mn + (np.asarray(index, dtype=np.float64) + 0.5) * cell


@dataclass(frozen=True)
class SumField:
    children: tuple

    def __post_init__(self):
        object.__setattr__(self, "children", tuple(self.children))
        if not self.children:
            raise ValueError("sum field needs at least one child")


@dataclass(frozen=True)
class Scene:
    root_box: Aabb
    field: object
    background: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "background", _rgb(self.background))


# ---- device-resident region fields ------------------------------------------------------

class RegionField:
    """One region's field on the GPU.  ``forward`` writes sig_rgb [n,4] float32 for
    the region's samples; ``backward`` consumes d(loss)/d(sig_rgb) and accumulates
    parameter gradients."""

    trainable = False

    def forward(self, rays, t0, t1, ray_id, n, sig_rgb, stream):
        raise NotImplementedError

    def backward(self, rays, t0, t1, ray_id, n, dsig_rgb, stream, sig_rgb=None):
        """sig_rgb: the forward's output for the same samples (optional; the hash-grid
        MLP backward uses it to scale its fp16 gradient operands)."""
        raise NotImplementedError(f"{type(self).__name__} has no parameters")

    def zero_grad(self):
        pass

    def step(self, lr, step):
        pass


def analytic_desc(f) -> _lib.VrAnalyticField:
    """Flatten GaussianBlobs / ConstantBox / SumField-of-those into VrAnalyticField."""
    children = list(f.children) if isinstance(f, SumField) else [f]
    if len(children) > _lib.VR_MAX_CHILDREN:
        raise ValueError("too many sum-field children")
    d = _lib.VrAnalyticField()
    d.n_children = len(children)
    nb = 0
    for c, ch in enumerate(children):
        if isinstance(ch, GaussianBlobs):
            d.child_kind[c] = 0
            d.child_blob_lo[c] = nb
            d.child_blob_cnt[c] = len(ch.blobs)
            for b in ch.blobs:
                if nb >= _lib.VR_MAX_BLOBS:
                    raise ValueError("too many blobs")
                for a in range(3):
                    d.blobs[nb].center[a] = b.center[a]
                    d.blobs[nb].color[a] = b.color[a]
                d.blobs[nb].amplitude = b.amplitude
                d.blobs[nb].scale = b.scale
                nb += 1
        elif isinstance(ch, ConstantBox):
            d.child_kind[c] = 1
            for a in range(3):
                d.box_mn[c][a] = ch.box.mn[a]
                d.box_mx[c][a] = ch.box.mx[a]
                d.box_color[c][a] = ch.color[a]
            d.box_density[c] = ch.density
        else:
            raise TypeError(f"analytic kernel does not support {type(ch).__name__}")
    d.n_blobs = nb
    return d


class AnalyticRegion(RegionField):
    """Analytic test field (no parameters) — GaussianBlobs/ConstantBox/SumField."""

    def __init__(self, f):
        self.desc = analytic_desc(f)

    def forward(self, rays, t0, t1, ray_id, n, sig_rgb, stream):
        _lib.call("vr_field_analytic_fwd", _lib.addr(self.desc), _lib.ptr(rays),
                  rays.shape[1], _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(ray_id), n,
                  _lib.ptr(sig_rgb), stream)


class VoxelRegion(RegionField):
    """A region's private copy of a VoxelGrid (segrender.py:175-178 deep-copies the
    grid per tile); densities are the trainable parameters (float64)."""

    trainable = True

    def __init__(self, grid: VoxelGrid, device):
        self.grid = grid
        d = _lib.VrVoxelDesc()
        for a in range(3):
            d.box_mn[a] = grid.box.mn[a]
            d.box_mx[a] = grid.box.mx[a]
            d.res[a] = grid.resolution[a]
        d.trilinear = 1 if grid.interpolation == "trilinear" else 0
        self.desc = d
        self.densities = torch.from_numpy(np.ascontiguousarray(grid.densities)).to(device)
        self.colors = torch.from_numpy(np.ascontiguousarray(grid.colors)).to(device)
        self.grad = torch.zeros_like(self.densities)

    def forward(self, rays, t0, t1, ray_id, n, sig_rgb, stream):
        _lib.call("vr_voxel_fwd", _lib.addr(self.desc), _lib.ptr(self.densities),
                  _lib.ptr(self.colors), _lib.ptr(rays), rays.shape[1], _lib.ptr(t0),
                  _lib.ptr(t1), _lib.ptr(ray_id), n, _lib.ptr(sig_rgb), stream)

    def backward(self, rays, t0, t1, ray_id, n, dsig_rgb, stream, sig_rgb=None):
        _lib.call("vr_voxel_bwd", _lib.addr(self.desc), _lib.ptr(rays), rays.shape[1],
                  _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(ray_id), n, _lib.ptr(dsig_rgb),
                  _lib.ptr(self.grad), stream)

    def zero_grad(self):
        self.grad.zero_()


@dataclass(frozen=True)
class HashGridConfig:
    """Instant-NGP encoding hyper-parameters (L=16, F=2 fixed by the kernels)."""

    log2_T: int = 19
    n_levels: int = 16
    base_res: int = 16
    max_res: int = 2048

    def level_params(self):
        """Per-level (scale float32, res, dense, size) and offsets; restated
        independently in oracle/hashmlp_oracle.py."""
        L = self.n_levels
        b = math.exp((math.log(self.max_res) - math.log(self.base_res)) / max(L - 1, 1))
        T = 1 << self.log2_T
        scales, res, dense, offs = [], [], [], [0]
        for lv in range(L):
            s = np.float32(self.base_res * (b ** lv) - 1.0)
            r = int(math.ceil(float(s))) + 2
            dn = r ** 3 <= T
            size = r ** 3 if dn else T
            size = (size + 7) // 8 * 8
            scales.append(s)
            res.append(r)
            dense.append(dn)
            offs.append(offs[-1] + size)
        return scales, res, dense, offs


def hash_desc(cfg: HashGridConfig, box: Aabb) -> _lib.VrHashGridDesc:
    if cfg.n_levels != 16:
        raise ValueError("the MLP consumes exactly 16 levels x 2 features")
    scales, res, dense, offs = cfg.level_params()
    d = _lib.VrHashGridDesc()
    d.n_levels = cfg.n_levels
    d.log2_T = cfg.log2_T
    for lv in range(cfg.n_levels):
        d.scale[lv] = float(scales[lv])
        d.res[lv] = res[lv]
        d.dense[lv] = 1 if dense[lv] else 0
    for lv in range(cfg.n_levels + 1):
        d.offset[lv] = offs[lv]
    for a in range(3):
        d.box_mn[a] = box.mn[a]
        d.box_mx[a] = box.mx[a]
    return d


class HashGridMLP(RegionField):
    """A region's own Instant-NGP model: hash table (float32, [entries][2]) + density
    and colour MLP (float32 masters, fp16 copies for the kernels).  Normalisation box:
    the region's leaf box (capacity scaling) or the root box (restriction of a single
    model, used for the split-vs-single equivalence check)."""

    trainable = True

    # tables larger than this are walked level-major (one level's slice live in L2)
    LEVEL_MAJOR_BYTES = 64 << 20

    def __init__(self, cfg: HashGridConfig, box: Aabb, device, seed=0, table_init=1e-4,
                 table=None, weights=None, mlp_impl: str = "fused", hash_order: str = "auto",
                 density_only: bool = False):
        if mlp_impl not in ("fused", "fused_fwd", "tc", "cuda"):
            raise ValueError(
                "mlp_impl: 'fused' (default: gather kernel + tcgen05 MLP forward, hash-grid "
                "backward fused into the tcgen05 MLP backward), 'fused_fwd' (also the forward "
                "in one kernel), 'tc' (separate kernels) or 'cuda' (CUDA-core reference MLP)")
        if hash_order not in ("auto", "sample", "level"):
            raise ValueError("hash_order: 'auto', 'sample' (all levels per sample) or 'level' "
                             "(level-major kernels for tables larger than L2)")
        if hash_order == "level" and mlp_impl == "fused_fwd":
            raise ValueError("hash_order='level' needs a separate hash-grid forward")
        if density_only and mlp_impl not in ("fused", "tc"):
            raise ValueError("density_only runs on the tensor-core kernels (mlp_impl fused/tc)")
        self.mlp_impl = mlp_impl
        # density branch only (a proposal field: sigma is all the interlevel loss reads, so
        # the colour head is neither evaluated nor trained); rgb outputs are 0
        self.density_only = bool(density_only)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)  # replaced by the pool's
        self.cfg = cfg
        self.box = box
        self.desc = hash_desc(cfg, box)
        n_entries = int(self.desc.offset[cfg.n_levels])
        self.n_entries = n_entries
        if hash_order == "auto":
            hash_order = ("level" if n_entries * 8 > self.LEVEL_MAJOR_BYTES
                          and mlp_impl != "fused_fwd" else "sample")
        self.hash_order = hash_order
        self._pos = None
        g = torch.Generator(device="cpu").manual_seed(seed)
        if table is None:
            dg = torch.Generator(device=device).manual_seed(seed)
            table = torch.rand((n_entries, 2), generator=dg, dtype=torch.float32, device=device)
            table.mul_(2.0).sub_(1.0).mul_(table_init)
        self.table = torch.as_tensor(table, dtype=torch.float32).to(device).contiguous()
        if weights is None:
            weights = init_mlp_weights(g)
        self.weights = torch.as_tensor(weights, dtype=torch.float32).to(device).contiguous()
        self.weights16 = torch.empty(_lib.VR_MLP_NPARAMS, dtype=torch.float16, device=device)
        self.grad_table = torch.zeros_like(self.table)
        self.grad_weights = torch.zeros_like(self.weights)
        self.adam = None
        self._enc = None
        self._hash_ws = None
        self.refresh_weights()

    def refresh_weights(self, stream=None):
        _lib.call("vr_cast_f32_f16", _lib.ptr(self.weights), _lib.ptr(self.weights16),
                  _lib.VR_MLP_NPARAMS, stream if stream is not None else _lib.stream_ptr())

    def _enc_buf(self, n, dev):
        need = 16 * max(n, 1)
        if self._enc is None or self._enc.numel() < need:
            self._enc = torch.empty(need, dtype=torch.float32, device=dev)  # half2 = 4 B
        return self._enc

    def _pos_buf(self, n, dev):
        if (self._pos is None or self._pos.numel() < 3 * n
                or getattr(self, "_pos_shared", False)):
            self._pos = torch.empty(3 * max(n, 1), dtype=torch.float32, device=dev)
        self._pos_shared = False
        return self._pos

    def positions(self, n):
        """This step's normalised positions [3][n] (written by the forward), or None."""
        return self._pos if getattr(self, "_pos_n", -1) == n and self._pos is not None else None

    def _workspace(self, dev):
        if self._hash_ws is None:
            nbytes = int(_lib.load().vr_hash_bwd_workspace_bytes(_lib.addr(self.desc)))
            self._hash_ws = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=dev)
        return self._hash_ws

    def forward(self, rays, t0, t1, ray_id, n, sig_rgb, stream, pos=None):
        """pos: the same samples' normalised positions [3][n] of a field with the same
        normalisation box (the region's NeRF field for its proposal): the gathers read them
        instead of recomputing them from the rays (no second position pass, no ray loads)."""
        if n == 0:
            return
        if pos is not None:
            self.forward_hash(rays, t0, t1, ray_id, n, stream, pos=pos)
            self.forward_mlp(rays, ray_id, n, sig_rgb, stream)
            return
        enc = self._enc_buf(n, rays.device)
        if self.mlp_impl == "fused_fwd":  # K2 + K3 in one tensor-core kernel
            self._pos_n = -1  # (no positions kept: the backward recomputes them)
            _lib.call("vr_field_fwd_tc", _lib.addr(self.desc), _lib.ptr(self.table),
                      _lib.ptr(self.weights16), _lib.ptr(rays), rays.shape[1], _lib.ptr(t0),
                      _lib.ptr(t1), _lib.ptr(ray_id), n, _lib.ptr(enc), _lib.ptr(sig_rgb),
                      stream)
            return
        # measured (c3): the standalone gather kernel (2048 threads/SM) + the tensor-core
        # MLP beat the fused forward (512 threads/SM left the gathers latency-bound)
        self.forward_hash(rays, t0, t1, ray_id, n, stream)
        self.forward_mlp(rays, ray_id, n, sig_rgb, stream)

    # the two halves of the non-fused forward; VolumePool overlaps region k's MLP with
    # region k+1's gathers on a second stream (L2-bound gathers || tensor-core MLP)
    splittable = property(lambda self: self.mlp_impl != "fused_fwd")

    def forward_hash(self, rays, t0, t1, ray_id, n, stream, pos=None):
        if n == 0:
            return
        enc = self._enc_buf(n, rays.device)
        if pos is not None:  # shared positions: one pass of level-grouped gathers from them
            self._pos, self._pos_shared, self._pos_n = pos, True, n
            _lib.call("vr_hash_fwd_lm", _lib.addr(self.desc), _lib.ptr(self.table),
                      _lib.ptr(pos), n, _lib.ptr(enc), stream)
            return
        self._pos_n = n
        if self.hash_order == "level":
            self._pos_buf(n, rays.device)
            _lib.call("vr_hash_positions", _lib.addr(self.desc), _lib.ptr(rays), rays.shape[1],
                      _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(ray_id), n, _lib.ptr(self._pos),
                      stream)
            _lib.call("vr_hash_fwd_lm", _lib.addr(self.desc), _lib.ptr(self.table),
                      _lib.ptr(self._pos), n, _lib.ptr(enc), stream)
            return
        # the positions are kept for the fused backward of the same step
        _lib.call("vr_hash_fwd", _lib.addr(self.desc), _lib.ptr(self.table), _lib.ptr(rays),
                  rays.shape[1], _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(ray_id), n,
                  _lib.ptr(enc), _lib.ptr(self._pos_buf(n, rays.device)), stream)

    def forward_mlp(self, rays, ray_id, n, sig_rgb, stream):
        if n == 0:
            return
        if self.density_only:
            _lib.call("vr_mlp_fwd_tc_density", _lib.ptr(self.weights16), _lib.ptr(self._enc), n,
                      _lib.ptr(sig_rgb), stream)
            return
        _lib.call("vr_mlp_fwd" if self.mlp_impl == "cuda" else "vr_mlp_fwd_tc",
                  _lib.ptr(self.weights16), _lib.ptr(self._enc), _lib.ptr(rays), rays.shape[1],
                  _lib.ptr(ray_id), n, _lib.ptr(sig_rgb), stream)

    def backward(self, rays, t0, t1, ray_id, n, dsig_rgb, stream, sig_rgb=None, rows=None):
        """rows: optional (rows, n_rows) device tensors of vr_active_rows — only those
        samples (the ones with a non-zero upstream gradient) are processed."""
        if n == 0:
            return
        enc = self._enc  # written by the forward of the same step
        rp = (_lib.ptr(rows[0]), _lib.ptr(rows[1])) if rows is not None else (None, None)
        if self.density_only:
            self.backward_scatter(self.backward_mlp(rays, ray_id, n, dsig_rgb, stream,
                                                    sig_rgb=sig_rgb, rows=rows), n, stream,
                                  rows=rows)
            return
        if self.mlp_impl in ("fused", "fused_fwd") and self.hash_order == "sample":
            ws = self._workspace(rays.device)
            _lib.call("vr_field_bwd_tc", _lib.addr(self.desc), _lib.ptr(self.weights16),
                      _lib.ptr(enc), _lib.ptr(rays), rays.shape[1], _lib.ptr(t0), _lib.ptr(t1),
                      _lib.ptr(ray_id), n, _lib.ptr(dsig_rgb), _lib.ptr(sig_rgb),
                      _lib.ptr(self.grad_weights), _lib.ptr(self.grad_table), _lib.ptr(ws),
                      ws.numel(), _lib.ptr(self.err),
                      _lib.ptr(self._pos) if self.mlp_impl == "fused" else None, *rp, stream)
            return
        denc = torch.empty(16 * n * 2, dtype=torch.float32, device=rays.device)
        if self.mlp_impl != "cuda":
            _lib.call("vr_mlp_bwd_tc", _lib.ptr(self.weights16), _lib.ptr(enc), _lib.ptr(rays),
                      rays.shape[1], _lib.ptr(ray_id), n, _lib.ptr(dsig_rgb), _lib.ptr(sig_rgb),
                      _lib.ptr(self.grad_weights), _lib.ptr(denc), _lib.ptr(self.err), 0, *rp,
                      stream)
        else:
            if rows is not None:
                raise ValueError("the CUDA-core MLP backward takes no row list")
            _lib.call("vr_mlp_bwd", _lib.ptr(self.weights16), _lib.ptr(enc), _lib.ptr(rays),
                      rays.shape[1], _lib.ptr(ray_id), n, _lib.ptr(dsig_rgb),
                      _lib.ptr(self.grad_weights), _lib.ptr(denc), stream)
        ws = self._workspace(rays.device)
        if self.hash_order == "level":  # positions of the same step's forward
            _lib.call("vr_hash_scatter", _lib.addr(self.desc), _lib.ptr(self._pos), n,
                      _lib.ptr(denc), _lib.ptr(self.grad_table), _lib.ptr(ws), ws.numel(), 1, 0,
                      *rp, stream)
            return
        if rows is not None:  # sample-order scatter of the compact d(enc) (stored positions)
            _lib.call("vr_hash_scatter", _lib.addr(self.desc), _lib.ptr(self._pos), n,
                      _lib.ptr(denc), _lib.ptr(self.grad_table), _lib.ptr(ws), ws.numel(), 0, 0,
                      *rp, stream)
            return
        _lib.call("vr_hash_bwd", _lib.addr(self.desc), _lib.ptr(rays), rays.shape[1],
                  _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(ray_id), n, _lib.ptr(denc),
                  _lib.ptr(self.grad_table), _lib.ptr(ws), ws.numel(), stream)

    # ---- split backward: the MLP part and the hash-grid scatter as separate launches, so
    # VolumePool can run region k's scatter (L2-atomic bound) on a side stream while the
    # tensor-core MLP backward of region k+1 runs on the main stream
    # (VR_SPLIT_BELOW_MB overrides the threshold; c3 re-measured with the capped MLP grid:
    # fused 56.7 vs split 58.0 ms)
    # measured: split + side-stream scatter beats the fused kernel for level-major tables
    # (c4 NeRF) and for small tables (c4 proposals, 12 MB: 549 -> 535 ms per c4 step); the
    # fused kernel wins for mid-size L2-resident tables (c3, 49 MB: 61.3 vs 64.8 ms)
    SPLIT_BELOW_BYTES = int(os.environ.get("VR_SPLIT_BELOW_MB", "16")) << 20

    @property
    def split_backward(self):
        return self.mlp_impl in ("fused", "tc") and (
            self.density_only or self.hash_order == "level"
            or self.n_entries * 8 < self.SPLIT_BELOW_BYTES)

    @property
    def takes_rows(self):
        """Whether backward / backward_mlp / backward_scatter accept a vr_active_rows list
        (every tensor-core path; not the CUDA-core MLP nor the sample-order d(enc) scatter)."""
        if self.mlp_impl == "cuda":
            return False
        return (self.split_backward or self.hash_order == "level"
                or self.mlp_impl in ("fused", "fused_fwd"))

    def backward_mlp(self, rays, ray_id, n, dsig_rgb, stream, max_ctas: int = 0, sig_rgb=None,
                     rows=None):
        """MLP backward of the step's samples; returns d(enc) [16][n] float2 (float32).
        max_ctas: grid cap when a scatter runs beside it (0: the full persistent grid);
        sig_rgb: the forward's output (gradient scaling, vr_capi.h vr_mlp_bwd_tc);
        rows: (rows, n_rows) of vr_active_rows — d(enc) is then written at compact positions."""
        denc = torch.empty(16 * max(n, 1) * 2, dtype=torch.float32, device=rays.device)
        if n:
            _lib.call("vr_mlp_bwd_tc_density" if self.density_only else "vr_mlp_bwd_tc",
                      _lib.ptr(self.weights16), _lib.ptr(self._enc),
                      _lib.ptr(rays), rays.shape[1], _lib.ptr(ray_id), n, _lib.ptr(dsig_rgb),
                      _lib.ptr(sig_rgb), _lib.ptr(self.grad_weights), _lib.ptr(denc),
                      _lib.ptr(self.err), int(max_ctas),
                      *((_lib.ptr(rows[0]), _lib.ptr(rows[1])) if rows is not None
                        else (None, None)), stream)
        return denc

    def backward_scatter(self, denc, n, stream, max_blocks=0, rows=None):
        """Hash-grid scatter of d(enc) at the positions stored by the forward (rows: the
        backward_mlp call's row list, d(enc) at compact positions)."""
        if n == 0:
            return
        ws = self._workspace(denc.device)
        _lib.call("vr_hash_scatter", _lib.addr(self.desc), _lib.ptr(self._pos), n,
                  _lib.ptr(denc), _lib.ptr(self.grad_table), _lib.ptr(ws), ws.numel(),
                  1 if self.hash_order == "level" else 0, int(max_blocks),
                  *((_lib.ptr(rows[0]), _lib.ptr(rows[1])) if rows is not None else (None, None)),
                  stream)

    def zero_grad(self):
        self.grad_table.zero_()
        self.grad_weights.zero_()

    def step(self, lr, step, betas=(0.9, 0.99), eps=1e-15, stream=None):
        """Adam on table and MLP, then refresh the fp16 copy."""
        s = stream if stream is not None else _lib.stream_ptr()
        if self.adam is None:
            self.adam = [torch.zeros_like(self.table), torch.zeros_like(self.table),
                         torch.zeros_like(self.weights), torch.zeros_like(self.weights)]
        mt, vt, mw, vw = self.adam
        # gated on the pool's device error word: a step that flagged an error leaves the
        # parameters and moments untouched (vr_capi.h vr_adam_step)
        _lib.call("vr_adam_step", _lib.ptr(self.table), _lib.ptr(self.grad_table), _lib.ptr(mt),
                  _lib.ptr(vt), self.table.numel(), lr, betas[0], betas[1], eps, step,
                  _lib.ptr(self.err), s)
        _lib.call("vr_adam_step", _lib.ptr(self.weights), _lib.ptr(self.grad_weights),
                  _lib.ptr(mw), _lib.ptr(vw), self.weights.numel(), lr, betas[0], betas[1], eps,
                  step, _lib.ptr(self.err), s)
        self.refresh_weights(s)


def init_mlp_weights(gen: torch.Generator) -> torch.Tensor:
    """N(0, 1/fan_in) weights in the packed layout of vr_capi.h (W3c rows 3..15 zero)."""
    w = torch.zeros(_lib.VR_MLP_NPARAMS, dtype=torch.float32)
    layout = [(_lib.VR_MLP_W1D, 64, 32), (_lib.VR_MLP_W2D, 16, 64), (_lib.VR_MLP_W1C, 64, 32),
              (_lib.VR_MLP_W2C, 64, 64), (_lib.VR_MLP_W3C, 3, 64)]
    for off, rows, cols in layout:
        w[off:off + rows * cols] = torch.randn(rows * cols, generator=gen) / math.sqrt(cols)
    return w


def region_field_for(scene_field, leaf, tree, device) -> RegionField:
    """The device field a region gets from a reference-style scene (spawn semantics)."""
    if isinstance(scene_field, VoxelGrid):
        return VoxelRegion(scene_field, device)
    if isinstance(scene_field, (GaussianBlobs, ConstantBox, SumField)):
        return AnalyticRegion(scene_field)
    if isinstance(scene_field, RegionField):
        return scene_field
    raise TypeError(f"no GPU field for {type(scene_field).__name__}")


# ---- scene config JSON (field.py:7-23 schema; field.py:326-356) -----------------------

def field_from_json(d: dict):
    kind = d["type"]
    if kind == "gaussian_blobs":
        return GaussianBlobs(tuple(
            GaussianBlob(vec3(b["center"]), float(b["amplitude"]), float(b["scale"]), vec3(b["color"]))
            for b in d["blobs"]))
    if kind == "constant_box":
        return ConstantBox(Aabb.from_json(d["box"]), float(d["density"]), vec3(d["color"]))
    if kind == "voxel_grid":
        res = tuple(int(v) for v in d["resolution"])
        return VoxelGrid(Aabb.from_json(d["box"]),
                         np.asarray(d["densities"], dtype=np.float64).reshape(res),
                         np.asarray(d["colors"], dtype=np.float64).reshape(res + (3,)),
                         d.get("interpolation", "trilinear"))
    if kind == "sum":
        return SumField(tuple(field_from_json(c) for c in d["children"]))
    raise ValueError(f"unknown field type {kind!r}")


def scene_from_json(d: dict) -> Scene:
    return Scene(Aabb.from_json(d["root_box"]), field_from_json(d["field"]), vec3(d["background"]))
