"""The reference's per-segment API and its gradient probe, on the GPU.

Names and semantics of segrender.py (SegmentAggregate, identity_aggregate,
aggregate_segment, compose_render, compose_distortion, ParamRef, DistributedLossProbe,
local_gradient_fd — segrender.py:51-251), quadrature.py's SampleInterval / fill_samples
(quadrature.py:22-46, :117-128) and field.py's Field protocol (field.py:46-59).

The arithmetic runs in the float64 kernels of csrc/segapi.cu (vr_segment_aggregate_f64,
vr_compose_f64) and csrc/fields.cu (vr_voxel_fwd_f64): round-to-nearest without FMA in
the reference's operation order, so composition of given packets is bitwise the
reference's and segment aggregation agrees to exp()'s last bit.  These entry points serve
per-ray callers (the reference's hand cases, the finite-difference probe); the batched
training and render path (engine.VolumePool) keeps float32 packets.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field
from typing import Protocol, runtime_checkable

import numpy as np
import torch

from . import _lib
from .engine import RayAggregate, VolumePool
from .errors import ParamNotOwnedError
from .fields import (AnalyticRegion, ConstantBox, GaussianBlobs, RegionField, Scene, SumField,
                     VoxelGrid, VoxelRegion)
from .geometry import Ray, rays_to_soa, vec3
from .partition import locate

__all__ = ["Field", "SampleInterval", "SegmentAggregate", "identity_aggregate", "fill_samples",
           "aggregate_segment", "compose_render", "compose_distortion", "ParamRef",
           "DistributedLossProbe", "local_gradient_fd", "DeviceFieldView"]


def _device(device=None) -> torch.device:
    return torch.device(device) if device is not None else torch.device("cuda")


# ---- field protocol (field.py:46-59) ------------------------------------------------------

@runtime_checkable
class Field(Protocol):
    """A radiance field: sigma >= 0 and rgb in [0, 1] at (n, 3) points."""

    def sigma_many(self, pts: np.ndarray) -> np.ndarray: ...

    def rgb_many(self, pts: np.ndarray, view_dir: np.ndarray) -> np.ndarray: ...


class DeviceFieldView:
    """The Field protocol over a device field (a RegionField, or a reference scene field
    value that maps onto one): points are evaluated by the field's kernel (float32
    sigma / rgb, as the training path sees them)."""

    def __init__(self, f, device=None):
        dev = _device(device)
        if isinstance(f, VoxelGrid):
            f = VoxelRegion(f, dev)
        elif isinstance(f, (GaussianBlobs, ConstantBox, SumField)):
            f = AnalyticRegion(f)
        if not isinstance(f, RegionField):
            raise TypeError(f"no device field for {type(f).__name__}")
        self.field, self.device = f, dev

    def _eval(self, pts, view_dir):
        pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
        n = pts.shape[0]
        rays = np.zeros((8, max(n, 1)))
        rays[0:3, :n] = pts.T
        d = vec3(view_dir) if view_dir is not None else np.array([1.0, 0.0, 0.0])
        rays[3:6] = d[:, None]
        rays[7] = 1.0
        rd = torch.from_numpy(rays).to(self.device)
        z = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)  # t0 = t1 = 0: p = o
        rid = torch.arange(max(n, 1), dtype=torch.int32, device=self.device)
        out = torch.empty((max(n, 1), 4), dtype=torch.float32, device=self.device)
        if n:
            self.field.forward(rd, z, z, rid, n, out, _lib.stream_ptr())
        return out[:n].double().cpu().numpy()

    def sigma_many(self, pts):
        return self._eval(pts, None)[:, 0]

    def rgb_many(self, pts, view_dir):
        return self._eval(pts, view_dir)[:, 1:4]


# ---- bins and packets (quadrature.py:22-46, segrender.py:51-68) ---------------------------

@dataclass
class SampleInterval:
    """One quadrature bin [t0, t1) with its midpoint, field values and owning tile."""

    t0: float
    t1: float
    sigma: float = 0.0
    rgb: np.ndarray = dc_field(default_factory=lambda: np.zeros(3))
    tile_id: int = -1

    def __post_init__(self):
        self.t0, self.t1 = float(self.t0), float(self.t1)
        if not self.t1 > self.t0:
            raise ValueError(f"degenerate bin [{self.t0}, {self.t1})")
        self.m = 0.5 * (self.t0 + self.t1)
        self.rgb = np.asarray(self.rgb, dtype=np.float64)

    @property
    def delta(self) -> float:
        return self.t1 - self.t0


@dataclass
class SegmentAggregate:
    """Per-tile per-ray packet (T, C, A, D, L) and the segment's entry distance."""

    transmittance: float
    color: np.ndarray
    alpha: float
    depth: float
    distortion: float
    order_t: float


def identity_aggregate(order_t: float = math.inf) -> SegmentAggregate:
    """The neutral segment (segrender.py:66-68)."""
    return SegmentAggregate(1.0, np.zeros(3), 0.0, 0.0, 0.0, order_t)


def fill_samples(field, ray: Ray, samples: list, device=None) -> list:
    """sigma / rgb of every bin at its midpoint, view direction = ray.dir
    (quadrature.py:117-128); ``field`` is a Field or a device field (DeviceFieldView)."""
    if not samples:
        return samples
    if not isinstance(field, Field):
        field = DeviceFieldView(field, device)
    pts = ray.points_at(np.array([s.m for s in samples]))
    sig = np.asarray(field.sigma_many(pts), dtype=np.float64)
    rgb = np.asarray(field.rgb_many(pts, ray.dir), dtype=np.float64)
    for i, s in enumerate(samples):
        s.sigma = float(sig[i])
        s.rgb = rgb[i]
    return samples


def aggregate_segments(t0, t1, sigma, rgb, seg_off, device=None) -> np.ndarray:
    """Batched aggregate_segment: float64 bins and segment offsets (host arrays or device
    tensors) -> [n_segs][8] {T, C[3], A, D, L, order_t} (vr_segment_aggregate_f64)."""
    dev = _device(device)

    def d(x, dt=torch.float64):
        return torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x,
                               dtype=dt).to(dev).contiguous()

    off = d(seg_off, torch.int64)
    n_segs = off.numel() - 1
    out = torch.empty((max(n_segs, 1), 8), dtype=torch.float64, device=dev)
    t0d, t1d, sd = d(t0), d(t1), d(sigma)
    rd = d(np.asarray(rgb).reshape(-1, 3) if not isinstance(rgb, torch.Tensor) else rgb)
    _lib.call("vr_segment_aggregate_f64", _lib.ptr(t0d), _lib.ptr(t1d), _lib.ptr(sd),
              _lib.ptr(rd), _lib.ptr(off), n_segs, _lib.ptr(out), _lib.stream_ptr())
    return out[:n_segs].cpu().numpy()


def aggregate_segment(field, ray, samples: list, device=None) -> SegmentAggregate:
    """Render one contiguous run of bins locally from T = 1 (segrender.py:71-90);
    ``field=None`` aggregates bins that already carry sigma / rgb."""
    if not samples:
        return identity_aggregate()
    if field is not None:
        fill_samples(field, ray, samples, device)
    n = len(samples)
    o = aggregate_segments([s.t0 for s in samples], [s.t1 for s in samples],
                           [s.sigma for s in samples], np.array([s.rgb for s in samples]),
                           [0, n], device)[0]
    return SegmentAggregate(float(o[0]), o[1:4].copy(), float(o[4]), float(o[5]), float(o[6]),
                            samples[0].t0)


def compose_packets(packets, counts, device=None, err=None) -> np.ndarray:
    """Batched compose: packets [R][K][7] {T, C[3], A, D, L} in (order_t, tile) order,
    counts [R] -> [R][7] {C[3], A, D, T, L} (vr_compose_f64).  Raises the reference's
    NonFiniteInputError / NegativeLossError."""
    dev = _device(device)
    p = torch.as_tensor(np.asarray(packets, dtype=np.float64)).to(dev).contiguous()
    R = p.shape[0]
    K = p.shape[1] if p.dim() == 3 else 0
    c = torch.as_tensor(np.asarray(counts, dtype=np.int32)).to(dev)
    out = torch.empty((max(R, 1), 7), dtype=torch.float64, device=dev)
    e = torch.zeros(1, dtype=torch.int32, device=dev) if err is None else err
    _lib.call("vr_compose_f64", _lib.ptr(p), _lib.ptr(c), K, R, _lib.ptr(out), _lib.ptr(e),
              _lib.stream_ptr())
    flags = int(e.item())
    if flags:
        e.zero_()
        _lib.raise_flags(flags, "in compose")
    return out[:R].cpu().numpy()


def _fold(segments: list, device=None) -> np.ndarray:
    pk = np.array([[s.transmittance, *np.asarray(s.color, dtype=np.float64), s.alpha, s.depth,
                    s.distortion] for s in segments], dtype=np.float64).reshape(1, -1, 7)
    return compose_packets(pk, [len(segments)], device)[0]


def compose_render(segments: list, device=None) -> RayAggregate:
    """Alpha-composite ordered packets (segrender.py:93-113); distortion left at 0 (use
    compose_distortion).  Non-finite packets raise NonFiniteInputError."""
    o = _fold(segments, device)
    return RayAggregate(o[0:3].copy(), float(o[3]), float(o[4]), float(o[5]), 0.0)


def compose_distortion(segments: list, device=None) -> float:
    """The composed pairwise distortion (segrender.py:116-142): T_pre^2 L_k + 2 T_pre
    (D_k A_pre - A_k D_pre) per segment; NonFiniteInputError / NegativeLossError below
    -1e-12, tinier negatives clamp to 0."""
    return float(_fold(segments, device)[6])


# ---- the gradient-locality probe (segrender.py:146-251) ------------------------------------

@dataclass(frozen=True)
class ParamRef:
    """One scalar density parameter: a voxel index in a tile's grid."""

    tile_id: int
    index: tuple


class DistributedLossProbe:
    """Finite-difference harness of the gradient-locality contract (segrender.py:146-251),
    on the GPU: every tile owns a private copy of the voxel grid (VoxelRegion), K1 caches
    each ray's bins, the float64 kernels give each tile's per-ray segment packets, and the
    loss (colour MSE against a constant target + composed distortion) is composed per ray
    in (order_t, tile) order.

      GLOBAL  re-evaluates every tile's packets for the perturbed parameter;
      LOCAL   re-evaluates only the owning tile, the others' cached packets are constants.

    ``analytic_gradient`` gives the same derivative from the training path's analytic
    backward (K5 bwd -> K4 bwd -> vr_voxel_bwd; float32 packets)."""

    def __init__(self, scene: Scene, tree, rays, dt: float, target=0.5, device=None):
        if not isinstance(scene.field, VoxelGrid):
            raise TypeError("gradient probe requires a voxel-grid scene field")
        self.dev = _device(device)
        self.scene, self.tree, self.dt = scene, tree, float(dt)
        self.target = float(target)
        self.rays = list(rays)
        self.grid = scene.field
        self.regions = [VoxelRegion(self.grid, self.dev) for _ in tree.leaves]
        self.pool = VolumePool(tree, self.regions, scene.background, self.dev)
        self.rays_dev = self.pool.rays_to_device(rays_to_soa(self.rays))
        self.b = self.pool.sample(self.rays_dev, self.dt)
        self.K, self.R = len(tree.leaves), len(self.rays)
        self._base = np.stack([self._region_packets(k) for k in range(self.K)])

    def _region_packets(self, k: int) -> np.ndarray:
        """[R][8] float64 packets {T, C[3], A, D, L, order_t} of tile k over the rays."""
        b, f = self.b, self.regions[k]
        lo, hi = b.region_slice(k)
        n = hi - lo
        sig = torch.empty(max(n, 1), dtype=torch.float64, device=self.dev)
        rgb = torch.empty((max(n, 1), 3), dtype=torch.float64, device=self.dev)
        s = _lib.stream_ptr()
        if n:
            _lib.call("vr_voxel_fwd_f64", _lib.addr(f.desc), _lib.ptr(f.densities),
                      _lib.ptr(f.colors), _lib.ptr(self.rays_dev), self.R, _lib.ptr(b.t0[lo:]),
                      _lib.ptr(b.t1[lo:]), _lib.ptr(b.ray_id[lo:]), n, _lib.ptr(sig),
                      _lib.ptr(rgb), s)
        off = (b.offsets[k * self.R:(k + 1) * self.R + 1] - lo).contiguous()
        return aggregate_segments(b.t0[lo:lo + max(n, 1)], b.t1[lo:lo + max(n, 1)], sig, rgb,
                                  off, self.dev)

    def _loss(self, packets: np.ndarray) -> float:
        """segrender.py:198-207 over [K][R][8] packets."""
        order_t = packets[:, :, 7]  # +inf for tiles without bins on the ray
        tiles = np.broadcast_to(np.arange(self.K)[:, None], order_t.shape)
        order = np.lexsort((tiles, order_t), axis=0)  # per ray, (order_t, tile)
        ordered = np.take_along_axis(packets, order[:, :, None], axis=0)  # [K][R][8]
        counts = np.isfinite(order_t).sum(axis=0)
        out = compose_packets(np.ascontiguousarray(ordered.transpose(1, 0, 2)[:, :, :7]),
                              counts, self.dev)
        bg = np.asarray(self.scene.background, dtype=np.float64)
        total = 0.0
        for r in range(self.R):
            pix = out[r, 0:3] + out[r, 5] * bg
            err = pix - self.target
            total += float(err @ err) + float(out[r, 6])
        return total

    def _check_owned(self, worker_k: int, param: ParamRef):
        idx = tuple(int(v) for v in param.index)
        res = self.grid.resolution
        if len(idx) != 3 or any(not 0 <= idx[a] < res[a] for a in range(3)):
            raise ParamNotOwnedError(f"voxel index {idx} outside grid {res}")
        owner = locate(self.tree, self.grid.voxel_center(idx))
        if param.tile_id != worker_k or owner != worker_k:
            raise ParamNotOwnedError(f"voxel {idx} (tile {owner}) is not owned by worker "
                                     f"{worker_k}")
        return idx

    def gradient_pair(self, worker_k: int, param: ParamRef, h: float):
        """(local, global) central-difference gradients (segrender.py:235-251)."""
        if h <= 0.0:
            raise ValueError("h must be > 0")
        idx = self._check_owned(worker_k, param)
        dens = self.regions[worker_k].densities
        base = float(dens[idx].item())
        res = {}
        for mode in ("local", "global"):
            vals = []
            for sign in (+1.0, -1.0):
                dens[idx] = base + sign * h
                if mode == "local":
                    pk = self._base.copy()
                    pk[worker_k] = self._region_packets(worker_k)
                else:
                    pk = np.stack([self._region_packets(k) for k in range(self.K)])
                vals.append(self._loss(pk))
                dens[idx] = base
            res[mode] = (vals[0] - vals[1]) / (2.0 * h)
        return res["local"], res["global"]

    def analytic_gradient(self, worker_k: int, param: ParamRef) -> float:
        """d loss / d density from the analytic backward of the training path."""
        idx = self._check_owned(worker_k, param)
        targets = np.full((self.R, 3), self.target)
        self.pool.zero_grad()
        self.pool.loss_and_grad(self.rays_dev, targets, self.dt)
        return float(self.regions[worker_k].grad[idx].item())


def local_gradient_fd(scene, tree, worker_k, param_ref, h, rays, dt, target=0.5, device=None):
    """One-shot (local, global) gradient pair (segrender.py:254-257)."""
    return DistributedLossProbe(scene, tree, rays, dt, target, device).gradient_pair(
        worker_k, param_ref, h)
