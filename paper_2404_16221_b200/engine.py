"""Per-rank engine: the B200 replacement of the reference's tile protocol.

Reference call stack replaced (distsim._run_ray, distsim.py:395-454):

    _prepare_samples + bin assignment   -> K1  vr_sample_stage / vr_scan_offsets / vr_sample_compact
    Worker.process_inbox: fill_samples  -> region field kernels (analytic / voxel / hash+MLP)
    Worker.process_inbox: composite     -> K4  vr_segment_fwd        (one packet per segment)
    transit + stats.record              -> vr_packets_pack, NCCL all-gather / gather,
                                           vr_packets_unpack (records of non-empty segments)
    _compose_tile / _broadcast_compose  -> K5  vr_global_fwd / vr_global_train
    (no reference)                      -> K5 bwd, K4 bwd, field bwd, Adam

One ``VolumePool`` per process (one process per GPU).  Rank r owns a contiguous
block of regions; every rank sees the whole (replicated) ray batch and produces
samples only for its own regions.
"""
from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, comm
from .errors import ProtocolMismatchError
from .fields import RegionField, Scene, region_field_for
from .geometry import Aabb, Camera, Ray, camera_rays, rays_to_soa, vec3
from .partition import PartitionTree
from .stats import COMPOSITOR, SCALARS_PER_SAMPLE, SCALARS_PER_TILE_PACKET, CommStats

PROTOCOLS = ("mono", "sample_broadcast", "tile_aggregate")
_ALIASES = {"sample": "sample_broadcast", "tile": "tile_aggregate"}


def canonical_protocol(name: str) -> str:
    name = _ALIASES.get(name, name)
    if name not in PROTOCOLS:
        raise ValueError(f"unknown protocol {name!r}; choose from {PROTOCOLS + tuple(_ALIASES)}")
    return name


@dataclass
class PacketRecords:
    """The sparse exchange's received records ([world * rows][width] float32: {global slab
    index, packet (, proposal T)}) with the [K][R] int32 index of their slots
    (vr_packets_index; -1 = empty segment): K5 and the interlevel prefix read the packets
    through it instead of a dense [K][R][8] slab."""
    recv: torch.Tensor
    width: int
    index: torch.Tensor
    n_regions: int


def _even(n: int) -> int:
    """Sample buffers hold an even number of float64: the K4 walks stage them by TMA in
    16-byte pairs."""
    return n + (n & 1)


@dataclass
class SampleBatch:
    """K1 output for one rank: region-major sample SoA plus per-segment metadata."""

    n_rays: int
    region_lo: int
    region_cnt: int
    counts: torch.Tensor  # int32 [cnt*R]
    seg_first: torch.Tensor  # int32 [cnt*R]
    offsets: torch.Tensor  # int64 [cnt*R + 1]
    ray_te: torch.Tensor  # float64 [R]
    ray_part: torch.Tensor  # int32 [R] (uint32 leaf-hit bitmask)
    ray_total: torch.Tensor  # int32 [R]
    t0: torch.Tensor  # float64 [N]
    t1: torch.Tensor  # float64 [N]
    ray_id: torch.Tensor  # int32 [N]
    region_bounds: list  # host: sample offset of each owned region, len cnt+1
    # sparse packet exchange: max over ranks of the non-empty segments (None: dense)
    seg_max: int | None = None

    @property
    def n_samples(self) -> int:
        return self.region_bounds[-1]

    def region_slice(self, kk: int):
        lo, hi = self.region_bounds[kk], self.region_bounds[kk + 1]
        return lo, hi


@dataclass
class RayAggregate:
    """Composed per-ray result (quadrature.py:49-59)."""

    color: np.ndarray
    alpha: float
    depth: float
    transmittance: float
    distortion: float


class VolumePool:
    """GPU-resident analogue of WorkerPool (distsim.py:347-364) for one rank."""

    def __init__(self, tree: PartitionTree, fields, background=(0.0, 0.0, 0.0), device=None,
                 rank: int = 0, world: int = 1, group=None, proposals=None):
        self.tree = tree
        self.tree_c = tree.to_c()
        self.n_regions = len(tree.leaves)
        self.rank, self.world, self.group = rank, world, group
        self.region_lo, self.region_cnt = comm.owned_regions(self.n_regions, rank, world)
        if len(fields) != self.region_cnt:
            raise ValueError(f"need {self.region_cnt} region fields, got {len(fields)}")
        self.fields = list(fields)
        # optional per-region proposal (density) fields for the interlevel loss
        self.proposals = list(proposals) if proposals is not None else None
        if self.proposals is not None and len(self.proposals) != self.region_cnt:
            raise ValueError("one proposal field per owned region")
        # a trainable field keeps per-step state (encodings, positions, gradients, scatter
        # workspace): one instance may serve only one region
        trainable = [f for f in self.fields + (self.proposals or []) if f.trainable]
        if len({id(f) for f in trainable}) != len(trainable):
            raise ValueError("each region needs its own trainable field instance (a shared "
                             "instance would mix the regions' encodings and gradients)")
        self.background = np.asarray(background, dtype=np.float64)
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._rows_ws = None  # vr_active_rows workspace
        for f in self.fields + (self.proposals or []):
            if hasattr(f, "err"):
                f.err = self.err  # kernels of the fields report into the pool's flag word
        self._ws = None
        self._side = None
        self.overlap_regions = os.environ.get("VR_OVERLAP_FWD", "0") == "1"
        # split backward (MLP here, hash-grid scatter on a side stream) for the fields that
        # prefer it (HashGridMLP.split_backward); the others use the fused tensor-core kernel
        # (vr_field_bwd_tc), measured faster on c3 (61.3 vs 64.8 ms: the MLP's shared-memory
        # traffic queues behind the scatter's atomics either way, and the fused kernel has no
        # d(enc) round trip).  On c4 the split pipeline saves ~15 ms of 550.
        self.overlap_backward = os.environ.get("VR_OVERLAP_BWD", "1") != "0"
        # sparse exchange: K5 reads the received records through an index (VR_RECORDS_K5=0:
        # rebuild the dense slab first, vr_packets_unpack)
        self.records_k5 = os.environ.get("VR_RECORDS_K5", "1") != "0"
        # K1 in one walk (count + staging, then a compaction copy) instead of count + fill
        self.stage_k1 = os.environ.get("VR_K1_STAGE", "1") != "0"
        self.stage_slots_per_ray = 96  # initial staging size; grown after an overflow
        # multi-rank K1: thread-per-ray prefilter of the rays that miss the own regions
        self.k1_prefilter = os.environ.get("VR_K1_PREFILTER", "1") != "0"
        # packets of non-empty segments only cross the link (dense slab if "0")
        self.sparse_exchange = os.environ.get("VR_SPARSE_EXCHANGE", "1") != "0"
        self._bg = (ctypes.c_float * 3)()
        # occupancy grid: bits of EVERY region (K1 indexes samples along
        # the whole ray, so each rank needs all regions' bits), density EMA of the own ones
        self.occ_bits = None
        self.occ_res = 0
        self._occ_density = None
        self._occ_desc = _lib.VrOccupancy()
        _lib.load()

    @property
    def num_workers(self) -> int:
        return self.n_regions

    # ---- helpers ----------------------------------------------------------------------
    def _side_stream(self):
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def _stream(self):
        return _lib.stream_ptr()

    def check(self, where: str = "") -> None:
        """Read and clear the device error word; raise the reference exception."""
        flags = int(self.err.item())
        if flags:
            self.err.zero_()
            _lib.raise_flags(flags, where)

    @staticmethod
    def _flag_stage(flags: int) -> str:
        """Which kernels of a training step set these flags."""
        if flags & (_lib.VR_FLAG_NONFINITE | _lib.VR_FLAG_NEG_LOSS):
            return "in the global composite (K5)"
        if flags & _lib.VR_FLAG_GRAD_OVERFLOW:
            return "in the field backward (tensor-core MLP)"
        if flags & (_lib.VR_FLAG_OVERFLOW | _lib.VR_FLAG_TOO_MANY_SEGS):
            return "in the packet exchange"
        return "in the training step"

    def rays_to_device(self, rays) -> torch.Tensor:
        if isinstance(rays, torch.Tensor):
            t = rays
        else:
            t = torch.from_numpy(np.ascontiguousarray(rays, dtype=np.float64))
        if t.dtype != torch.float64 or t.dim() != 2 or t.shape[0] != 8:
            raise ValueError("rays must be float64 SoA [8][R]")
        return t.to(self.device, non_blocking=True).contiguous()

    def _sum_scratch(self) -> torch.Tensor:
        if getattr(self, "_sum_ws", None) is None:
            self._sum_ws = torch.empty(_lib.VR_SUM_PARTIALS, dtype=torch.float64,
                                       device=self.device)
        return self._sum_ws

    def _workspace(self, n: int) -> torch.Tensor:
        need = int(_lib.load().vr_scan_workspace_bytes(n))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    # ---- occupancy grid ------------------------------------------------------------------
    def _occ_arg(self):
        return _lib.addr(self._occ_desc) if self.occ_res else None

    @staticmethod
    def occupancy_words(res: int) -> int:
        return (res ** 3 + 31) // 32

    def set_occupancy(self, bits, res: int) -> None:
        """Install an occupancy grid: bits [n_regions][occupancy_words(res)] (int32 / uint32
        words, VrOccupancy layout in vr_capi.h) for every region, or None to sample
        everything.  Samples in empty cells are skipped by K1 from the next sample()."""
        if bits is None:
            self.occ_bits, self.occ_res = None, 0
            self._occ_desc.bits, self._occ_desc.res = None, 0
            return
        t = torch.as_tensor(bits)
        if t.dtype not in (torch.int32, torch.uint32):
            t = torch.as_tensor(np.ascontiguousarray(np.asarray(bits, dtype=np.uint32)).view(
                np.int32))
        t = t.view(torch.int32).to(self.device).contiguous()
        if tuple(t.shape) != (self.n_regions, self.occupancy_words(res)):
            raise ValueError(f"occupancy bits must be [{self.n_regions}][{self.occupancy_words(res)}]")
        self.occ_bits, self.occ_res = t, int(res)
        self._occ_desc.bits = t.data_ptr()
        self._occ_desc.res = int(res)

    @staticmethod
    def pack_occupancy(mask) -> np.ndarray:
        """bool [n_regions][res][res][res] (indexed [cz][cy][cx]) -> uint32 words."""
        m = np.asarray(mask, dtype=bool)
        k, res = m.shape[0], m.shape[1]
        flat = m.reshape(k, -1)
        pad = (-flat.shape[1]) % 32
        flat = np.concatenate([flat, np.zeros((k, pad), dtype=bool)], axis=1)
        return np.packbits(flat, axis=1, bitorder="little").view("<u4").reshape(k, -1)

    def update_occupancy(self, res: int = 128, threshold: float = 0.01, decay: float = 0.95,
                         seed: int = 0, fields=None) -> float:
        """One Instant-NGP-style grid update: every owned region's field at one jittered
        point per cell (vr_occupancy_points), density EMA and threshold
        (vr_occupancy_update); the ranks' bits are all-gathered.  Returns the occupied
        fraction of the owned cells."""
        fields = self.fields if fields is None else fields
        res = int(res)
        words = self.occupancy_words(res)
        n = res ** 3
        if self._occ_density is None or self._occ_density.shape != (self.region_cnt, n):
            self._occ_density = torch.zeros((self.region_cnt, n), dtype=torch.float32,
                                            device=self.device)
        own = torch.empty((self.region_cnt, words), dtype=torch.int32, device=self.device)
        s = self._stream()
        rays = torch.empty((8, n), dtype=torch.float64, device=self.device)
        z = torch.zeros(n, dtype=torch.float64, device=self.device)
        rid = torch.arange(n, dtype=torch.int32, device=self.device)
        sig = torch.empty((n, 4), dtype=torch.float32, device=self.device)
        for kk, f in enumerate(fields):
            leaf = self.tree.leaves[self.region_lo + kk].box
            mn = (ctypes.c_double * 3)(*leaf.mn)
            mx = (ctypes.c_double * 3)(*leaf.mx)
            _lib.call("vr_occupancy_points", _lib.addr(mn), _lib.addr(mx), res,
                      (int(seed) * 1000003 + self.region_lo + kk) & 0xFFFFFFFF, _lib.ptr(rays), s)
            f.forward(rays, z, z, rid, n, sig, s)
            _lib.call("vr_occupancy_update", _lib.ptr(sig), res, float(decay), float(threshold),
                      _lib.ptr(self._occ_density[kk]), _lib.ptr(own[kk]), s)
        allb = comm.all_gather_packets(own, self.group, self.world)
        self.set_occupancy(allb, res)
        frac = (self._occ_density > threshold).float().mean()
        return float(frac.item())

    # ---- K1 ----------------------------------------------------------------------------
    def sample(self, rays: torch.Tensor, dt: float, all_regions: bool = False,
               stats: bool = False, exchange: bool = False) -> SampleBatch:
        """K1 for the owned regions (or every region: sample-broadcast protocol).  stats:
        also the per-ray participation masks and sample totals (reference CommStats) —
        this makes the kernel walk every ray entirely; without it a rank skips the rays and
        bins that cannot reach its regions.  exchange: the batch's packets will be
        exchanged (collective: every rank calls it) — size the sparse exchange here, in
        the step's one host sync."""
        if not dt > 0.0:
            raise ValueError("dt must be > 0")
        R = rays.shape[1]
        region_lo, cnt = (0, self.n_regions) if all_regions else (self.region_lo,
                                                                  self.region_cnt)
        dev = self.device
        s = self._stream()
        counts = torch.empty(cnt * R, dtype=torch.int32, device=dev)
        seg_first = torch.empty(cnt * R, dtype=torch.int32, device=dev)
        ray_te = torch.empty(R, dtype=torch.float64, device=dev)
        full = stats or all_regions
        ray_part = torch.empty(R, dtype=torch.int32, device=dev) if full else None
        ray_total = torch.empty(R, dtype=torch.int32, device=dev) if full else None
        tc = _lib.addr(self.tree_c)
        stage = self.stage_k1 and R > 0
        if stage:  # one walk: count + staging (vr_sample_stage), compaction after the scan
            blocks = int(_lib.load().vr_sample_stage_blocks(R))
            st0, st1 = self._staging(R)
            info = torch.zeros(2, dtype=torch.int64, device=dev)
            sslot = torch.empty(R, dtype=torch.int64, device=dev)
            ray_list = (torch.empty(R + 1, dtype=torch.int32, device=dev)
                        if self.k1_prefilter else None)
            _lib.call("vr_sample_stage", tc, _lib.ptr(rays), rays.shape[1], R, float(dt),
                      region_lo, cnt, _lib.ptr(counts), _lib.ptr(seg_first), _lib.ptr(ray_te),
                      _lib.ptr(ray_part), _lib.ptr(ray_total), _lib.ptr(st0), _lib.ptr(st1),
                      st0.numel(), _lib.ptr(sslot), _lib.ptr(info), _lib.ptr(ray_list),
                      self._occ_arg(), _lib.ptr(self.err), s)
        else:
            _lib.call("vr_sample_count", tc, _lib.ptr(rays), rays.shape[1], R, float(dt),
                      region_lo, cnt, _lib.ptr(counts), _lib.ptr(seg_first), _lib.ptr(ray_te),
                      _lib.ptr(ray_part), _lib.ptr(ray_total), self._occ_arg(), _lib.ptr(self.err),
                      s)
        offsets = torch.empty(cnt * R + 1, dtype=torch.int64, device=dev)
        ws = self._workspace(cnt * R)
        _lib.call("vr_scan_offsets", _lib.ptr(counts), cnt * R, _lib.ptr(offsets), _lib.ptr(ws),
                  ws.numel(), s)
        # the single host sync of a step: sample totals per region (allocation sizes)
        meta = offsets[torch.arange(cnt + 1, device=dev) * R]
        sparse = exchange and self.world > 1 and self.sparse_exchange and not all_regions
        if sparse:  # records of the sparse exchange: non-empty segments, max over ranks
            nz = (counts > 0).sum(dtype=torch.int64).reshape(1)
            meta = torch.cat((meta, comm.all_reduce_max_(nz, self.group, self.world)))
        if stage:
            meta = torch.cat((meta, info))
        meta = meta.cpu().tolist()
        bounds = meta[:cnt + 1]
        seg_max = int(meta[cnt + 1]) if sparse else None
        self.check("in sampling")
        N = int(bounds[-1])
        t0 = torch.empty(_even(max(N, 1)), dtype=torch.float64, device=dev)
        t1 = torch.empty(_even(max(N, 1)), dtype=torch.float64, device=dev)
        ray_id = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
        staged = stage and meta[-1] <= st0.numel() // blocks
        if stage and not staged:  # a slice was too small: grow the staging for next time
            self._stage_cap = int(meta[-1] * blocks * 1.15) + blocks
        self.last_k1 = "stage" if staged else "fill"
        if N and staged:
            _lib.call("vr_sample_compact", R, cnt, _lib.ptr(counts), _lib.ptr(seg_first),
                      _lib.ptr(offsets), _lib.ptr(sslot), _lib.ptr(st0), _lib.ptr(st1),
                      _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(ray_id), N, _lib.ptr(self.err), s)
        elif N:
            _lib.call("vr_sample_fill", tc, _lib.ptr(rays), rays.shape[1], R, float(dt),
                      region_lo, cnt, _lib.ptr(offsets), _lib.ptr(seg_first), _lib.ptr(t0),
                      _lib.ptr(t1), _lib.ptr(ray_id), N, self._occ_arg(), _lib.ptr(self.err), s)
        return SampleBatch(R, region_lo, cnt, counts, seg_first, offsets, ray_te, ray_part,
                           ray_total, t0, t1, ray_id, [int(b) for b in bounds], seg_max)

    def _staging(self, R: int):
        """Persistent staging buffers of the one-walk K1 (grown when a slice overflowed)."""
        cap = max(getattr(self, "_stage_cap", 0), self.stage_slots_per_ray * R)
        st = getattr(self, "_stage", None)
        if st is None or st[0].numel() < cap:
            self._stage = None
            st = (torch.empty(cap, dtype=torch.float64, device=self.device),
                  torch.empty(cap, dtype=torch.float64, device=self.device))
            self._stage = st
        return st

    # ---- K1 one step ahead --------------------------------------------------------------
    # Sampling depends only on the rays, not on the parameters, so the next batch's K1 can
    # run on its own stream while this step's field kernels run (K1 is fp64/ALU-latency
    # bound, the hash-grid kernels L2-bound).  The fill goes into buffers sized from the
    # previous batch; a batch that does not fit is re-filled synchronously.
    def _k1_stream(self):
        if getattr(self, "_k1", None) is None:
            self._k1 = torch.cuda.Stream(device=self.device)
        return self._k1

    def sample_async(self, rays: torch.Tensor, dt: float, capacity: int, ready=None):
        """Enqueue K1 for the owned regions of ``rays`` on the sampling stream (after the
        current stream's work and the optional event ``ready``, e.g. the rays' H2D copy);
        returns a pending batch for :meth:`resolve_sample`."""
        if not dt > 0.0:
            raise ValueError("dt must be > 0")
        R = rays.shape[1]
        lo, cnt = self.region_lo, self.region_cnt
        dev = self.device
        main = torch.cuda.current_stream()
        k1 = self._k1_stream()
        k1.wait_stream(main)
        if ready is not None:
            k1.wait_event(ready)
        rays.record_stream(k1)
        tc = _lib.addr(self.tree_c)
        with torch.cuda.stream(k1):
            s = _lib.stream_ptr()
            err = torch.zeros(1, dtype=torch.int32, device=dev)
            counts = torch.empty(cnt * R, dtype=torch.int32, device=dev)
            seg_first = torch.empty(cnt * R, dtype=torch.int32, device=dev)
            ray_te = torch.empty(R, dtype=torch.float64, device=dev)
            _lib.call("vr_sample_count", tc, _lib.ptr(rays), R, R, float(dt), lo, cnt,
                      _lib.ptr(counts), _lib.ptr(seg_first), _lib.ptr(ray_te), None, None,
                      self._occ_arg(), _lib.ptr(err), s)
            offsets = torch.empty(cnt * R + 1, dtype=torch.int64, device=dev)
            ws = torch.empty(int(_lib.load().vr_scan_workspace_bytes(cnt * R)), dtype=torch.uint8,
                             device=dev)
            _lib.call("vr_scan_offsets", _lib.ptr(counts), cnt * R, _lib.ptr(offsets),
                      _lib.ptr(ws), ws.numel(), s)
            bounds_dev = offsets[torch.arange(cnt + 1, device=dev) * R]
            bounds_host = torch.empty(cnt + 1, dtype=torch.int64, pin_memory=True)
            bounds_host.copy_(bounds_dev, non_blocking=True)
            cap = max(int(capacity), 1)
            t0 = torch.empty(_even(cap), dtype=torch.float64, device=dev)
            t1 = torch.empty(_even(cap), dtype=torch.float64, device=dev)
            ray_id = torch.empty(cap, dtype=torch.int32, device=dev)
            _lib.call("vr_sample_fill", tc, _lib.ptr(rays), R, R, float(dt), lo, cnt,
                      _lib.ptr(offsets), _lib.ptr(seg_first), _lib.ptr(t0), _lib.ptr(t1),
                      _lib.ptr(ray_id), cap, self._occ_arg(), _lib.ptr(err), s)
            done = torch.cuda.Event()
            done.record(k1)
        return dict(rays=rays, dt=dt, R=R, counts=counts, seg_first=seg_first, ray_te=ray_te,
                    offsets=offsets, bounds=bounds_host, t0=t0, t1=t1, ray_id=ray_id, err=err,
                    cap=cap, done=done, tensors=(err, counts, seg_first, ray_te, offsets, ws,
                                                 t0, t1, ray_id))

    def resolve_sample(self, p) -> SampleBatch:
        """The SampleBatch of a :meth:`sample_async` (waits for its K1)."""
        main = torch.cuda.current_stream()
        main.wait_event(p["done"])
        for t in p["tensors"]:
            t.record_stream(main)
        p["done"].synchronize()  # the host needs the per-region sample totals
        bounds = [int(x) for x in p["bounds"].tolist()]
        N = bounds[-1]
        cnt, R = self.region_cnt, p["R"]
        t0, t1, ray_id = p["t0"], p["t1"], p["ray_id"]
        flags = int(p["err"].item()) | int(self.err.item())
        self.err.zero_()
        if N > p["cap"]:  # did not fit: fill again on this stream
            flags &= ~_lib.VR_FLAG_OVERFLOW
            t0 = torch.empty(_even(N), dtype=torch.float64, device=self.device)
            t1 = torch.empty(_even(N), dtype=torch.float64, device=self.device)
            ray_id = torch.empty(N, dtype=torch.int32, device=self.device)
            _lib.call("vr_sample_fill", _lib.addr(self.tree_c), _lib.ptr(p["rays"]), R, R,
                      float(p["dt"]), self.region_lo, cnt, _lib.ptr(p["offsets"]),
                      _lib.ptr(p["seg_first"]), _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(ray_id), N,
                      self._occ_arg(), _lib.ptr(self.err), self._stream())
        _lib.raise_flags(flags, "in sampling")
        return SampleBatch(R, self.region_lo, cnt, p["counts"], p["seg_first"], p["offsets"],
                           p["ray_te"], None, None, t0, t1, ray_id, bounds)

    # ---- fields -------------------------------------------------------------------------
    def evaluate(self, rays: torch.Tensor, b: SampleBatch, fields=None,
                 pos_from=None) -> torch.Tensor:
        """Region fields' (sigma, rgb) of the batch's samples.  pos_from: fields evaluated
        earlier in the step over the same samples (the NeRF fields, for the proposals): a
        field whose normalisation box equals its partner's reads the partner's positions."""
        fields = self.fields if fields is None else fields
        base = self.region_lo - b.region_lo  # an all-region batch: skip the peers' regions
        # (an all-region batch leaves the peers' rows zero until the exchange fills them)
        alloc = torch.zeros if base or len(fields) < b.region_cnt else torch.empty
        sig_rgb = alloc((max(b.n_samples, 1), 4), dtype=torch.float32, device=self.device)
        s = self._stream()
        # Off by default (VR_OVERLAP_FWD=1): with the old 52 KB-smem MLP forward the step got
        # slower (c3 76.7 vs 67.6 ms); with the 20 KB TS-mode forward it is a wash at c3
        # (56.6 vs 56.7 ms) and slower at c5 (86.9 vs 84.2; with the MLP grid capped at 2 / 1
        # / 0.5 CTAs per SM: 87.3 / 97.2 / 118.8) — the gathers are L2-request bound and the
        # MLP CTAs still take their issue slots.
        split = (self.overlap_regions and len(fields) > 1
                 and all(getattr(f, "splittable", False) for f in fields))
        if not split:
            for kk, f in enumerate(fields):
                lo, hi = b.region_slice(base + kk)
                if hi > lo:
                    pos = self._shared_positions(f, pos_from[kk], hi - lo) if pos_from else None
                    f.forward(rays, b.t0[lo:], b.t1[lo:], b.ray_id[lo:], hi - lo, sig_rgb[lo:], s,
                              **({"pos": pos} if pos is not None else {}))
            return sig_rgb
        # two-stream pipeline over regions: gathers of region k+1 (L2-bound) run while the
        # tensor-core MLP of region k runs on the side stream
        main = torch.cuda.current_stream()
        side = self._side_stream()
        side.wait_stream(main)
        for kk, f in enumerate(fields):
            lo, hi = b.region_slice(base + kk)
            if hi <= lo:
                continue
            f.forward_hash(rays, b.t0[lo:], b.t1[lo:], b.ray_id[lo:], hi - lo, s)
            ev = torch.cuda.Event()
            ev.record(main)
            with torch.cuda.stream(side):
                side.wait_event(ev)
                f.forward_mlp(rays, b.ray_id[lo:], hi - lo, sig_rgb[lo:], _lib.stream_ptr())
        main.wait_stream(side)
        return sig_rgb

    @staticmethod
    def _shared_positions(f, partner, n):
        """partner's positions of this step's n samples if f normalises by the same box."""
        if not (hasattr(f, "positions") and hasattr(partner, "positions")):
            return None
        if not (np.array_equal(f.box.mn, partner.box.mn)
                and np.array_equal(f.box.mx, partner.box.mx)):
            return None
        return partner.positions(n)

    # side-stream scatter grid: 0 = the kernel's full grid (measured best: 148 or 296 co-
    # resident 128-thread blocks left the scatter far below the L2 atomic rate)
    SCATTER_BLOCKS = int(os.environ.get("VR_SCATTER_BLOCKS", "0"))
    # the MLP backward's grid while the previous region's scatter runs on the side stream
    # (0: the full persistent grid, 2 CTAs per SM).  Once the MLP backward's prefetch stopped
    # stalling on its loads it became the longer of the two backward chains, and the full
    # grid won (c4 ms per step, scripts/sweep_ctas.sh: 185 CTAs 327.3, 222 312.7, 259 310.8,
    # 296 308.0; before that change 1.25 CTAs per SM was best: 185 388, 296 413)
    MLP_CTAS_BESIDE_SCATTER = int(os.environ.get("VR_MLP_BWD_CTAS", "0"))

    # sparse backward: only the samples with a non-zero upstream gradient go through the
    # MLP backward and the hash-grid scatter (vr_active_rows; VR_ACTIVE_ROWS=0 disables)
    ACTIVE_ROWS = os.environ.get("VR_ACTIVE_ROWS", "1") != "0"

    def _active_rows(self, dsig_rgb: torch.Tensor, n: int):
        """(rows, n_rows) device tensors: the ordered indices of the samples in
        dsig_rgb[:n] (float4 rows) with a non-zero upstream gradient, and their count."""
        need = int(_lib.load().vr_active_rows_workspace_bytes(n))
        if self._rows_ws is None or self._rows_ws.numel() < need:
            self._rows_ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
        rows = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        cnt = torch.empty(1, dtype=torch.int32, device=self.device)
        _lib.call("vr_active_rows", _lib.ptr(dsig_rgb), n, _lib.ptr(rows), _lib.ptr(cnt),
                  _lib.ptr(self._rows_ws), self._rows_ws.numel(), self._stream())
        return rows, cnt

    def field_backward(self, rays, b: SampleBatch, dsig_rgb: torch.Tensor, fields=None,
                       sig_rgb: torch.Tensor | None = None) -> None:
        self.field_backward_jobs(rays, b, [(self.fields if fields is None else fields, dsig_rgb,
                                            sig_rgb)])

    def field_backward_jobs(self, rays, b: SampleBatch, jobs) -> None:
        """Backward of several field sets of the same batch ([(fields, dsig_rgb, sig_rgb),
        ...]: the NeRF fields and the proposals) as one pipeline; sig_rgb is the fields'
        forward output (may be None)."""
        s = self._stream()
        base = self.region_lo - b.region_lo  # an all-region batch: skip the peers' regions
        split = [all(getattr(f, "split_backward", False) for f in fields if f.trainable)
                 for fields, _, _ in jobs]
        if self.overlap_backward and any(split):
            # region k's hash-grid scatter (L2-atomic bound) runs on the side stream while
            # the tensor-core MLP backward of the next region (of any field set) runs here
            main = torch.cuda.current_stream()
            side = self._side_stream()
            # every row list first: once the side stream's persistent scatter grids hold the
            # SMs, a small kernel queued behind them waits for a whole scatter
            row_lists = {}
            for j, (fields, dsig_rgb, _) in enumerate(jobs):
                for kk, f in enumerate(fields):
                    lo, hi = b.region_slice(base + kk)
                    if (hi > lo and f.trainable and self.ACTIVE_ROWS
                            and getattr(f, "takes_rows", False)):
                        row_lists[j, kk] = self._active_rows(dsig_rgb[lo:], hi - lo)
            side.wait_stream(main)
            for j, ((fields, dsig_rgb, sig_rgb), sp) in enumerate(zip(jobs, split)):
                for kk, f in enumerate(fields):
                    lo, hi = b.region_slice(base + kk)
                    if hi <= lo or not f.trainable:
                        continue
                    sig = sig_rgb[lo:] if sig_rgb is not None else None
                    rows = row_lists.get((j, kk))
                    if not sp:
                        f.backward(rays, b.t0[lo:], b.t1[lo:], b.ray_id[lo:], hi - lo,
                                   dsig_rgb[lo:], s, sig_rgb=sig,
                                   **({"rows": rows} if rows is not None else {}))
                        continue
                    denc = f.backward_mlp(rays, b.ray_id[lo:], hi - lo, dsig_rgb[lo:], s,
                                          self.MLP_CTAS_BESIDE_SCATTER, sig_rgb=sig, rows=rows)
                    ev = torch.cuda.Event()
                    ev.record(main)
                    with torch.cuda.stream(side):
                        side.wait_event(ev)
                        denc.record_stream(side)
                        if rows is not None:
                            rows[0].record_stream(side)
                            rows[1].record_stream(side)
                        f.backward_scatter(denc, hi - lo, _lib.stream_ptr(), self.SCATTER_BLOCKS,
                                           rows=rows)
            main.wait_stream(side)
            return
        for fields, dsig_rgb, sig_rgb in jobs:
            for kk, f in enumerate(fields):
                lo, hi = b.region_slice(base + kk)
                if hi > lo and f.trainable:
                    extra = ({"rows": self._active_rows(dsig_rgb[lo:], hi - lo)}
                             if self.ACTIVE_ROWS and getattr(f, "takes_rows", False) else {})
                    f.backward(rays, b.t0[lo:], b.t1[lo:], b.ray_id[lo:], hi - lo,
                               dsig_rgb[lo:], s,
                               sig_rgb=sig_rgb[lo:] if sig_rgb is not None else None, **extra)

    # ---- K4 ----------------------------------------------------------------------------
    def local_packets(self, b: SampleBatch, sig_rgb: torch.Tensor,
                      totals: torch.Tensor | None = None) -> torch.Tensor:
        """K4 forward; totals (float64 [cnt*R*7], training): the segments' unrounded totals,
        which spare vr_segment_bwd its first sweep."""
        pk = torch.empty((b.region_cnt, b.n_rays, 8), dtype=torch.float32, device=self.device)
        _lib.call("vr_segment_fwd", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(sig_rgb),
                  _lib.ptr(b.offsets), _lib.ptr(b.seg_first), _lib.ptr(b.ray_te), b.n_rays,
                  b.region_cnt, _lib.ptr(pk), _lib.ptr(totals), _lib.ptr(self.err),
                  self._tma_n(b.n_samples, b.t0, b.t1, sig_rgb), self._stream())
        return pk

    @staticmethod
    def _tma_n(n: int, t0, t1, sr) -> int:
        """n_samples for the K4 walks' TMA staging (vr_capi.h vr_segment_fwd): the sample
        count when t0 / t1 hold an even number >= n of elements (the staging reads 16-byte
        pairs) and sig_rgb >= n rows, else 0 (per-lane loads)."""
        ok = (t0.numel() >= n and t1.numel() >= n and t0.numel() % 2 == 0
              and t1.numel() % 2 == 0 and sr.shape[0] >= n)
        return n if ok else 0

    def _segment_totals(self, n_segs: int) -> torch.Tensor:
        return torch.empty(max(n_segs, 1) * 7, dtype=torch.float64, device=self.device)

    def exchange_packets(self, b: SampleBatch, local: torch.Tensor, extra=None,
                         dst: int | None = None):
        """The packet exchange: [K_own][R][8] (+ optional per-segment proposal T
        [K_own][R]) of every rank -> the global [K][R][8] (and [K][R]) slabs on every rank
        (dst None, training) or on rank dst only (render; None elsewhere).  Dense: one
        all-gather / gather of the slabs.  Sparse (b.seg_max set): only the records of
        non-empty segments travel (vr_packets_pack / vr_packets_unpack), which gives the
        same slabs bit for bit."""
        if self.world == 1:
            return local, extra
        if b.seg_max is None:
            if dst is None:
                allp = comm.all_gather_packets(local, self.group, self.world)
                all_e = (comm.all_gather_packets(extra, self.group, self.world)
                         if extra is not None else None)
                return allp, all_e
            allp = comm.gather_packets(local, self.group, self.world, self.rank, dst)
            if extra is not None:
                raise ValueError("extra slabs are exchanged in training only")
            return allp, None
        s = self._stream()
        R = b.n_rays
        width = 9 if extra is None else 10
        cap = max(int(b.seg_max), 1)
        send = torch.empty((cap + 1, width), dtype=torch.float32, device=self.device)
        n_dev = torch.empty(1, dtype=torch.int32, device=self.device)
        _lib.call("vr_packets_pack", _lib.ptr(local), _lib.ptr(extra), _lib.ptr(b.counts), R,
                  b.region_lo, b.region_cnt, _lib.ptr(send), cap, _lib.ptr(n_dev),
                  _lib.ptr(self.err), s)
        if dst is None:
            recv = comm.all_gather_packets(send, self.group, self.world)
        else:
            recv = comm.gather_packets(send, self.group, self.world, self.rank, dst)
            if recv is None:
                return None, None
        if self.records_k5:  # K5 reads the records through a 4-byte-per-segment index
            index = torch.empty((self.n_regions, R), dtype=torch.int32, device=self.device)
            _lib.call("vr_packets_index", _lib.ptr(recv), self.world, cap + 1, width, R,
                      self.n_regions, _lib.ptr(index), _lib.ptr(self.err), s)
            rec = PacketRecords(recv, width, index, self.n_regions)
            return rec, (rec if extra is not None else None)
        allp = torch.empty((self.n_regions, R, 8), dtype=torch.float32, device=self.device)
        all_e = (torch.empty((self.n_regions, R), dtype=torch.float32, device=self.device)
                 if extra is not None else None)
        _lib.call("vr_packets_unpack", _lib.ptr(recv), self.world, cap + 1, width, R,
                  self.n_regions, _lib.ptr(allp), _lib.ptr(all_e), _lib.ptr(self.err), s)
        return allp, all_e

    # ---- K5 ----------------------------------------------------------------------------
    def _set_bg(self, background):
        bg = self.background if background is None else vec3(background)
        for c in range(3):
            self._bg[c] = float(bg[c])
        return self._bg

    def compose(self, packets, b: SampleBatch, background=None,
                clip: bool = True) -> torch.Tensor:
        out = torch.empty((7, b.n_rays), dtype=torch.float32, device=self.device)
        if isinstance(packets, PacketRecords):
            _lib.call("vr_global_fwd_records", _lib.ptr(packets.recv), packets.width,
                      _lib.ptr(packets.index), packets.n_regions, b.n_rays, _lib.ptr(b.ray_te),
                      _lib.addr(self._set_bg(background)), 1 if clip else 0, _lib.ptr(out),
                      _lib.ptr(self.err), self._stream())
            return out
        _lib.call("vr_global_fwd", _lib.ptr(packets), packets.shape[0], b.n_rays,
                  _lib.ptr(b.ray_te), _lib.addr(self._set_bg(background)), 1 if clip else 0, _lib.ptr(out),
                  _lib.ptr(self.err), self._stream())
        return out

    # ---- entry points ------------------------------------------------------------------
    def render_rays(self, rays, dt: float, background=None, clip: bool = True,
                    protocol: str = "tile", stats: bool = False):
        """Batched render.  Returns (out [7][R] on rank 0 / None elsewhere, batch);
        out rows: r, g, b (C + T*bg clipped, or raw C if clip=False), alpha, depth, T, L.
        protocol: "tile" (segment packets, the NeRF-XL path), "sample" (per-sample
        broadcast) or "mono" (one composite over the whole ray, no exchange)."""
        rays = self.rays_to_device(rays)
        protocol = canonical_protocol(protocol)
        if protocol != "tile_aggregate":
            b, res = self._sample_protocol_forward(rays, dt, train=False)
            if res is None:
                return None, b
            _, ray_off, (t0r, t1r, srr) = res
            pk = self._whole_ray_packets(b, ray_off, t0r, t1r, srr)
            return self.compose(pk, b, background, clip), b
        b = self.sample(rays, dt, stats=stats, exchange=True)
        sig_rgb = self.evaluate(rays, b)
        local = self.local_packets(b, sig_rgb)
        allp, _ = self.exchange_packets(b, local, dst=0)
        if allp is None:
            return None, b
        return self.compose(allp, b, background, clip), b

    # ---- sample-broadcast / mono protocols --------------------------------------------
    # The reference's per-sample protocols (distsim.py:311-316, _compose_samples
    # distsim.py:385-392, mono distsim.py:398-404): every rank samples every region, its
    # own regions' (sigma, rgb) cross the link (16 B per sample instead of 32 B per
    # (ray, region) packet), and whole rays are composited in t order — the region-major
    # samples are permuted ray-major so K4 (region_cnt = 1) sees one segment per ray.
    def _ray_major(self, b: SampleBatch):
        R = b.n_rays
        s = self._stream()
        ray_off = torch.empty(R + 1, dtype=torch.int64, device=self.device)
        ws = self._workspace(R)
        _lib.call("vr_scan_offsets", _lib.ptr(b.ray_total), R, _lib.ptr(ray_off), _lib.ptr(ws),
                  ws.numel(), s)
        return ray_off

    def _permute(self, b: SampleBatch, ray_off, src: torch.Tensor, to_ray_major: bool):
        dst = torch.empty_like(src)
        _lib.call("vr_segment_permute", _lib.ptr(b.offsets), _lib.ptr(b.seg_first),
                  _lib.ptr(ray_off), b.n_rays, b.region_cnt, _lib.ptr(src), _lib.ptr(dst),
                  src.element_size() * (src.shape[1] if src.dim() == 2 else 1),
                  1 if to_ray_major else 0, self._stream())
        return dst

    def _whole_ray_packets(self, b: SampleBatch, ray_off, t0r, t1r, srr, totals=None):
        R = b.n_rays
        pk = torch.empty((1, R, 8), dtype=torch.float32, device=self.device)
        first = torch.zeros(R, dtype=torch.int32, device=self.device)  # one packet per ray
        _lib.call("vr_segment_fwd", _lib.ptr(t0r), _lib.ptr(t1r), _lib.ptr(srr),
                  _lib.ptr(ray_off), _lib.ptr(first), _lib.ptr(b.ray_te), R, 1, _lib.ptr(pk),
                  _lib.ptr(totals), _lib.ptr(self.err),
                  self._tma_n(b.n_samples, t0r, t1r, srr), self._stream())
        return pk

    def _sample_protocol_forward(self, rays, dt: float, train: bool):
        b = self.sample(rays, dt, all_regions=True)
        sig_rgb = self.evaluate(rays, b)
        got = comm.exchange_samples(sig_rgb, b.region_bounds, self.n_regions, self.group,
                                    self.world, self.rank, None if train else 0)
        if not got:
            return b, None
        ray_off = self._ray_major(b)
        rm = [self._permute(b, ray_off, x, True) for x in (b.t0, b.t1, sig_rgb)]
        return b, (sig_rgb, ray_off, rm)

    def loss_and_grad(self, rays, targets, dt: float, lambda_dist: float = 1.0,
                      background=None, lambda_interlevel: float = 0.0, eps: float = 1e-7,
                      protocol: str = "tile", batch: SampleBatch | None = None,
                      check_errors: bool = True):
        """Forward + backward of the NeRF-XL loss (segrender.py:198-207 definition:
        sum over rays of |C + T*bg - target|^2 + lambda * distortion), plus, with
        proposal fields and lambda_interlevel > 0, the interlevel loss of csrc/interlevel.cu
        (summed over the ranks: identical on every rank, like the main term).
        Gradients accumulate into the owned region fields; returns (loss [1] float64
        device tensor, out [7][R], batch).  check_errors: read the device error word at
        the end (one host sync) and raise the reference exception of a flagged non-finite
        packet / negative distortion / overflow (segrender.py:124-141)."""
        rays = self.rays_to_device(rays)
        tg = torch.as_tensor(targets, dtype=torch.float32).to(self.device, non_blocking=True)
        tg = tg.reshape(-1, 3).contiguous()
        if tg.shape[0] != rays.shape[1]:
            raise ValueError("targets must be (R, 3)")
        s = self._stream()
        protocol = canonical_protocol(protocol)
        if protocol != "tile_aggregate":
            if lambda_interlevel > 0.0:
                raise ValueError("the interlevel loss is defined on the tile protocol")
            res = self._sample_protocol_train(rays, tg, dt, lambda_dist, background)
            if check_errors:
                self.check_step()
            return res
        # batch: sample_async
        b = batch if batch is not None else self.sample(rays, dt, exchange=True)
        sig_rgb = self.evaluate(rays, b)
        totals = self._segment_totals(b.region_cnt * b.n_rays)
        local = self.local_packets(b, sig_rgb, totals)
        interlevel = self.proposals is not None and lambda_interlevel > 0.0
        prop_T = None
        if interlevel:
            # the proposal of a region shares its NeRF field's box: its gathers read the
            # positions the NeRF forward kept
            sig_prop = self.evaluate(rays, b, self.proposals, pos_from=self.fields)
            # only the proposal transmittance of each segment crosses the link
            prop_T = torch.empty((b.region_cnt, b.n_rays), dtype=torch.float32,
                                 device=self.device)
            _lib.call("vr_segment_transmittance", _lib.ptr(b.t0), _lib.ptr(b.t1),
                      _lib.ptr(sig_prop), _lib.ptr(b.offsets), b.n_rays, b.region_cnt,
                      _lib.ptr(prop_T), s)
        allp, all_T = self.exchange_packets(b, local, prop_T)
        R = b.n_rays
        out = torch.empty((7, R), dtype=torch.float32, device=self.device)
        ray_loss = torch.empty(R, dtype=torch.float64, device=self.device)
        dpk = torch.empty((b.region_cnt, R, 8), dtype=torch.float32, device=self.device)
        if isinstance(allp, PacketRecords):
            _lib.call("vr_global_train_records", _lib.ptr(allp.recv), allp.width,
                      _lib.ptr(allp.index), allp.n_regions, R, _lib.ptr(b.ray_te),
                      _lib.addr(self._set_bg(background)), _lib.ptr(tg), float(lambda_dist),
                      self.region_lo, self.region_cnt, _lib.ptr(out), _lib.ptr(ray_loss),
                      _lib.ptr(dpk), _lib.ptr(self.err), s)
        else:
            _lib.call("vr_global_train", _lib.ptr(allp), allp.shape[0], R, _lib.ptr(b.ray_te),
                      _lib.addr(self._set_bg(background)), _lib.ptr(tg), float(lambda_dist),
                      self.region_lo, self.region_cnt, _lib.ptr(out), _lib.ptr(ray_loss),
                      _lib.ptr(dpk), _lib.ptr(self.err), s)
        loss = torch.empty(1, dtype=torch.float64, device=self.device)
        _lib.call("vr_sum_f64", _lib.ptr(ray_loss), R, _lib.ptr(loss),
                  _lib.ptr(self._sum_scratch()), s)
        if interlevel:
            prefix = torch.empty((b.region_cnt, R, 2), dtype=torch.float32, device=self.device)
            if isinstance(allp, PacketRecords):
                _lib.call("vr_prefix_train_records", _lib.ptr(allp.recv), _lib.ptr(allp.index),
                          allp.n_regions, R, self.region_lo, self.region_cnt, _lib.ptr(prefix), s)
            else:
                _lib.call("vr_prefix_train", _lib.ptr(allp), _lib.ptr(all_T), allp.shape[0], R,
                          self.region_lo, self.region_cnt, _lib.ptr(prefix), s)
            seg_loss = torch.empty(b.region_cnt * R, dtype=torch.float64, device=self.device)
            # every sample of a segment is written (no zero fill of the N x 16 B array)
            dsig_prop = torch.empty((max(b.n_samples, 1), 4), dtype=torch.float32,
                                    device=self.device)
            _lib.call("vr_interlevel", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(sig_rgb),
                      _lib.ptr(sig_prop), _lib.ptr(b.offsets), _lib.ptr(prefix), R,
                      b.region_cnt, float(lambda_interlevel), float(eps), _lib.ptr(seg_loss),
                      _lib.ptr(dsig_prop), s)
            il = torch.empty(1, dtype=torch.float64, device=self.device)
            _lib.call("vr_sum_f64", _lib.ptr(seg_loss), seg_loss.numel(), _lib.ptr(il),
                      _lib.ptr(self._sum_scratch()), s)
            # each rank sums its own segments' terms: the all-reduce makes the reported loss
            # the whole batch's on every rank (the main term already is)
            loss = loss + comm.all_reduce_scalar(il, self.group, self.world)
        # vr_segment_bwd writes every sample (no zero fill of the N x 16 B array)
        dsig = torch.empty((max(b.n_samples, 1), 4), dtype=torch.float32, device=self.device)
        _lib.call("vr_segment_bwd", _lib.ptr(b.t0), _lib.ptr(b.t1), _lib.ptr(sig_rgb),
                  _lib.ptr(b.offsets), _lib.ptr(b.ray_te), R, b.region_cnt, _lib.ptr(dpk),
                  _lib.ptr(totals), _lib.ptr(dsig), s)
        # NeRF fields and proposals in one backward pipeline (the proposals' MLP backward
        # overlaps the NeRF scatter on the side stream)
        jobs = [(self.fields, dsig, sig_rgb)]
        if interlevel:
            jobs.append((self.proposals, dsig_prop, sig_prop))
        self.field_backward_jobs(rays, b, jobs)
        if check_errors:
            self.check_step()
        return loss, out, b

    def check_step(self, updated: bool = False) -> None:
        """Read the step's device error word (one host sync) and raise the reference
        exception with the stage that set it; the word is cleared.  A flagged step never
        reaches the parameters: vr_adam_step is gated on the same word."""
        flags = int(self.err.item())
        if flags:
            self.err.zero_()
            _lib.raise_flags(flags, self._flag_stage(flags) + (" (parameters not updated)"
                                                          if updated else ""))

    def _sample_protocol_train(self, rays, tg, dt, lambda_dist, background):
        """Training through the sample-broadcast protocol: every rank composites whole rays
        from all samples, takes the gradients of its own samples (no gradient exchange
        either way)."""
        s = self._stream()
        b, (sig_rgb, ray_off, (t0r, t1r, srr)) = self._sample_protocol_forward(rays, dt, True)
        R = b.n_rays
        totals = self._segment_totals(R)
        pk = self._whole_ray_packets(b, ray_off, t0r, t1r, srr, totals)
        out = torch.empty((7, R), dtype=torch.float32, device=self.device)
        ray_loss = torch.empty(R, dtype=torch.float64, device=self.device)
        dpk = torch.empty((1, R, 8), dtype=torch.float32, device=self.device)
        _lib.call("vr_global_train", _lib.ptr(pk), 1, R, _lib.ptr(b.ray_te),
                  _lib.addr(self._set_bg(background)), _lib.ptr(tg), float(lambda_dist), 0, 1,
                  _lib.ptr(out), _lib.ptr(ray_loss), _lib.ptr(dpk), _lib.ptr(self.err), s)
        loss = torch.empty(1, dtype=torch.float64, device=self.device)
        _lib.call("vr_sum_f64", _lib.ptr(ray_loss), R, _lib.ptr(loss),
                  _lib.ptr(self._sum_scratch()), s)
        dsr = torch.zeros_like(srr)
        _lib.call("vr_segment_bwd", _lib.ptr(t0r), _lib.ptr(t1r), _lib.ptr(srr), _lib.ptr(ray_off),
                  _lib.ptr(b.ray_te), R, 1, _lib.ptr(dpk), _lib.ptr(totals), _lib.ptr(dsr), s)
        dsig = self._permute(b, ray_off, dsr, False)
        self.field_backward(rays, b, dsig, sig_rgb=sig_rgb)
        return loss, out, b

    def zero_grad(self):
        for f in self.fields + (self.proposals or []):
            f.zero_grad()

    def train_step(self, rays, targets, dt: float, lr: float = 1e-2, step: int = 1,
                   lambda_dist: float = 1.0, background=None, lambda_interlevel: float = 0.0,
                   protocol: str = "tile", batch: SampleBatch | None = None):
        """One training iteration: zero grads, fwd+bwd, Adam.  Returns the device loss.
        batch: the rays' samples from :meth:`sample_async` / :meth:`resolve_sample` (K1
        prefetched during the previous step)."""
        self.zero_grad()
        loss, _, _ = self.loss_and_grad(rays, targets, dt, lambda_dist, background,
                                        lambda_interlevel, protocol=protocol, batch=batch,
                                        check_errors=False)
        for f in self.fields + (self.proposals or []):
            if f.trainable:
                f.step(lr, step)  # skipped on the device if the step flagged an error
        self.check_step(updated=True)
        return loss

    # ---- accounting ----------------------------------------------------------------------
    def comm_stats(self, b: SampleBatch, broadcast_all: bool = False,
                   protocol: str = "tile") -> CommStats:
        """Reference-style scalar counts (distsim.py:415-446) from the K1 outputs."""
        protocol = canonical_protocol(protocol)
        st = CommStats()
        st.rays = b.n_rays
        if protocol == "mono":  # one field, no workers (distsim.py:398-404)
            return st
        part = b.ray_part.to(torch.int64) & 0xFFFFFFFF
        per_leaf = [int(((part >> k) & 1).sum().item()) for k in range(self.n_regions)]
        st.participations = int(sum(per_leaf))
        st.samples_assigned = int(b.ray_total.to(torch.int64).sum().item())
        if protocol == "sample_broadcast":
            # one SamplePayload per participation: 1 + 6 scalars per bin (distsim.py:151)
            for k, n in enumerate(per_leaf):
                if n:
                    bins = b.region_bounds[k + 1] - b.region_bounds[k]
                    st.record(k, COMPOSITOR, n + SCALARS_PER_SAMPLE * bins, n)
            if self.world > 1:
                per = self.n_regions // self.world
                blk = [b.region_bounds[(r + 1) * per] - b.region_bounds[r * per]
                       for r in range(self.world)]
                st.link_bytes = (self.world - 1) * max(blk) * 16
            else:
                st.link_bytes = 0
            return st
        for k, n in enumerate(per_leaf):
            if n:
                st.record(k, COMPOSITOR, SCALARS_PER_TILE_PACKET * n, n)
        if broadcast_all:
            nparts = torch.zeros_like(part)
            for k in range(self.n_regions):
                nparts += (part >> k) & 1
            for k in range(self.n_regions):
                mine = (part >> k) & 1
                # leaf k receives every other participant's packet on rays it joins
                recv = int((mine * (nparts - 1)).sum().item())
                if recv:
                    st._party(k).scalars_received += SCALARS_PER_TILE_PACKET * recv
                    st._party(k).messages_received += recv
                sent = int((mine * (nparts - 1)).sum().item())
                st._party(k).scalars_sent += SCALARS_PER_TILE_PACKET * sent
                st._party(k).messages_sent += sent
        if self.world == 1:
            st.link_bytes = 0
        elif b.seg_max is not None:  # sparse exchange: padded 36-byte records
            st.link_bytes = (self.world - 1) * (b.seg_max + 1) * 36
        else:
            st.link_bytes = (self.world - 1) * self.region_cnt * b.n_rays * 32
        return st


def spawn(tree: PartitionTree, scene: Scene, device=None, rank: int = 0, world: int = 1,
          group=None) -> VolumePool:
    """One region field per owned leaf (spawn, distsim.py:358-364)."""
    lo, cnt = comm.owned_regions(len(tree.leaves), rank, world)
    dev = torch.device(device) if device is not None else torch.device("cuda")
    if isinstance(scene.field, RegionField) and scene.field.trainable and cnt > 1:
        raise ValueError("a trainable RegionField cannot be spawned over several regions: "
                         "build one field per region and pass them to VolumePool")
    fields = [region_field_for(scene.field, tree.leaves[k], tree, dev) for k in range(lo, lo + cnt)]
    return VolumePool(tree, fields, scene.background, dev, rank, world, group)


def _aggregate_from_out(out: np.ndarray, i: int) -> RayAggregate:
    return RayAggregate(out[0:3, i].astype(np.float64), float(out[3, i]), float(out[4, i]),
                        float(out[5, i]), float(out[6, i]))


def render_ray(pool: VolumePool, ray: Ray, protocol: str, dt: float, rng=None,
               broadcast_all: bool = False):
    """One ray (distsim.py:478-490); returns (RayAggregate, CommStats).  ``rng`` is
    accepted for API parity: the GPU composite is order-independent by construction."""
    if pool.num_workers == 0:
        raise ProtocolMismatchError("worker pool is empty")
    protocol = canonical_protocol(protocol)
    out, b = pool.render_rays(rays_to_soa([ray]), dt, clip=False, protocol=protocol, stats=True)
    st = pool.comm_stats(b, broadcast_all, protocol)
    if out is None:
        return None, st
    return _aggregate_from_out(out.cpu().numpy(), 0), st


def render_image(pool: VolumePool, camera: Camera, protocol: str, dt: float, background=None,
                 threads: int = 1, shuffle_seed=None, broadcast_all: bool = False):
    """One primary ray per pixel (distsim.py:495-542); returns ((h,w,3) float64 image
    with pixel = clip(C + T*bg, 0, 1), CommStats).  ``threads``/``shuffle_seed`` are
    accepted for API parity (the GPU path is scheduling-independent)."""
    if pool.num_workers == 0:
        raise ProtocolMismatchError("worker pool is empty")
    protocol = canonical_protocol(protocol)
    t0 = time.perf_counter()
    rays = camera_rays(camera, pool.tree.root_box)
    out, b = pool.render_rays(rays, dt, background=background, clip=True, protocol=protocol,
                              stats=True)
    st = pool.comm_stats(b, broadcast_all, protocol)
    if out is None:
        return None, st
    img = out[0:3].T.contiguous().cpu().numpy().astype(np.float64)
    pool.check("in render_image")
    st.add_time("render", time.perf_counter() - t0)
    return img.reshape(camera.height, camera.width, 3), st


def write_ppm(path, image: np.ndarray) -> None:
    """Binary PPM, quantisation floor(c*255 + 0.5) (distsim.py:545-551)."""
    h, w = image.shape[:2]
    data = np.floor(np.clip(image, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    with open(path, "wb") as f:
        f.write(f"P6\n{w} {h}\n255\n".encode("ascii"))
        f.write(data.tobytes())
