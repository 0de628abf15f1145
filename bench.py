"""Benchmark: NeRF-XL distributed training step (fwd+bwd+Adam) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

N>1 is launched by the driver with torch.distributed.run (one rank per GPU, NCCL).
A step = sample rays (K1) -> hash grid + MLP fwd (K2, K3) -> segment composite (K4)
-> all-gather of packets -> global composite + loss + its backward (K5) -> K4 bwd ->
MLP/hash bwd -> Adam, over one batch of synthetic rays (BASELINE.json configs; see
paper_2404_16221_b200/workloads.py).  Rank 0 prints ONE JSON line.

The headline is config 4 (the largest single-GPU configuration, where SURVEY §8(d) judges
the hash-encode HBM target): 8-region city, 4M rays/step, T=2^22, mse + distortion +
interlevel.  The same line carries config 3 (train) and config 5 (render) as sub-results.
Every timed step trains on its own batch (a rotation of distinct pre-built batches), from
a steady training state: before the driver's warm-up the model is trained for --burnin
steps (the step time falls ~15-20 % over the first ~15 Adam steps from random init, as
opaque regions form and the samples behind them get exactly-zero gradients that skip
their atomics — measured, scripts/drift.py), and every timed pass restarts from the same
post-warm-up snapshot.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "train rays/sec (fwd+bwd)"
RENDER_METRIC = "render rays/sec"
UNIT = "rays/s"

# Algorithmic cost per unit of work: bytes (hbm) or flops (tensor)
# per sample for the per-sample kernels.
# entry point -> (bound, algorithmic bytes or flops per sample, index of the sample-count
# argument in the C-ABI call); bench sums the samples each launch processed
KERNEL_COST = {
    # t0,t1 (16) + ray id (4) + 16 levels x 8 corners x float2 (1024) + enc fp16 (64)
    "vr_hash_fwd": ("hbm", 1108.0, 7),
    # t0,t1,ray id (20) + denc f32 (128) + 16 x 8 float2 atomics (1024)
    "vr_hash_bwd": ("hbm", 1172.0, 6),
    # level-major: pos (12 per level read) + 8 float2 gathers (64) + enc (4), x 16 levels
    "vr_hash_fwd_lm": ("hbm", 16 * (12 + 64 + 4.0), 3),
    # level-major: pos (12) + denc (8) + 8 float2 atomics (64), x 16 levels
    "vr_hash_bwd_lm": ("hbm", 16 * (12 + 8 + 64.0), 2),
    # split backward's scatter: pos (12) + denc f32 (128) + 16 x 8 float2 atomics (1024)
    "vr_hash_scatter": ("hbm", 1164.0, 2),
    # 2 * (32*64 + 64*16 + 32*64 + 64*64 + 64*3)
    "vr_mlp_fwd": ("tensor", 18816.0, 5),
    "vr_mlp_fwd_tc": ("tensor", 18816.0, 5),
    # recomputed forward + activation grads + weight grads
    "vr_mlp_bwd": ("tensor", 3 * 18816.0, 5),
    "vr_mlp_bwd_tc": ("tensor", 3 * 18816.0, 5),
    # density branch only: 2 * (32*64 + 64*16) fwd, x3 with the backward
    "vr_mlp_fwd_tc_density": ("tensor", 6144.0, 2),
    "vr_mlp_bwd_tc_density": ("tensor", 3 * 6144.0, 5),
    # fused K2+K3 forward: t0,t1,id (20) + 128 corner gathers (1024) + enc out (64) + sig_rgb (16)
    "vr_field_fwd_tc": ("hbm", 1124.0, 8),
    # fused K3+K2 backward: enc (64) + dsig_rgb (16) + t0,t1,id (20) + 1024 atomic payload
    "vr_field_bwd_tc": ("hbm", 1124.0, 8),
    # t0,t1 (16) + sig_rgb (16); packets amortised
    "vr_segment_fwd": ("hbm", 32.0, None),
    # t0,t1 (16) + sig_rgb (16) + dsig_rgb (16)
    "vr_segment_bwd": ("hbm", 48.0, None),
    # t0,t1 (16) + sigma (4)
    "vr_segment_transmittance": ("hbm", 20.0, None),
}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": float(d["hbm_gbs"]), "tensor": float(d["bf16_tflops_sustained"]),
                "tensor_burst": float(d["bf16_tflops"]), "source": "measured",
                "sm_max_mhz": d.get("sm_max_mhz")}
    return {"hbm": 6650.0, "tensor": 1400.0, "tensor_burst": 1590.0, "source": "fallback",
            "sm_max_mhz": 1965.0}


# entry points that take a vr_active_rows list: index of the device row-count argument (the
# launch processes that many samples, not the sample-count argument's n)
ROW_COUNT_ARG = {"vr_mlp_bwd_tc": 13, "vr_mlp_bwd_tc_density": 13, "vr_hash_scatter": 10,
                 "vr_field_bwd_tc": 18}


class _DevInt32:
    """A device int32 at a raw address, viewable by torch (CUDA array interface)."""

    def __init__(self, addr):
        self.__cuda_array_interface__ = {"shape": (1,), "typestr": "<i4", "data": (addr, False),
                                         "version": 3}


class EventTimer:
    """CUDA events around every C-ABI call (current stream); per-entry-point totals."""

    def __init__(self):
        import torch

        self.torch = torch
        self.pending = []
        self.open = {}
        self.samples = {}
        self.row_counts = {}  # name -> device copies of the row counts of sparse launches
        self.dense = {}  # name -> the samples those sparse launches were given

    def before(self, name, args=()):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.open[name] = e
        cost = KERNEL_COST.get(name)
        ri = ROW_COUNT_ARG.get(name)
        if ri is not None and args[ri]:  # a row list: its device count, copied in stream order
            v = self.torch.as_tensor(_DevInt32(args[ri]), device="cuda")
            self.row_counts.setdefault(name, []).append(v.to(self.torch.int64, copy=True))
            self.dense[name] = self.dense.get(name, 0) + int(args[cost[2]])
        elif cost and cost[2] is not None:  # samples this launch processes
            self.samples[name] = self.samples.get(name, 0) + int(args[cost[2]])

    def after(self, name):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.pending.append((name, self.open.pop(name), e))

    def totals(self):
        for name, vs in self.row_counts.items():
            self.samples[name] = self.samples.get(name, 0) + int(sum(int(v) for v in vs))
        self.row_counts = {}
        out = {}
        for name, a, b in self.pending:
            ms = a.elapsed_time(b)
            t, n = out.get(name, (0.0, 0))
            out[name] = (t + ms, n + 1)
        return out


class ClockSampler:
    """SM clock / throttle reasons sampled during the timed region with NVML from a
    background thread (nvidia-smi polling was measured to stall this workload's
    launches; in-process NVML queries do not)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index: int, period: float = 0.1):
        self.index = index
        self.period = period
        self.rows = []
        self.thread = None
        self.stop_flag = False

    def start(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - NVML missing: report no clocks
            self.nv = None
            return

        def loop():
            nv = self.nv
            while not self.stop_flag:
                try:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                    self.rows.append((sm, rs, util))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(self.period)

        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if self.nv is None:
            return None
        self.stop_flag = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        rows = self.rows
        if not rows:
            return None
        reasons = sorted({name for (_, rs, _) in rows for bit, name in self.REASONS.items()
                          if rs & bit})
        loaded = [r for r in rows if r[2] > 50] or rows
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "source": "nvml"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def build_pool(w, rank, world, dev, group, seed_base=1):
    import paper_2404_16221_b200 as vr

    tree = w.tree
    lo, cnt = vr.owned_regions(len(tree.leaves), rank, world)
    cfg = vr.HashGridConfig(log2_T=w.log2_T, max_res=w.max_res)
    # kernel experiments only: force an MLP implementation / hash-grid traversal order
    impl = os.environ.get("VR_BENCH_MLP_IMPL", "fused")
    order = os.environ.get("VR_BENCH_HASH_ORDER", "auto")
    fields = [vr.HashGridMLP(cfg, tree.leaves[k].box, dev, seed=seed_base + k, mlp_impl=impl,
                             hash_order=order) for k in range(lo, lo + cnt)]
    props = None
    if w.interlevel > 0:  # config 4: proposal fields for the interlevel loss
        pcfg = vr.HashGridConfig(log2_T=w.prop_log2_T, max_res=w.prop_max_res)
        # the proposal's colour head is never read: density branch only
        porder = os.environ.get("VR_BENCH_PROP_HASH_ORDER", "auto")
        props = [vr.HashGridMLP(pcfg, tree.leaves[k].box, dev, seed=1000 + k, density_only=True,
                                hash_order=porder)
                 for k in range(lo, lo + cnt)]
    return vr.VolumePool(tree, fields, (0.05, 0.05, 0.08), dev, rank, world, group,
                         proposals=props)


def cpu_baseline_port(w, n_rays: int, seed: int = 0, reps: int = 1, min_seconds: float = 0.0):
    """Oracle port of the training step (sampling, hash-grid + MLP forward, composite, fold,
    loss incl. the interlevel term with proposal fields when the workload has it, torch
    fp64 autograd backward) on a bounded ray sample, 1 thread; the field is evaluated once
    per region over the sample (grad_oracle.field_loss_batched).  Repeats until reps and
    min_seconds are both reached; returns (rays/s, seconds per repetition)."""
    import torch

    from oracle import grad_oracle, hashmlp_oracle as hmo, volray_oracle as vo
    import paper_2404_16221_b200 as vr
    from paper_2404_16221_b200.workloads import make_rays

    torch.set_num_threads(1)
    tree = w.tree
    otree = vo.Tree(vr.tree_to_json(tree))
    rays = make_rays(w, seed, n_rays)
    targets = np.random.default_rng(2).uniform(0, 1, size=(n_rays, 3))
    rng = np.random.default_rng(1)
    runs = grad_oracle.RayRuns(otree, rays.T, w.dt)

    # the port keeps only the table entries this ray sample touches (a dense float64
    # table of 2^19..2^22 entries per region would dominate the CPU time)
    def model(k, log2_T, max_res):
        box = tree.leaves[k].box
        wts = rng.normal(size=hmo.NPARAMS).astype(np.float32) * 0.1
        return hmo.CompactHashMLPModel(
            lambda e: rng.uniform(-1e-4, 1e-4, size=(e.size, 2)).astype(np.float32), wts,
            log2_T, box.mn, box.mx, runs.pts[k], max_res=max_res)

    models = {k: model(k, w.log2_T, w.max_res) for k in runs.regions}
    props = ({k: model(k, w.prop_log2_T, w.prop_max_res) for k in runs.regions}
             if w.interlevel > 0 else None)
    t = time.perf_counter()
    done = 0
    while done < reps or time.perf_counter() - t < min_seconds:
        loss, _, _ = grad_oracle.field_loss_batched(
            otree, lambda k, p, d: models[k].eval_dirs(p, d), rays.T, targets,
            (0.05, 0.05, 0.08), w.dt,
            prop_batch=(lambda k, p, d: props[k].eval_dirs(p, d)) if props else None,
            lambda_int=w.interlevel, runs=runs)
        loss.backward()
        done += 1
    dt = (time.perf_counter() - t) / done
    return n_rays / dt, dt


def _ref_worker(args):
    cfg_name, n_rays, seed = args
    from paper_2404_16221_b200.workloads import CONFIGS

    return cpu_baseline_port(CONFIGS[cfg_name], n_rays, seed)


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle port of the path on all host cores (one process
    per core; each step = every core runs the fwd+bwd of its own ray sample)."""
    if rank != 0:
        return
    from concurrent.futures import ProcessPoolExecutor

    from paper_2404_16221_b200.workloads import CONFIGS

    w = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    per = 64
    with ProcessPoolExecutor(max_workers=cores) as ex:
        for s in range(args.warmup):
            list(ex.map(_ref_worker, [(args.config, per, 1000 + s * cores + c) for c in range(cores)]))
        step_s = []
        for s in range(args.steps):
            res = list(ex.map(_ref_worker, [(args.config, per, s * cores + c) for c in range(cores)]))
            step_s.append(max(dt for _, dt in res))  # cores run concurrently
    sample = cores * per
    value = sample * args.steps / sum(step_s)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * sum(step_s) / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "rays_per_step_sample": sample, "dt": w.dt},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{per} rays per core per step ({sample} rays) of {w.name}: "
                                       "oracle sampling + hash-grid + MLP fwd (+ proposal / "
                                       "interlevel where the workload has it), torch fp64 "
                                       "autograd bwd; 1 process per core, timed region excludes "
                                       "model construction"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


KERNEL_BOUNDS = ROOT / "profiles" / "kernel_bounds.json"


def kernel_bounds(workload: str) -> dict:
    """ncu evidence per kernel for a workload: DRAM bytes per sample and the bound the
    capture shows (profiles/kernel_bounds.json, written from profiles/r2/*)."""
    if not KERNEL_BOUNDS.exists():
        return {}
    d = json.loads(KERNEL_BOUNDS.read_text())
    return d.get(workload.split("-")[0], {})


def nvlink_sweep(group, world, dev, red_dev):
    """all_gather_into_tensor bus bandwidth over 1 MB - 1 GB per rank (the measured NVLink
    peak of this node: max over sizes of the per-rank received bytes / time, max-over-ranks
    time)."""
    import torch
    import torch.distributed as dist

    rows = []
    for mb in (1, 4, 16, 64, 256, 1024):
        n = mb * (1 << 20) // 4
        src = torch.zeros(n, dtype=torch.float32, device=dev)
        out = torch.empty(world * n, dtype=torch.float32, device=dev)
        for _ in range(3):
            dist.all_gather_into_tensor(out, src, group=group)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10 if mb <= 256 else 4
        a.record()
        for _ in range(reps):
            dist.all_gather_into_tensor(out, src, group=group)
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        recv = (world - 1) * n * 4
        rows.append({"mb_per_rank": mb, "ms": round(ms, 4),
                     "gbs_received_per_rank": round(recv / (ms / 1e3) / 1e9, 1)})
        del src, out
    return {"sweep": rows, "peak_gbs": max(r["gbs_received_per_rank"] for r in rows)}


def run_workload(cfg_name, args, rank, world, local, dev, group, red_dev, headline=True):
    """Bench one configuration; returns the fields of its JSON object."""
    import torch
    import torch.distributed as dist

    import paper_2404_16221_b200 as vr
    from paper_2404_16221_b200 import _lib
    from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets

    w = CONFIGS[cfg_name]
    if args.rays:
        w.n_rays = args.rays
    R = w.n_rays
    pool = build_pool(w, rank, world, dev, group)
    train = w.train
    metric = METRIC if train else RENDER_METRIC
    # the interlevel loss is defined on the tile protocol's segments
    interlevel = w.interlevel if args.protocol == "tile" else 0.0
    # distinct batches, rotated step by step (same seeds on every rank: the ray batch is
    # replicated, each rank samples its own regions)
    nb = max(1, args.batches)
    host = [(make_rays(w, seed=s), make_targets(R, seed=100 + s)) for s in range(nb)]
    batches = [(torch.from_numpy(r).to(dev), torch.from_numpy(t).to(dev)) for r, t in host]

    step = 0
    prefetch = train and args.protocol == "tile" and args.prefetch
    pipe = {"pending": None, "cap": 1}

    def one_step(r, t, r_next=None, ready=None):
        nonlocal step
        step += 1
        if train and prefetch:
            if pipe["pending"] is None:
                pipe["pending"] = pool.sample_async(r, w.dt, pipe["cap"])
            b = pool.resolve_sample(pipe["pending"])
            pipe["cap"] = b.n_samples
            pipe["pending"] = pool.sample_async(r if r_next is None else r_next, w.dt,
                                                pipe["cap"], ready)
            return pool.train_step(r, t, w.dt, lr=args.lr, step=step,
                                   lambda_interlevel=interlevel, protocol=args.protocol,
                                   batch=b)
        if train:
            return pool.train_step(r, t, w.dt, lr=args.lr, step=step,
                                   lambda_interlevel=interlevel, protocol=args.protocol)
        out, _ = pool.render_rays(r, w.dt, protocol=args.protocol)  # gathered to rank 0
        return out

    # render: no training state, but one untimed pass over every batch so no timed step is
    # the first to see a batch's buffer sizes (a first-time allocation costs a step ~60 ms)
    burnin = args.burnin if train else nb
    for k in range(burnin + args.warmup):
        one_step(*batches[k % nb])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def f_state(f):
        return [f.table, f.weights] + list(f.adam or [])

    all_fields = pool.fields + (pool.proposals or [])
    snap = [[t.clone() for t in f_state(f)] for f in all_fields]
    snap_step = step
    one_step(*batches[0])  # absorbs the allocator's reaction to the snapshot copies

    def restore():
        nonlocal step
        for f, ts in zip(all_fields, snap):
            for dst, src in zip(f_state(f), ts):
                dst.copy_(src)
            f.refresh_weights()
        step = snap_step
        torch.cuda.synchronize()

    # ---- timed region: inputs resident in HBM -------------------------------------
    restore()
    clocks = ClockSampler(local) if headline else None
    _lib.CALLS.clear()
    _lib.LAUNCHED.clear()
    if clocks:
        clocks.start()
        time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    start.record()
    marks[0].record()
    for k in range(args.steps):
        loss = one_step(*batches[k % nb])
        marks[k + 1].record()
    end.record()
    torch.cuda.synchronize()
    step_ms = [marks[k].elapsed_time(marks[k + 1]) for k in range(args.steps)]
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    calls = dict(_lib.CALLS)
    launched = dict(_lib.LAUNCHED)

    # ---- second pass, same steps, CUDA events around every C-ABI launch: per-kernel
    # durations for the rooflines (kept out of the headline number: the per-launch event
    # records add host work after the step's sync point)
    timer = EventTimer()
    restore()
    _lib.TIMER = timer
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record()
    for k in range(args.steps):
        one_step(*batches[k % nb])
    p1.record()
    torch.cuda.synchronize()
    _lib.TIMER = None
    ms_instrumented = p0.elapsed_time(p1) / args.steps
    ms = start.elapsed_time(end) / args.steps
    t_ms = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms = float(t_ms.item())
    value = R / (ms / 1e3)
    launches = sum(launched.values())
    if world > 1:  # k_sample_prefilter + the walk
        launches += calls.get("vr_sample_stage", 0)
    final_loss = float(loss.item()) if train else None

    # samples per step (for per-sample kernel costs), batch 0
    b = pool.sample(batches[0][0], w.dt)
    n_samples_rank = b.n_samples
    n_samples = torch.tensor([n_samples_rank], dtype=torch.int64, device=red_dev)
    if world > 1:
        dist.all_reduce(n_samples)
    n_samples = int(n_samples.item())
    n_live = (b.counts > 0).sum(dtype=torch.int64).reshape(1).to(red_dev)
    if world > 1:
        dist.all_reduce(n_live)
    n_live = int(n_live.item())

    link = None
    if world > 1 and args.protocol == "tile" and headline:
        b_ex = pool.sample(batches[0][0], w.dt, exchange=True)
        rows = (b_ex.seg_max or 0) + 1
        width = 10 if interlevel else 9
        buf = torch.zeros((rows, width), dtype=torch.float32, device=dev)
        for _ in range(3):
            vr.comm.all_gather_packets(buf, group, world)
        torch.cuda.synchronize()
        dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        for _ in range(10):
            vr.comm.all_gather_packets(buf, group, world)
        eb.record()
        torch.cuda.synchronize()
        x_ms = torch.tensor([ea.elapsed_time(eb) / 10], dtype=torch.float64, device=red_dev)
        dist.all_reduce(x_ms, op=dist.ReduceOp.MAX)
        x_ms = float(x_ms.item())
        recv = (world - 1) * rows * width * 4
        sweep = nvlink_sweep(group, world, dev, red_dev) if args.backend == "nccl" else None
        peak = sweep["peak_gbs"] if sweep else 900.0
        link = {"collective": "all_gather_into_tensor of the sparse packet records",
                "bytes_received_per_rank": recv, "ms": x_ms,
                "achieved": recv / (x_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": recv / (x_ms / 1e3) / 1e9 / peak,
                "peak_source": ("measured: max over an all_gather_into_tensor sweep of "
                                "1 MB - 1 GB per rank on this node" if sweep else
                                "nominal NVLink 5 per direction (gloo run)"),
                "sweep": sweep["sweep"] if sweep else None, "backend": args.backend}

    # ---- rooflines (events over the timed region) -----------------------------------
    totals = timer.totals()
    peaks = load_peaks()
    evidence = kernel_bounds(w.name)
    ceilings = (json.loads(KERNEL_BOUNDS.read_text()).get("ceilings", {})
                if KERNEL_BOUNDS.exists() else {})
    per_kernel = {k: {"ms_per_step": t / args.steps, "launches": n} for k, (t, n) in totals.items()}

    def roof(k):
        bound, per_unit, _ = KERNEL_COST[k]
        t_total, n_launch = totals[k]
        units = timer.samples.get(k, n_samples_rank * args.steps)
        avg_s = (t_total / 1e3) / n_launch
        per_launch = per_unit * units / n_launch
        if bound == "hbm":
            achieved, peak, unit = per_launch / avg_s / 1e9, peaks["hbm"], "GB/s"
        else:
            achieved, peak, unit = per_launch / avg_s / 1e12, peaks["tensor"], "TFLOP/s"
        ev = evidence.get(k, {})
        dram = ev.get("dram_bytes_per_sample")
        traffic = dram * units / n_launch if dram else None
        out = {"kernel": k, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
               "frac": achieved / peak, "traffic": traffic,
               "algorithmic_per_launch": per_launch,
               "dram_frac": (traffic / avg_s / 1e9 / peaks["hbm"]) if traffic else None,
               "ncu_bound": ev.get("bound"), "evidence": ev.get("source"),
               "ms_per_step": t_total / args.steps,
               "share_of_step": t_total / args.steps / ms_instrumented}
        reqs = ev.get("l2_read_requests_per_sample", 0.0) + ev.get("l2_red_requests_per_sample", 0.0)
        if reqs > 1.0 and ("hash" in k or k == "vr_field_bwd_tc"):
            # the hash-grid gather / scatter kernels: the L2 request roofline they run against
            ceil = ceilings.get("l2_red_requests_per_s" if ev.get("l2_red_requests_per_sample", 0)
                                > ev.get("l2_read_requests_per_sample", 0)
                                else "l2_gather_requests_per_s")
            # the rate of the ncu capture (one launch timed alone): a launch timed with
            # events inside the step overlaps the other stream's kernels
            got = ev["l2_requests_per_s"]
            # the contract's "bound" is hbm | tensor; what binds these kernels is the L2
            # request rate (their DRAM traffic is a fraction of the logical bytes)
            out["binding"] = "L2 request rate (request_roofline)"
            out["request_roofline"] = {"achieved": got / 1e9, "ceiling": ceil / 1e9,
                                       "unit": "G L2 requests/s", "frac": got / ceil,
                                       "requests_per_sample": reqs,
                                       "measured": "ncu --set full capture of one launch "
                                                   "(requests / its duration)",
                                       "ceiling_source": ceilings.get("source")}
        return out

    costed = [k for k in totals if k in KERNEL_COST and totals[k][0] > 0]
    dom = max(costed, key=lambda k: totals[k][0], default=None)
    roofline = roof(dom) if dom else None
    if roofline:
        roofline["peak_source"] = peaks["source"]
        roofline["ms_per_step_instrumented"] = ms_instrumented
    rooflines = {}
    for k in costed:
        r = roof(k)
        rooflines[k] = {key: (round(v, 4) if isinstance(v, float) else v) for key, v in r.items()
                        if key not in ("kernel", "algorithmic_per_launch")}

    # ---- end to end through the public API with host buffers ------------------------
    e2e = None
    if not args.no_e2e:
        pinned = [(torch.from_numpy(r).pin_memory(), torch.from_numpy(t).pin_memory())
                  for r, t in host]
        restore()
        if world > 1:
            dist.barrier()
        copy_stream = torch.cuda.Stream(device=dev)
        main_stream = torch.cuda.current_stream()

        def fetch(k):  # render needs no targets
            rh, th = pinned[k % nb]
            with torch.cuda.stream(copy_stream):
                r = rh.to(dev, non_blocking=True)
                t = th.to(dev, non_blocking=True) if train else None
                ev = torch.cuda.Event()
                ev.record(copy_stream)
            return r, t, ev

        out_h = None if train else torch.empty((3, R), dtype=torch.float32, pin_memory=True)

        def e2e_loop(steps):
            nxt = fetch(0)
            for k in range(steps):
                r_d, t_d, ev = nxt
                main_stream.wait_event(ev)
                r_d.record_stream(main_stream)
                if t_d is not None:
                    t_d.record_stream(main_stream)
                if k + 1 < steps:
                    nxt = fetch(k + 1)
                    res = one_step(r_d, t_d, nxt[0], nxt[2])
                else:
                    res = one_step(r_d, t_d)
                if train:
                    _ = float(res.item())  # D2H read of the step's loss
                elif res is not None:  # D2H read of the rendered colours
                    out_h.copy_(res[0:3], non_blocking=True)
                    torch.cuda.current_stream().synchronize()

        e2e_loop(max(args.warmup, nb))  # untimed warm-up of the pipeline, every batch
        torch.cuda.synchronize()
        restore()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        e2e_loop(args.steps)
        t1.record()
        torch.cuda.synchronize()
        e_ms = torch.tensor([t0.elapsed_time(t1) / args.steps], dtype=torch.float64,
                            device=red_dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": R / (float(e_ms.item()) / 1e3), "unit": UNIT,
               "input_pipeline": f"{nb} distinct pinned host batches rotated, H2D on a copy "
                                 "stream one step ahead",
               "h2d_bytes_per_step": host[0][0].nbytes + (host[0][1].nbytes if train else 0),
               "d2h_bytes_per_step": 8 if train else 3 * 4 * R, "ms_per_step": float(e_ms.item())}
        del pinned

    half = max(1, args.steps // 2)
    first, second = step_ms[:half], step_ms[half:] or step_ms[:half]
    trend = (statistics.mean(second) - statistics.mean(first)) / statistics.mean(first)
    res = {"metric": metric, "value": value, "unit": UNIT, "ms_per_step": ms,
           "ms_per_step_median": statistics.median(step_ms),
           "step_ms": [round(x, 3) for x in step_ms],
           "step_ms_trend": round(trend, 4),
           "config": {"workload": w.name, "rays_per_step": R, "samples_per_step": n_samples,
                      "samples_per_ray": n_samples / R, "regions": len(w.tree.leaves),
                      "regions_per_gpu": len(w.tree.leaves) // world, "log2_T": w.log2_T,
                      "dt": w.dt, "parallelism": f"region-parallel x{world}",
                      "partition": (f"sample-balanced median splits (data/{w.partition})"
                                    if w.partition != "grid" else "uniform grid"),
                      "batches": f"{nb} distinct ray batches rotated (seeds 0..{nb - 1})",
                      "state": (f"trained {burnin} + {args.warmup} steps before timing; every "
                                "timed pass restarts from that snapshot" if train else
                                f"random-init fields; {burnin} + {args.warmup} untimed steps"),
                      "l2": "inputs larger than L2 (tables+rays+samples >> 126 MB)",
                      "optimizer": "adam" if train else None,
                      "loss": (("mse+distortion+interlevel" if interlevel else
                                "mse+distortion") if train else None),
                      "protocol": args.protocol},
           "exchange": {
               "protocol": args.protocol,
               "wire": ("36 B/non-empty segment" + (" (+4 B proposal T)" if interlevel else "")
                        if args.protocol == "tile" else "16 B/sample (sigma, rgb)"),
               "nonempty_segments": n_live, "segments": len(w.tree.leaves) * R,
               "bytes_per_step_1_region_per_gpu": (n_live * (40 if interlevel else 36)
                                                   if args.protocol == "tile"
                                                   else n_samples * 16),
               "dense_slab_bytes": len(w.tree.leaves) * R * (36 if interlevel else 32),
               "tile_vs_sample_bytes": (n_live * (40 if interlevel else 36))
               / max(1, n_samples * 16)},
           "roofline": roofline, "rooflines": rooflines, "nvlink": link, "e2e": e2e,
           "gpu_launches": launches, "clocks": clk, "loss": final_loss, "kernels": per_kernel,
           # sparse backward: the fraction of each field backward's samples with a non-zero
           # upstream gradient (the rest sit behind opaque surfaces: exactly zero gradients)
           "active_rows": {k: round(timer.samples.get(k, 0) / v, 4)
                           for k, v in timer.dense.items() if v},
           # K4's forward stages its inputs by TMA when tensor maps can be encoded
           "tma": bool(_lib.load().vr_tma_available())}
    del pool, batches
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res, w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--sub", default="c3,c5",
                    help="further configs reported in the same line (sub_results); '' for none")
    ap.add_argument("--burnin", type=int, default=24,
                    help="training steps before the warm-up (steady training state)")
    ap.add_argument("--batches", type=int, default=4, help="distinct ray batches rotated")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lr", type=float, default=1e-2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--rays", type=int, default=None, help="override rays per step")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo + --same-device: exercise the multi-rank path on one GPU")
    ap.add_argument("--same-device", action="store_true", help="all ranks on cuda:0 (testing)")
    ap.add_argument("--prefetch", action="store_true",
                    help="sample the next batch one step ahead on a second stream (measured "
                         "54.4 vs 53.2 ms/step at c3, e2e 63.1 vs 54.5: K1 finds few free SM "
                         "slots next to the field kernels and slows them down)")
    ap.add_argument("--protocol", default="tile", choices=["tile", "sample"],
                    help="tile: NeRF-XL segment packets; sample: per-sample broadcast baseline")
    args = ap.parse_args()
    rank, world, local = dist_env()

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
        group = dist.group.WORLD
    red_dev = dev if args.backend == "nccl" else torch.device("cpu")

    res, w = run_workload(args.config, args, rank, world, local, dev, group, red_dev)
    subs = {}
    for name in [c for c in args.sub.split(",") if c and c not in (args.config, "none")]:
        r, _ = run_workload(name, args, rank, world, local, dev, group, red_dev, headline=False)
        subs[name] = {k: r[k] for k in ("metric", "value", "unit", "ms_per_step",
                                        "ms_per_step_median", "step_ms_trend", "config", "e2e",
                                        "roofline", "rooflines", "gpu_launches", "exchange")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and w.train:
        # a bounded ray sample of the headline workload, repeated: ~10-30 s of single-thread
        # CPU work (larger samples make the port's compact tables and autograd graph slower
        # per ray, not more representative)
        n_cpu = 256
        v, per_rep = cpu_baseline_port(w, n_cpu, reps=2, min_seconds=10.0)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{n_cpu} rays of {w.name}, repeated for >= 10 s ({per_rep:.2f} s per "
                         "repetition): oracle sampling + hash+MLP fwd (+ proposal / interlevel), "
                         "composite, loss, torch fp64 autograd bwd, single thread"}

    if rank == 0:
        line = {"metric": res["metric"], "value": res["value"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32+f16", "data": "synthetic"}
        line.update({k: v for k, v in res.items() if k not in ("metric", "value", "unit",
                                                                "ms_per_step")})
        line["cpu_baseline"] = cpu
        line["sub_results"] = subs
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
