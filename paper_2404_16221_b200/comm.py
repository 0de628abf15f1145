"""The paper's communication step: exchange of per-(region, ray) packets.

Replaces the simulated transit of TilePayloads to the compositor (distsim.py:435-446)
and the training-mode broadcast (distsim.py:457-475).  One process per GPU; rank r
owns the contiguous region block [r*K/N, (r+1)*K/N), so the concatenation of every
rank's packet slab in rank order IS the global [K][R][8] slab — one all-gather, no
reordering.  Only forward partials cross the link; there is no gradient collective.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def owned_regions(n_regions: int, rank: int, world: int) -> tuple[int, int]:
    """(region_lo, region_cnt) of a rank; regions split evenly and contiguously
    (leaves are depth-first, so each block is a subtree, partitioner.py:145-149)."""
    if world < 1 or n_regions % world != 0:
        raise ValueError(f"{n_regions} regions cannot be split evenly over {world} ranks")
    cnt = n_regions // world
    return rank * cnt, cnt


def _host_staged(group, t: torch.Tensor) -> bool:
    """gloo moves host memory: stage CUDA tensors through the CPU (tests / single-GPU
    multi-rank runs); NCCL moves device memory over NVLink directly."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def all_gather_packets(local: torch.Tensor, group=None, world: int = 1) -> torch.Tensor:
    """[K_own, R, 8] on every rank -> [world*K_own, R, 8] on every rank (training); any
    tensor is concatenated along dim 0 (the sparse exchange's [rows][width] buffers)."""
    if world == 1:
        return local
    src = local.contiguous()
    if _host_staged(group, src):
        cpu = src.cpu()
        parts = [torch.empty_like(cpu) for _ in range(world)]
        dist.all_gather(parts, cpu, group=group)
        return torch.cat(parts, dim=0).to(local.device)
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out


def exchange_samples(sig_rgb: torch.Tensor, bounds, n_regions: int, group=None, world: int = 1,
                     rank: int = 0, dst=None):
    """Sample-broadcast protocol (distsim.py:311-316): every rank sampled all regions and
    evaluated its own block [bounds[lo], bounds[lo+cnt]) of the region-major [N, 4]
    (sigma, r, g, b) array; the other ranks' blocks are filled in place.  dst=None:
    all-gather (training, every rank composes); dst=r: gather to rank r only (render).
    16 B per sample cross the link (t0/t1 are recomputed by every rank's K1).  Returns
    False on ranks that did not receive (gather)."""
    if world == 1:
        return True
    per = n_regions // world
    blocks = [(int(bounds[r * per]), int(bounds[(r + 1) * per])) for r in range(world)]
    m = max(1, max(hi - lo for lo, hi in blocks))
    lo, hi = blocks[rank]
    mine = torch.zeros((m, 4), dtype=sig_rgb.dtype, device=sig_rgb.device)
    mine[: hi - lo] = sig_rgb[lo:hi]
    staged = _host_staged(group, mine)
    src = mine.cpu() if staged else mine
    if dst is None:
        if staged:
            parts = [torch.empty_like(src) for _ in range(world)]
            dist.all_gather(parts, src, group=group)
            allp = torch.cat(parts, dim=0).to(sig_rgb.device)
        else:
            allp = torch.empty((world * m, 4), dtype=sig_rgb.dtype, device=sig_rgb.device)
            dist.all_gather_into_tensor(allp, src, group=group)
    else:
        if rank == dst:
            parts = [torch.empty_like(src) for _ in range(world)]
            dist.gather(src, gather_list=parts, dst=dst, group=group)
            allp = torch.cat(parts, dim=0).to(sig_rgb.device)
        else:
            dist.gather(src, gather_list=None, dst=dst, group=group)
            return False
    for r, (blo, bhi) in enumerate(blocks):
        if r != rank and bhi > blo:
            sig_rgb[blo:bhi] = allp[r * m: r * m + (bhi - blo)]
    return True


def gather_packets(local: torch.Tensor, group=None, world: int = 1, rank: int = 0, dst: int = 0):
    """Inference: packets only need to reach one compositor rank."""
    if world == 1:
        return local
    src = local.contiguous()
    staged = _host_staged(group, src)
    if staged:
        src = src.cpu()
    if rank == dst:
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.gather(src, gather_list=parts, dst=dst, group=group)
        return torch.cat(parts, dim=0).to(local.device)
    dist.gather(src, gather_list=None, dst=dst, group=group)
    return None


def all_reduce_max_(t: torch.Tensor, group=None, world: int = 1) -> torch.Tensor:
    """In-place MAX over the ranks of a small tensor (the sparse exchange's record count)."""
    if world == 1:
        return t
    if _host_staged(group, t):
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MAX, group=group)
        t.copy_(c)
        return t
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def all_reduce_scalar(x: torch.Tensor, group=None, world: int = 1) -> torch.Tensor:
    """In-place SUM over the ranks of a per-rank scalar (the interlevel loss: each rank sums
    its own segments' terms; the main loss term is already identical everywhere)."""
    if world == 1:
        return x
    if _host_staged(group, x):
        c = x.cpu()
        dist.all_reduce(c, group=group)
        x.copy_(c)
        return x
    dist.all_reduce(x, group=group)
    return x
