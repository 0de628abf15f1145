"""One rank's share of the c4 training step at N ranks, timed on one GPU.

Each rank r of N owns K/N regions; its step runs K1 for its regions over the whole
(replicated) ray batch, its fields, K4, the packet exchange, K5 over all rays, the
interlevel loss and the backward of its own regions.  Here rank r's pool (world = N, no
process group) trains in lockstep with a one-GPU pool of all K regions on the same batches:
the one-GPU pool's packets stand in for the other ranks' (what they would send: every
region's parameters follow the same updates — no gradient crosses ranks), so rank r sees
the real global composite and the real sparsity of its backward.  Only the NVLink transfer
of the records is absent (bench.py's `nvlink` sweep times it on a multi-GPU node).
Steady state as in bench.py: 24 + 3 burn-in steps over four rotating batches, then timed
steps; the one-GPU pool's steps are not timed.

    python scripts/rank_share.py [N=8] [ranks...]"""
import gc
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch

import bench
from paper_2404_16221_b200 import _lib, comm
from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ranks = [int(a) for a in sys.argv[2:]] or list(range(N))
w = CONFIGS["c4"]
DEV = "cuda:0"
comm.all_reduce_scalar = lambda x, group=None, world=1: x  # (the interlevel term's SUM)

batches = [(torch.from_numpy(make_rays(w, seed=s)).to(DEV),
            torch.from_numpy(make_targets(w.n_rays, seed=100 + s)).to(DEV)) for s in range(4)]
res, kern = {}, {}
for r in ranks:
    full = bench.build_pool(w, 0, 1, DEV, None)
    rp = bench.build_pool(w, r, N, DEV, None)
    rp.sparse_exchange = False  # the stand-in exchange hands over dense slabs
    stash = {}
    orig_full = full.exchange_packets

    def full_exchange(b, local, extra=None, dst=None, orig=orig_full):
        stash["pk"], stash["T"] = local, extra
        return orig(b, local, extra, dst)

    def rank_exchange(b, local, extra=None, dst=None, rp=rp):
        lo, cnt = rp.region_lo, rp.region_cnt
        pk = stash["pk"].clone()
        pk[lo:lo + cnt] = local
        T = None
        if extra is not None:
            T = stash["T"].clone()
            T[lo:lo + cnt] = extra
        return pk, T

    full.exchange_packets = full_exchange
    rp.exchange_packets = rank_exchange
    step = 0

    def one(k, timed, timer=None):
        global step
        step += 1
        rr, tt = batches[k % 4]
        full.train_step(rr, tt, w.dt, lr=1e-2, step=step, lambda_interlevel=w.interlevel)
        torch.cuda.synchronize()  # (no empty_cache here: re-allocating inside the timed step
        # leaves the GPU idle behind the host's cudaMalloc calls)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _lib.TIMER = timer
        e0.record()
        rp.train_step(rr, tt, w.dt, lr=1e-2, step=step, lambda_interlevel=w.interlevel)
        e1.record()
        torch.cuda.synchronize()
        _lib.TIMER = None
        return e0.elapsed_time(e1)

    for k in range(27):
        one(k, False)
    ms = [one(k, True) for k in range(8)]
    res[r] = sorted(ms)[len(ms) // 2]
    if r == ranks[0]:  # per-kernel breakdown (CUDA events around every C-ABI call)
        timer = bench.EventTimer()
        for k in range(4):
            one(k, True, timer)
        tot = timer.totals()
        kern[r] = {k: t / 4 for k, (t, _) in tot.items()}
        print(f"rank {r}: " + ", ".join(f"{k} {t:.2f}" for k, t in sorted(
            kern[r].items(), key=lambda x: -x[1]) if t > 0.2), flush=True)
    print(f"rank {r} of {N} (regions {rp.region_lo}..{rp.region_lo + rp.region_cnt - 1}): "
          f"{res[r]:.2f} ms per step (median of 8)", flush=True)
    # the closures hold both pools: drop them before the next rank's pools are built
    stash.clear()
    del full_exchange, rank_exchange, one, orig_full, full, rp
    gc.collect()
    torch.cuda.empty_cache()
print(f"max over ranks {max(res.values()):.2f} ms (ranks timed: {sorted(res)})")
