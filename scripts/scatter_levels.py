"""Per-level cost of the level-major hash scatter / gather on real c4 samples.

Trains the c4 pool a few steps (so d(enc) has the steady state's exact zeros), captures
region 0's d(enc) and positions, then times vr_hash_scatter / vr_hash_fwd_lm on one level at
a time (a one-level descriptor over that level's table slice), and counts the duplicate
table indices among the 16 samples of each warp step (what a warp-level pre-reduction of
equal addresses would save)."""
import ctypes
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib as L
from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets

DEV = "cuda:0"
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
pool = bench.build_pool(w, 0, 1, DEV, None)
rays = torch.from_numpy(make_rays(w)).to(DEV)
tg = torch.from_numpy(make_targets(w.n_rays, seed=100)).to(DEV)
for s in range(steps):
    pool.train_step(rays, tg, w.dt, lr=1e-2, step=s + 1, lambda_interlevel=w.interlevel)
torch.cuda.synchronize()

cap = {}
for name, f in (("nerf", pool.fields[0]), ("prop", (pool.proposals or [None])[0])):
    if f is None:
        continue
    orig = f.backward_scatter

    def grab(denc, n, stream, max_blocks=0, rows=None, f=f, orig=orig, name=name):
        rw = (rows[0].clone(), rows[1].clone()) if rows is not None else None
        cap[name] = (f, denc.clone(), n, f._pos[:3 * n].clone(), rw)
        return orig(denc, n, stream, max_blocks, rows=rows)

    f.backward_scatter = grab
pool.train_step(rays, tg, w.dt, lr=1e-2, step=steps + 1, lambda_interlevel=w.interlevel)
torch.cuda.synchronize()
s = L.stream_ptr()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / reps


for name, (f, denc, n, pos, rw) in cap.items():
    if rw is not None:  # a sparse backward ran: time the scatter over its row list
        grad = torch.zeros_like(f.grad_table)
        ws = f._workspace(DEV)
        tr = timeit(lambda: L.call("vr_hash_scatter", L.addr(f.desc), L.ptr(pos), n, L.ptr(denc),
                                   L.ptr(grad), L.ptr(ws), ws.numel(), 1, 0, L.ptr(rw[0]),
                                   L.ptr(rw[1]), s))
        print(f"== {name}: sparse scatter over {rw[1].item()} of {n} rows: {tr:.3f} ms")
        continue
    d = f.desc
    grad = torch.zeros_like(f.grad_table)
    ws = f._workspace(DEV)
    tot = timeit(lambda: L.call("vr_hash_scatter", L.addr(d), L.ptr(pos), n, L.ptr(denc),
                                L.ptr(grad), L.ptr(ws), ws.numel(), 1, 0, None, None, s))
    dv = denc.view(16, n, 2)
    nz = (dv != 0).any(-1).float().mean(1).cpu().numpy()
    print(f"== {name}: {n} samples, full scatter {tot:.3f} ms, passes "
          f"{L.load().vr_hash_lm_passes(L.addr(d))}", flush=True)
    # indices of all 16 levels for a sample subset (duplicates within warp steps)
    m = min(n, 1 << 20)
    idx = torch.empty((16, m, 8), dtype=torch.int32, device=DEV)
    # positions -> indices: reuse vr_hash_indices needs rays; compute from pos on host
    pu = pos.view(3, n)[:, :m].cpu().numpy()
    for l in range(16):
        one = L.VrHashGridDesc()
        one.n_levels = 1
        one.log2_T = d.log2_T
        one.scale[0] = d.scale[l]
        one.res[0] = d.res[l]
        one.dense[0] = d.dense[l]
        one.offset[0] = 0
        one.offset[1] = d.offset[l + 1] - d.offset[l]
        for a in range(3):
            one.box_mn[a] = d.box_mn[a]
            one.box_mx[a] = d.box_mx[a]
        g_l = grad[d.offset[l]:]
        t_l = f.table[d.offset[l]:]
        dl = dv[l].contiguous()
        enc = torch.empty(n, dtype=torch.float32, device=DEV)
        ts = timeit(lambda: L.call("vr_hash_scatter", L.addr(one), L.ptr(pos), n, L.ptr(dl),
                                   L.ptr(g_l), None, 0, 1, 0, None, None, s))
        tf = timeit(lambda: L.call("vr_hash_fwd_lm", L.addr(one), L.ptr(t_l), L.ptr(pos), n,
                                   L.ptr(enc), s))
        # duplicate corner indices among the 16 consecutive samples of a warp step
        sc = np.float32(d.scale[l])
        p = (pu * sc).astype(np.float32) + np.float32(0.5)
        gi = np.clip(np.floor(p).astype(np.int64), 0, d.res[l] - 2)
        key = gi[0] + 4096 * (gi[1] + 4096 * gi[2])
        kk = key[: (m // 16) * 16].reshape(-1, 16)
        uniq = np.mean([len(np.unique(r)) for r in kk[:20000]])
        print(f"  level {l:2d} res {d.res[l]:5d} {'dense' if d.dense[l] else 'hash '} "
              f"entries {int(one.offset[1]):9d}: scatter {ts:.3f} ms  gather {tf:.3f} ms  "
              f"nonzero d(enc) {nz[l]:.3f}  unique cells per 16 {uniq:.2f}", flush=True)
