"""Diagnose C1 gradient differences: per-sample d(enc) (GPU split MLP backward) vs the
oracle's d(enc), then the table gradient by level."""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_16221_b200 as vr  # noqa: E402
from oracle import grad_oracle, hashmlp_oracle as hmo, volray_oracle as vo  # noqa: E402
from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets  # noqa: E402
from test_gpu_configs import BG, _c1_model  # noqa: E402

w = CONFIGS["c1"]
tree = w.tree
table, wts = _c1_model()
cfg = vr.HashGridConfig(log2_T=w.log2_T, max_res=w.max_res)
box = tree.leaves[0].box
f = vr.HashGridMLP(cfg, box, "cuda", table=torch.from_numpy(table), weights=torch.from_numpy(wts))
pool = vr.VolumePool(tree, [f], BG, "cuda")
rays = make_rays(w)
tg = make_targets(w.n_rays).astype(np.float64)

# capture d(enc) of the split backward
captured = {}
orig = f.backward_mlp


def cap(*a, **k):
    d = orig(*a, **k)
    captured["denc"] = d
    return d


f.backward_mlp = cap
orig_jobs = pool.field_backward_jobs


def jobs_cap(rays_, b_, jobs):
    captured["dsig"] = jobs[0][1].clone()
    return orig_jobs(rays_, b_, jobs)


pool.field_backward_jobs = jobs_cap
pool.zero_grad()
loss, out, b = pool.loss_and_grad(rays, tg, w.dt)
torch.cuda.synchronize()
n = b.n_samples
denc = captured["denc"].view(16, -1, 2)[:, :n].permute(1, 0, 2).reshape(n, 32).cpu().numpy()
# GPU sample order (region-major, ray-major inside) -> oracle order (ray-major)
rid = b.ray_id[:n].cpu().numpy()
t0g = b.t0[:n].cpu().numpy()

m = hmo.HashMLPModel(table, wts, w.log2_T, box.mn, box.mx, max_res=w.max_res)
otree = vo.Tree(vr.tree_to_json(tree))
runs = grad_oracle.RayRuns(otree, rays.T, w.dt)
encs = {}
orig_enc = m.encode


def enc_cap(pts):
    e = orig_enc(pts)
    e.retain_grad()
    encs["e"] = e
    return e


m.encode = enc_cap
orig_mlp = m.mlp


def mlp_cap(enc, dirs32):
    sg, rg = orig_mlp(enc, dirs32)
    sg.retain_grad()
    rg.retain_grad()
    encs["sig"], encs["rgb"] = sg, rg
    return sg, rg


m.mlp = mlp_cap
oloss, oout, _ = grad_oracle.field_loss_batched(otree, lambda k, p, d: m.eval_dirs(p, d), rays.T, tg,
                                                BG, w.dt, runs=runs)
oloss.backward()
oden = encs["e"].grad.numpy()
dsig = captured["dsig"][:n].cpu().numpy().astype(np.float64)
odsig = np.concatenate([encs["sig"].grad.numpy()[:, None], encs["rgb"].grad.numpy()], 1)
e_up = np.abs(dsig - odsig) / (np.abs(odsig).max(1, keepdims=True) + 1e-30)
print("upstream d(sigma,rgb) rel err quantiles", np.quantile(e_up.max(1), [0.5, 0.9, 0.99, 0.999, 1.0]))
# MLP alone: the oracle MLP driven by the GPU's own upstream gradient and encodings
enc16 = torch.tensor(encs["e"].detach().numpy(), requires_grad=True)
sg, rg = orig_mlp(enc16, runs.dirs[0].astype(np.float32))
torch.autograd.backward([sg, rg], [torch.from_numpy(dsig[:, 0]), torch.from_numpy(dsig[:, 1:4])])
e_mlp = np.abs(denc - enc16.grad.numpy()) / (np.abs(enc16.grad.numpy()).max(1, keepdims=True) + 1e-30)
print("MLP-only d(enc) rel err quantiles", np.quantile(e_mlp.max(1), [0.5, 0.9, 0.99, 0.999, 1.0]))
print("n", n, runs.n_samples, "loss", loss.item(), oloss.item())
# oracle order is ray-major with t order (region 0 only): same as GPU order for K=1
assert np.array_equal(runs.t0, t0g)
err = np.abs(denc - oden)
scale = np.abs(oden).max(1, keepdims=True) + 1e-30
rel = (err / scale).max(1)
print("per-sample d(enc) rel err (max over 32 / max |d(enc)| of the sample): quantiles",
      np.quantile(rel, [0.5, 0.9, 0.99, 0.999, 1.0]))
print("margins of the worst samples", m.last_margin[np.argsort(rel)[-10:]], rel[np.argsort(rel)[-10:]])
gt, gw = m.grads()
mine = f.grad_table.cpu().numpy()
gmax = np.abs(gt).max()
lv, _ = hmo.levels(w.log2_T, max_res=w.max_res)
for l, (s, r, dn, off) in enumerate(lv):
    hi = lv[l + 1][3] if l + 1 < len(lv) else gt.shape[0]
    a, bb = mine[off:hi], gt[off:hi]
    big = np.abs(bb) > 1e-3 * gmax
    e = np.abs(a - bb)
    bad = np.where(big, e > 1e-3 * np.abs(bb), e > 1e-6 * gmax)
    print(f"level {l:2d} res {r:4d} dense {dn}: max|g| {np.abs(bb).max() / gmax:.2e}*max, "
          f"max abs err {e.max() / gmax:.2e}*max, bad {int(bad.sum())} of {bb.size}")
# reconstruct the table gradient from the GPU d(enc) with the oracle's float64 scatter
u = hmo.normalize(runs.pts[0], box.mn, box.mx)
rec = np.zeros_like(gt)
for l, (s, r, dn, off) in enumerate(lv):
    idx, wt = hmo.corners(u, s, r, dn, w.log2_T)
    for c in range(8):
        np.add.at(rec, idx[:, c].astype(np.int64) + off, wt[:, c:c + 1].astype(np.float64) * denc[:, 2 * l:2 * l + 2])
e = np.abs(mine - rec)
print("scatter only: max abs err", e.max() / gmax, "bad", int(((e > 1e-3 * np.abs(rec)) & (np.abs(rec) > 1e-3 * gmax)).sum()))

# per-entry: sum of |contributions| (oracle) and the largest single contribution error
S = np.zeros_like(gt)
big_c = np.zeros_like(gt)
for l, (s, r, dn, off) in enumerate(lv):
    idx, wt = hmo.corners(u, s, r, dn, w.log2_T)
    for c in range(8):
        ii = idx[:, c].astype(np.int64) + off
        np.add.at(S, ii, np.abs(wt[:, c:c + 1].astype(np.float64) * oden[:, 2 * l:2 * l + 2]))
big = np.abs(gt) > 1e-3 * gmax
e = np.abs(mine - gt)
bad = big & (e > 1e-3 * np.abs(gt))
cf = S[bad] / np.abs(gt[bad])
print("failing entries: cancellation factor S/|g| quantiles", np.quantile(cf, [0, 0.1, 0.5, 0.9, 1.0]))
print("all big entries: S/|g| quantiles", np.quantile(S[big] / np.abs(gt[big]), [0.5, 0.9, 0.99, 0.999]))
print("failing entries: err/S quantiles", np.quantile(e[bad] / S[bad], [0, 0.5, 0.9, 1.0]))
print("all entries: err/S quantiles", np.quantile(e[S > 0] / S[S > 0], [0.5, 0.9, 0.99, 0.999, 1.0]))
# the worst per-sample outliers: forward values
worst = np.argsort(rel)[-5:]
sig_o, rgb_o = m.eval_dirs(runs.pts[0][worst], runs.dirs[0][worst])
print("worst samples sigma (oracle)", sig_o.detach().numpy(), "margin", m.last_margin)
print("their |d(enc)| max", np.abs(oden[worst]).max(1), "median sample", np.median(np.abs(oden).max(1)))

# theory check: the same MLP backward with the upstream gradient scaled by 2^10 (linear)
from paper_2404_16221_b200 import _lib  # noqa: E402
for sc in (1.0, 2.0 ** 6, 2.0 ** 10):
    dsr = (captured["dsig"][:n] * sc).contiguous()
    gwt = torch.zeros_like(f.grad_weights)
    de = torch.empty(16 * n * 2, dtype=torch.float32, device="cuda")
    err_w = torch.zeros(1, dtype=torch.int32, device="cuda")
    rd = pool.rays_to_device(rays)
    _lib.call("vr_mlp_bwd_tc", _lib.ptr(f.weights16), _lib.ptr(f._enc), _lib.ptr(rd), rd.shape[1],
              _lib.ptr(b.ray_id), n, _lib.ptr(dsr), None, _lib.ptr(gwt), _lib.ptr(de), _lib.ptr(err_w), 0,
              None, None, _lib.stream_ptr())
    torch.cuda.synchronize()
    d2 = (de.view(16, -1, 2)[:, :n].permute(1, 0, 2).reshape(n, 32).cpu().numpy() / sc)
    e2 = np.abs(d2 - enc16.grad.numpy()) / (np.abs(enc16.grad.numpy()).max(1, keepdims=True) + 1e-30)
    gwo = gwt.cpu().numpy() / sc
    print(f"scale {sc}: MLP-only d(enc) rel err quantiles", np.quantile(e2.max(1), [0.5, 0.9, 0.99, 0.999, 1.0]),
          "flags", err_w.item(), "weights norm rel", np.linalg.norm(gwo - gw) / np.linalg.norm(gw))
