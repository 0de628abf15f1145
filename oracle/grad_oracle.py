"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Differentiable float64 restatement (torch CPU autograd) of the NeRF-XL training
loss on top of the reference tile protocol, used to check the CUDA analytic
backward (K5 bwd -> K4 bwd -> field bwd).  The loss is the reference probe's
definition (segrender.py:198-207): sum over rays of |C + T*bg - target|^2 plus the
composed distortion; sample geometry comes from volray_oracle.sample_ray.

Pinned against the reference's own finite-difference gradients
(DistributedLossProbe.gradient_pair, segrender.py:235-251) by
tests/test_oracle_golden.py::test_voxel_grad_oracle_matches_reference_fd.
"""
from __future__ import annotations

import numpy as np
import torch

from . import volray_oracle as vo


def segment_packet_t(t0, t1, sigma, rgb):
    """Torch version of volray_oracle.segment_packet (quadrature.py:141-188)."""
    mids = 0.5 * (t0 + t1)
    alpha = 1.0 - torch.exp(-sigma * (t1 - t0))
    keep = torch.cat([torch.ones(1, dtype=sigma.dtype), 1.0 - alpha])
    trans = torch.cumprod(keep, 0)
    w = trans[:-1] * alpha
    C = (w[:, None] * rgb).sum(0)
    gaps = (mids[:, None] - mids[None, :]).abs()
    L = w @ gaps @ w
    return trans[-1], C, w.sum(), (w * mids).sum(), L


def fold_t(packets):
    T = torch.ones((), dtype=torch.float64)
    A = torch.zeros((), dtype=torch.float64)
    D = torch.zeros((), dtype=torch.float64)
    L = torch.zeros((), dtype=torch.float64)
    C = torch.zeros(3, dtype=torch.float64)
    for (Tk, Ck, Ak, Dk, Lk) in packets:
        L = L + T * T * Lk + 2.0 * T * (Dk * A - Ak * D)
        C = C + T * Ck
        A = A + T * Ak
        D = D + T * Dk
        T = T * Tk
    return C, A, D, T, L


def voxel_eval_t(doc, dens_t, pts):
    """Differentiable trilinear/nearest voxel lookup w.r.t. the density tensor."""
    ids, ws, nearest, inside = vo.voxel_stencil(doc, pts)
    res = tuple(doc["resolution"])
    cols = np.asarray(doc["colors"], dtype=np.float64).reshape(res + (3,))
    flat = dens_t.reshape(-1)
    if doc.get("interpolation", "trilinear") == "nearest":
        lin = (nearest[:, 0] * res[1] + nearest[:, 1]) * res[2] + nearest[:, 2]
        sig = flat[torch.from_numpy(lin)]
        rgb = cols[nearest[:, 0], nearest[:, 1], nearest[:, 2]]
    else:
        sig = torch.zeros(pts.shape[0], dtype=torch.float64)
        rgb = np.zeros((pts.shape[0], 3))
        for c in range(8):
            ix = ids[:, c]
            lin = (ix[:, 0] * res[1] + ix[:, 1]) * res[2] + ix[:, 2]
            sig = sig + flat[torch.from_numpy(lin)] * torch.from_numpy(ws[:, c])
            rgb = rgb + cols[ix[:, 0], ix[:, 1], ix[:, 2]] * ws[:, c][:, None]
    mask = torch.from_numpy(inside.astype(np.float64))
    sig = sig * mask
    rgb = np.where(inside[:, None], np.clip(rgb, 0.0, 1.0), 0.0)
    return sig, torch.from_numpy(rgb)


def field_loss(tree: vo.Tree, eval_t, rays, targets, bg, dt, lambda_dist=1.0):
    """Loss over rays (R, 8) with a differentiable owner field
    ``eval_t(tile, pts (n,3) float64 numpy, dir (3,)) -> (sigma (n,), rgb (n,3)) torch``.
    Returns (loss, per-ray (C, A, D, T, L) numpy array (R, 7))."""
    total = torch.zeros((), dtype=torch.float64)
    outs = np.zeros((len(rays), 7))
    bg_t = torch.as_tensor(np.asarray(bg, dtype=np.float64))
    for i, r in enumerate(rays):
        o, d, tn, tf = r[0:3], r[3:6], r[6], r[7]
        t0, t1, tile = vo.sample_ray(tree, o, d, tn, tf, dt)
        packets = []
        for k in sorted(set(tile.tolist())):
            sel = np.nonzero(tile == k)[0]
            a, b = t0[sel], t1[sel]
            mids = 0.5 * (a + b)
            pts = np.asarray(o) + mids[:, None] * np.asarray(d)
            sig, rgb = eval_t(k, pts, np.asarray(d))
            start = 0
            for j in range(1, len(sel) + 1):
                if j == len(sel) or a[j] != b[j - 1]:
                    pk = segment_packet_t(torch.from_numpy(a[start:j]), torch.from_numpy(b[start:j]),
                                          sig[start:j], rgb[start:j])
                    packets.append((float(a[start]), k, pk))
                    start = j
        packets.sort(key=lambda s: (s[0], s[1]))
        C, A, D, T, L = fold_t([p[2] for p in packets])
        pix = C + T * bg_t
        err = pix - torch.as_tensor(np.asarray(targets[i], dtype=np.float64))
        total = total + (err * err).sum() + lambda_dist * L
        outs[i] = [C[0].item(), C[1].item(), C[2].item(), A.item(), D.item(), T.item(), L.item()]
    return total, outs


def field_loss_interlevel(tree: vo.Tree, eval_t, prop_t, rays, targets, bg, dt,
                          lambda_dist=1.0, lambda_int=1.0, eps=1e-7):
    """field_loss plus the interlevel (proposal) loss of csrc/interlevel.cu — PARITY
    UNPINNED (no reference code).  ``prop_t`` has eval_t's signature (its sigma is used).

        L_int = lambda_int * sum_i max(0, w_i - wh_i)^2 / (w_i + eps)
        w_i  = sg(P_s) T_i alpha_i   (stop-gradient: trains the proposal only)
        wh_i = sg(Ph_s) Th_i alphah_i
    P_s / Ph_s: NeRF / proposal transmittance in front of segment s (constants, like
    peers' packets in NeRF-XL).  Returns (main + interlevel loss, outs, interlevel part)."""
    main, outs = field_loss(tree, eval_t, rays, targets, bg, dt, lambda_dist)
    total = torch.zeros((), dtype=torch.float64)
    for r in rays:
        o, d, tn, tf = r[0:3], r[3:6], r[6], r[7]
        t0, t1, tile = vo.sample_ray(tree, o, d, tn, tf, dt)
        segs = []
        for k in sorted(set(tile.tolist())):
            sel = np.nonzero(tile == k)[0]
            segs.append((float(t0[sel[0]]), k, sel))
        segs.sort(key=lambda x: (x[0], x[1]))
        P = 1.0
        Ph = 1.0
        for _, k, sel in segs:
            a, b = t0[sel], t1[sel]
            mids = 0.5 * (a + b)
            pts = np.asarray(o) + mids[:, None] * np.asarray(d)
            sig, _ = eval_t(k, pts, np.asarray(d))
            sigh, _ = prop_t(k, pts, np.asarray(d))
            dl = torch.from_numpy(b - a)
            alpha = 1.0 - torch.exp(-sig.detach() * dl)
            Tl = torch.cumprod(torch.cat([torch.ones(1, dtype=torch.float64), 1.0 - alpha]), 0)
            w = P * Tl[:-1] * alpha
            alphah = 1.0 - torch.exp(-sigh * dl)
            Thl = torch.cumprod(torch.cat([torch.ones(1, dtype=torch.float64), 1.0 - alphah]), 0)
            wh = Ph * Thl[:-1] * alphah
            dd = torch.clamp(w - wh, min=0.0)
            total = total + lambda_int * (dd * dd / (w + eps)).sum()
            P = P * float(Tl[-1])
            Ph = Ph * float(Thl[-1].detach())
    return main + total, outs, total


class RayRuns:
    """Sample geometry of a ray batch under the tile protocol (volray_oracle.sample_ray per
    ray: distsim.py:369-373 + :406-414), grouped for batched field evaluation.

    pts[k], dirs[k]: every point owned by region k over the whole batch (float64);
    segs: one row per contiguous run (quadrature.py:191-206) = (ray, order_t, tile,
    global sample start, length); a segment's samples are [start, start+length) of the
    region-concatenated sample arrays t0 / t1 (regions in tile order)."""

    def __init__(self, tree: vo.Tree, rays, dt, occ=None):
        rays = np.asarray(rays, dtype=np.float64)
        per = {k: ([], [], [], []) for k in range(tree.n_leaves)}  # pts, dirs, t0, t1
        raw = []  # (ray, order_t, tile, local start, length)
        fill = {k: 0 for k in range(tree.n_leaves)}
        for i, r in enumerate(rays):
            o, d = r[0:3], r[3:6]
            t0, t1, tile = vo.sample_ray(tree, o, d, r[6], r[7], dt, occ)
            for k in sorted(set(tile.tolist())):
                sel = np.nonzero(tile == k)[0]
                a, b = t0[sel], t1[sel]
                mids = 0.5 * (a + b)
                P, Dd, A0, B0 = per[k]
                P.append(o + mids[:, None] * d)
                Dd.append(np.broadcast_to(d, (len(sel), 3)))
                A0.append(a)
                B0.append(b)
                start = 0
                for j in range(1, len(sel) + 1):
                    if j == len(sel) or a[j] != b[j - 1]:
                        raw.append((i, float(a[start]), k, fill[k] + start, j - start))
                        start = j
                fill[k] += len(sel)
        self.n_rays = len(rays)
        self.regions = [k for k in range(tree.n_leaves) if fill[k]]
        cat = lambda xs, w: np.concatenate(xs) if xs else np.zeros((0,) + w)  # noqa: E731
        self.pts = {k: cat(per[k][0], (3,)) for k in self.regions}
        self.dirs = {k: cat(per[k][1], (3,)) for k in self.regions}
        base, b = {}, 0
        for k in range(tree.n_leaves):
            base[k] = b
            b += fill[k]
        self.n_samples = b
        self.t0 = np.concatenate([cat(per[k][2], ()) for k in range(tree.n_leaves)] or [np.zeros(0)])
        self.t1 = np.concatenate([cat(per[k][3], ()) for k in range(tree.n_leaves)] or [np.zeros(0)])
        self.segs = [(i, ot, k, base[k] + s, n) for (i, ot, k, s, n) in raw]


def _padded(runs: RayRuns, values: torch.Tensor):
    """[S, Lmax(, c)] view of per-sample values per segment, plus the validity mask."""
    S = len(runs.segs)
    lmax = max((s[4] for s in runs.segs), default=1)
    start = np.array([s[3] for s in runs.segs], dtype=np.int64)
    length = np.array([s[4] for s in runs.segs], dtype=np.int64)
    ar = np.arange(lmax)
    mask = ar[None, :] < length[:, None]
    idx = np.where(mask, start[:, None] + ar[None, :], start[:, None])
    return values[torch.from_numpy(idx)], torch.from_numpy(mask), idx, mask


def _segment_packets(runs: RayRuns, sig_all, rgb_all, chunk_elems=1 << 24):
    """composite_samples (quadrature.py:141-165) + distortion_bruteforce
    (quadrature.py:179-188) of every segment at once: (T, C[S,3], A, D, L, w[S,Lmax])."""
    sig, maskt, idx, mask = _padded(runs, sig_all)
    rgb = rgb_all[torch.from_numpy(idx)]
    t0 = runs.t0[idx]
    t1 = runs.t1[idx]
    delta = torch.from_numpy(np.where(mask, t1 - t0, 0.0))
    mids = 0.5 * (t0 + t1)
    alpha = 1.0 - torch.exp(-sig * delta)
    keep = torch.cat([torch.ones((alpha.shape[0], 1), dtype=torch.float64), 1.0 - alpha], 1)
    trans = torch.cumprod(keep, 1)
    w = trans[:, :-1] * alpha * maskt
    C = (w[:, :, None] * rgb).sum(1)
    A = w.sum(1)
    D = (w * torch.from_numpy(mids)).sum(1)
    lmax = w.shape[1]
    step = max(1, chunk_elems // max(lmax * lmax, 1))
    Ls = []
    for s0 in range(0, w.shape[0], step):
        m = mids[s0:s0 + step]
        gaps = torch.from_numpy(np.abs(m[:, :, None] - m[:, None, :]))
        ws = w[s0:s0 + step]
        Ls.append(torch.einsum("si,sij,sj->s", ws, gaps, ws))
    L = torch.cat(Ls) if Ls else torch.zeros(0, dtype=torch.float64)
    return trans[:, -1], C, A, D, L, w, maskt, delta


def _eval_regions(runs: RayRuns, eval_batch):
    sig, rgb = [], []
    for k in runs.regions:
        s, c = eval_batch(k, runs.pts[k], runs.dirs[k])
        sig.append(s)
        rgb.append(c)
    return torch.cat(sig), torch.cat(rgb)


def field_loss_batched(tree: vo.Tree, eval_batch, rays, targets, bg, dt, lambda_dist=1.0,
                       prop_batch=None, lambda_int=0.0, eps=1e-7, runs: RayRuns | None = None,
                       keep: dict | None = None):
    """field_loss (and field_loss_interlevel with ``prop_batch``) over a whole ray batch:
    the same per-segment arithmetic (composite_samples, the O(N^2) distortion, the
    compose_render / compose_distortion fold in (order_t, tile) order, segrender.py:93-142,
    the probe's loss segrender.py:198-207), with each region's field evaluated ONCE over
    all its points — ``eval_batch(tile, pts (n,3), dirs (n,3)) -> (sigma (n,), rgb (n,3))``
    torch float64 — so C1-sized batches (4096 rays, 265k samples) finish in seconds.
    keep (optional dict): receives the field outputs "sig", "rgb" (and the proposal's
    "sigh"), concatenated over runs.regions, so a caller can take the loss's gradient
    with respect to them (the upstream of the field backward).
    Returns (loss, outs (R,7) numpy [C, A, D, T, L], interlevel part or None)."""
    runs = runs if runs is not None else RayRuns(tree, rays, dt)
    R = runs.n_rays
    outs = np.zeros((R, 7))
    outs[:, 5] = 1.0
    if not runs.segs:
        z = torch.zeros((), dtype=torch.float64)
        return z, outs, (z if prop_batch is not None else None)
    sig_all, rgb_all = _eval_regions(runs, eval_batch)
    if keep is not None:
        keep["sig"], keep["rgb"] = sig_all, rgb_all
    Tk, Ck, Ak, Dk, Lk, wk, maskt, delta = _segment_packets(runs, sig_all, rgb_all)
    # per ray: its segments in (order_t, tile) order (_compose_tile, distsim.py:376-382)
    order = sorted(range(len(runs.segs)), key=lambda s: (runs.segs[s][0], runs.segs[s][1],
                                                         runs.segs[s][2]))
    per_ray = [[] for _ in range(R)]
    for s in order:
        per_ray[runs.segs[s][0]].append(s)
    kmax = max(len(p) for p in per_ray)
    S = len(runs.segs)
    slot = np.full((R, kmax), S, dtype=np.int64)  # S = the identity packet
    for i, p in enumerate(per_ray):
        slot[i, :len(p)] = p
    one = torch.ones(1, dtype=torch.float64)
    zero = torch.zeros(1, dtype=torch.float64)
    Tp = torch.cat([Tk, one])
    Ap, Dp, Lp = (torch.cat([x, zero]) for x in (Ak, Dk, Lk))
    Cp = torch.cat([Ck, torch.zeros((1, 3), dtype=torch.float64)])
    T = torch.ones(R, dtype=torch.float64)
    A = torch.zeros(R, dtype=torch.float64)
    D = torch.zeros(R, dtype=torch.float64)
    L = torch.zeros(R, dtype=torch.float64)
    C = torch.zeros((R, 3), dtype=torch.float64)
    prefix = torch.ones(S + 1, dtype=torch.float64)  # NeRF transmittance before a segment
    for j in range(kmax):
        sj = torch.from_numpy(slot[:, j])
        L = L + T * T * Lp[sj] + 2.0 * T * (Dp[sj] * A - Ap[sj] * D)
        C = C + T[:, None] * Cp[sj]
        A = A + T * Ap[sj]
        D = D + T * Dp[sj]
        prefix = prefix.index_copy(0, sj, T.detach())
        T = T * Tp[sj]
    pix = C + T[:, None] * torch.as_tensor(np.asarray(bg, dtype=np.float64))
    err = pix - torch.as_tensor(np.asarray(targets, dtype=np.float64))
    loss = (err * err).sum() + lambda_dist * L.sum()
    outs = np.concatenate([C.detach().numpy(), A.detach().numpy()[:, None],
                           D.detach().numpy()[:, None], T.detach().numpy()[:, None],
                           L.detach().numpy()[:, None]], axis=1)
    if prop_batch is None:
        return loss, outs, None
    # interlevel (csrc/interlevel.cu; PARITY UNPINNED): w = sg(P_s T_i alpha_i) with the
    # NeRF's own sigma, wh = sg(Ph_s) Th_i alphah_i with the proposal's
    sigh_all, _ = _eval_regions(runs, prop_batch)
    if keep is not None:
        keep["sigh"] = sigh_all
    sigh, _, _, _ = _padded(runs, sigh_all)
    alphah = 1.0 - torch.exp(-sigh * delta)
    keeph = torch.cat([torch.ones((alphah.shape[0], 1), dtype=torch.float64), 1.0 - alphah], 1)
    transh = torch.cumprod(keeph, 1)
    wh_loc = transh[:, :-1] * alphah * maskt
    Thp = torch.cat([transh[:, -1].detach(), one])
    Ph = torch.ones(R, dtype=torch.float64)
    prefh = torch.ones(S + 1, dtype=torch.float64)
    for j in range(kmax):
        sj = torch.from_numpy(slot[:, j])
        prefh = prefh.index_copy(0, sj, Ph)
        Ph = Ph * Thp[sj]
    w = (prefix[:S, None] * wk).detach()
    wh = prefh[:S, None] * wh_loc
    dd = torch.clamp(w - wh, min=0.0)
    if keep is not None:  # per-sample w and wh (the clamp's kink is at w == wh)
        _, _, idx, msk = _padded(runs, sigh_all)
        for key, v in (("w", w), ("wh", wh)):
            out = np.zeros(runs.n_samples)
            out[idx[msk]] = v.detach().numpy()[msk]
            keep[key] = out
    il = lambda_int * (dd * dd / (w + eps) * maskt).sum()
    return loss + il, outs, il


def voxel_loss(tree: vo.Tree, grid_doc: dict, region_dens, rays, targets, bg, dt,
               lambda_dist=1.0):
    """Loss with a private density copy per region (segrender.py:175-178);
    ``region_dens``: list of float64 torch tensors (one per leaf)."""
    return field_loss(tree, lambda k, pts, d: voxel_eval_t(grid_doc, region_dens[k], pts),
                      rays, targets, bg, dt, lambda_dist)
