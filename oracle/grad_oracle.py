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


def voxel_loss(tree: vo.Tree, grid_doc: dict, region_dens, rays, targets, bg, dt,
               lambda_dist=1.0):
    """Loss with a private density copy per region (segrender.py:175-178);
    ``region_dens``: list of float64 torch tensors (one per leaf)."""
    return field_loss(tree, lambda k, pts, d: voxel_eval_t(grid_doc, region_dens[k], pts),
                      rays, targets, bg, dt, lambda_dist)
