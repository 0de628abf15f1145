"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.  PARITY UNPINNED.

Restatement of the per-region NeRF-XL model that the reference does not implement:
an Instant-NGP multiresolution hash grid (named only at PAPER.md:386-388) feeding a
density MLP and a view-conditioned colour MLP.  No reference code,
third-party source or golden vector exists for it, so this file
IS the specification the CUDA kernels are checked against:

  * hash-table indices are bit-exact (numpy uint32 / float32 with the kernel's op order);
  * features and MLP activations use the kernel's fp16 quantisation points, computed
    here in float64 (straight-through for gradients);
  * gradients come from torch float64 autograd.

Level parameters are derived here independently of the product's host code.
"""
from __future__ import annotations

import math

import numpy as np
import torch

PRIMES = (1, 2654435761, 805459861)

# packed MLP layout (include/vr_capi.h VR_MLP_*)
W1D, W2D, W1C, W2C, W3C = 0, 2048, 3072, 5120, 9216
NPARAMS = 10240

SH_C = (0.28209479177387814, 0.48860251190291987, 1.0925484305920792, 0.94617469575755997,
        0.31539156525251999, 0.54627421529603959, 0.59004358992664352, 2.8906114426405538,
        0.45704579946446572, 0.3731763325901154, 1.4453057213202769)


def levels(log2_T: int, n_levels: int = 16, base_res: int = 16, max_res: int = 2048):
    """[(scale float32, res, dense, offset)] and total entries."""
    growth = math.exp((math.log(max_res) - math.log(base_res)) / max(n_levels - 1, 1))
    T = 1 << log2_T
    out, off = [], 0
    for lv in range(n_levels):
        scale = np.float32(base_res * growth ** lv - 1.0)
        res = int(math.ceil(float(scale))) + 2
        dense = res ** 3 <= T
        size = ((res ** 3 if dense else T) + 7) // 8 * 8
        out.append((scale, res, dense, off))
        off += size
    return out, off


def normalize(pts, box_mn, box_mx):
    """float32 of (p - mn) / (mx - mn), computed in float64 (kernel norm_pos)."""
    mn = np.asarray(box_mn, dtype=np.float64)
    mx = np.asarray(box_mx, dtype=np.float64)
    return ((np.asarray(pts, dtype=np.float64) - mn) / (mx - mn)).astype(np.float32)


def corners(u32, scale, res, dense, log2_T):
    """Corner indices (n,8) uint32 and weights (n,8) float32 of one level."""
    u32 = np.asarray(u32, dtype=np.float32)
    pos = (u32 * np.float32(scale)).astype(np.float32) + np.float32(0.5)
    g = np.floor(pos).astype(np.int64)
    g = np.clip(g, 0, res - 2)
    frac = (pos - g.astype(np.float32)).astype(np.float32)
    idx = np.empty((u32.shape[0], 8), dtype=np.uint32)
    w = np.empty((u32.shape[0], 8), dtype=np.float32)
    mask = np.uint32((1 << log2_T) - 1)
    one = np.float32(1.0)
    for c in range(8):
        bits = np.array([c & 1, (c >> 1) & 1, (c >> 2) & 1])
        xyz = (g + bits).astype(np.uint32)
        if dense:
            r = np.uint32(res)
            idx[:, c] = xyz[:, 0] + r * (xyz[:, 1] + r * xyz[:, 2])
        else:
            h = (xyz[:, 0] * np.uint32(PRIMES[0])) ^ (xyz[:, 1] * np.uint32(PRIMES[1])) ^ \
                (xyz[:, 2] * np.uint32(PRIMES[2]))
            idx[:, c] = h & mask
        wa = [frac[:, a] if bits[a] else (one - frac[:, a]).astype(np.float32) for a in range(3)]
        w[:, c] = ((wa[0] * wa[1]).astype(np.float32) * wa[2]).astype(np.float32)
    return idx, w


def feature32(w, vals):
    """The kernel's float32 feature of one level: corners with cx = 0 (c = 0, 2, 4, 6) and
    cx = 1 (c = 1, 3, 5, 7) each summed in that order from 0 (round-to-nearest, no FMA),
    then added (csrc/hashgrid.cuh gather_half / gather_level).  w (n, 8) float32, vals
    (n, 8, 2) float32."""
    halves = []
    for p in (0, 1):
        acc = np.zeros((w.shape[0], 2), dtype=np.float32)
        for c in range(p, 8, 2):
            acc = (acc + (w[:, c:c + 1] * vals[:, c]).astype(np.float32)).astype(np.float32)
        halves.append(acc)
    return (halves[0] + halves[1]).astype(np.float32)


def all_indices(pts, box_mn, box_mx, log2_T, max_res=2048):
    """Per-level corner indices [L][n][8] int64 (for the bit-exact parity test)."""
    lv, _ = levels(log2_T, max_res=max_res)
    u = normalize(pts, box_mn, box_mx)
    return np.stack([corners(u, s, r, dn, log2_T)[0].astype(np.int64) for (s, r, dn, _) in lv])


def _q16(x: torch.Tensor) -> torch.Tensor:
    """fp16 rounding, straight-through for gradients."""
    return x + (x.to(torch.float16).to(torch.float64) - x).detach()


def sh16_t(d: torch.Tensor) -> torch.Tensor:
    x, y, z = d[..., 0], d[..., 1], d[..., 2]
    c = SH_C
    xy, xz, yz, x2, y2, z2 = x * y, x * z, y * z, x * x, y * y, z * z
    return torch.stack([
        torch.full_like(x, c[0]), -c[1] * y, c[1] * z, -c[1] * x,
        c[2] * xy, -c[2] * yz, c[3] * z2 - c[4], -c[2] * xz,
        c[5] * x2 - c[5] * y2, c[6] * y * (-3.0 * x2 + y2), c[7] * xy * z,
        c[8] * y * (1.0 - 5.0 * z2), c[9] * z * (5.0 * z2 - 3.0), c[8] * x * (1.0 - 5.0 * z2),
        c[10] * z * (x2 - y2), c[6] * x * (-x2 + 3.0 * y2)], dim=-1)


class HashMLPModel:
    """One region's model with float64 torch parameters (table, packed weights)."""

    def __init__(self, table: np.ndarray, weights: np.ndarray, log2_T: int, box_mn, box_mx,
                 max_res: int = 2048, quantize: bool = True):
        self.table = torch.tensor(np.asarray(table, dtype=np.float64), requires_grad=True)
        # the kernels consume fp16 copies of the float32 master weights; quantize=False is
        # the ideal float64 model (no fp16 weights/activations, float64 features): it bounds
        # the quantisation error of the kernels' precision choice separately from parity
        self.quantize = quantize
        w = np.asarray(weights, dtype=np.float32)
        w = w.astype(np.float16).astype(np.float64) if quantize else w.astype(np.float64)
        self.weights = torch.tensor(w, requires_grad=True)
        self.log2_T = log2_T
        self.box_mn, self.box_mx = box_mn, box_mx
        self.max_res = max_res
        self.levels, self.n_entries = levels(log2_T, max_res=max_res)

    def encode(self, pts) -> torch.Tensor:
        """(n, 32) features, fp16-rounded."""
        u = normalize(pts, self.box_mn, self.box_mx)
        feats = []
        tab32 = self.table.detach().numpy().astype(np.float32)
        for (scale, res, dense, off) in self.levels:
            idx, w = corners(u, scale, res, dense, self.log2_T)
            gidx = idx.astype(np.int64) + off
            rows = self.table[torch.from_numpy(gidx)]  # (n, 8, 2)
            f = (rows * torch.from_numpy(w.astype(np.float64))[:, :, None]).sum(1)
            if self.quantize:
                # forward value: the kernel's float32 sum (bit-exact, feature32 order);
                # gradient: the exact linear map
                f32 = feature32(w, tab32[gidx])
                f = f + (torch.from_numpy(f32.astype(np.float64)) - f).detach()
            feats.append(f)
        return self._q(torch.cat(feats, dim=1))

    def _q(self, x: torch.Tensor) -> torch.Tensor:
        return _q16(x) if getattr(self, "quantize", True) else x

    def _linear(self, a: torch.Tensor, Wm: torch.Tensor) -> torch.Tensor:
        """a @ Wm^T, recorded (output with its gradient retained, input) so weight_contrib
        can size each weight gradient's terms."""
        x = a @ Wm.T
        if x.requires_grad:
            x.retain_grad()
        self._layers.append((x, a))
        return x

    def weight_contrib(self) -> np.ndarray:
        """Per packed weight: sum over samples of |dL/d(layer output)| * |layer input| —
        the magnitude of the terms its gradient sums (of the last backward through the last
        mlp() call; layers in the packed order W1d, W2d, W1c, W2c, W3c)."""
        S = np.zeros(NPARAMS)
        offs = [W1D, W2D, W1C, W2C, W3C]
        for (x, a), off in zip(self._layers, offs):
            if x.grad is None:
                continue
            m = (x.grad.abs().T @ a.detach().abs()).numpy()
            S[off:off + m.size] = m.ravel()
        return S

    def clear_layer_grads(self):
        for x, _ in getattr(self, "_layers", []):
            x.grad = None

    def _relu(self, a: torch.Tensor, Wm: torch.Tensor, margins: list) -> torch.Tensor:
        """fp16(relu(a @ Wm^T)) with the kernels' derivative: 1 where the fp16 activation
        is non-zero (csrc/mlp_tc.cu relu_mask8).  Records each row's relative kink margin
        min_j |x_j| / sum_i |a_i W_ji|: where it is below the float32 accumulation error
        (~K * 2^-24), float32 and float64 can take different sides of the ReLU kink."""
        x = self._linear(a, Wm)
        with torch.no_grad():
            mag = a.detach().abs() @ Wm.detach().abs().T
            margins.append((x.detach().abs() / mag.clamp_min(1e-300)).min(1).values)
        if not getattr(self, "quantize", True):
            return torch.relu(x)
        hq = torch.relu(x).detach().to(torch.float16).to(torch.float64)
        keep = (hq != 0).to(torch.float64)
        return x * keep + (hq - x * keep).detach()

    def mlp(self, enc: torch.Tensor, dirs32: np.ndarray):
        _q16 = self._q  # noqa: N806 - the quantisation points of the kernels
        margins = []
        self._layers = []
        W = self.weights
        W1d = W[W1D:W2D].reshape(64, 32)
        W2d = W[W2D:W1C].reshape(16, 64)
        W1c = W[W1C:W2C].reshape(64, 32)
        W2c = W[W2C:W3C].reshape(64, 64)
        W3c = W[W3C:W3C + 3 * 64].reshape(3, 64)
        h = self._relu(enc, W1d, margins)
        od = self._linear(h, W2d)
        x0 = od[:, 0]
        inside = ((x0 > -15.0) & (x0 < 15.0)).to(torch.float64)
        # exp(clamp(x)) with d/dx = sigma inside the clamp range, 0 outside
        xc = torch.clamp(x0, -15.0, 15.0)
        sigma = torch.exp(x0 * inside + (xc * (1 - inside)).detach())
        sh = _q16(sh16_t(torch.from_numpy(np.asarray(dirs32, dtype=np.float32).astype(np.float64))))
        cin = torch.cat([_q16(od), sh], dim=1)
        h1 = self._relu(cin, W1c, margins)
        h2 = self._relu(h1, W2c, margins)
        rgb = torch.sigmoid(self._linear(h2, W3c))
        # per-sample relative ReLU kink margin of this call (see _relu)
        self.last_margin = torch.stack(margins).min(0).values.numpy()
        return sigma, rgb

    def eval_t(self, pts, d):
        n = np.asarray(pts).shape[0]
        dirs = np.broadcast_to(np.asarray(d, dtype=np.float64).astype(np.float32), (n, 3))
        return self.mlp(self.encode(pts), dirs)

    def eval_dirs(self, pts, dirs):
        """Batched evaluation with one view direction per point (grad_oracle.RayRuns).
        The encodings are kept (last_enc, gradient retained) so tests can compare the
        per-sample d(enc) of the kernels."""
        enc = self.encode(pts)
        enc.retain_grad()
        self.last_enc = enc
        self.last_pts = np.asarray(pts, dtype=np.float64)
        return self.mlp(enc, np.asarray(dirs, dtype=np.float64).astype(np.float32))

    def grads(self):
        return (self.table.grad.numpy().copy(), self.weights.grad.numpy().copy())


class CompactHashMLPModel(HashMLPModel):
    """The same model storing only the table entries a known point set touches.

    Used to time the CPU port on the big configs (T = 2^19..2^22 per region) without
    dense float64 tables and dense autograd gradients dominating the measurement;
    arithmetic is identical to HashMLPModel on those points."""

    def __init__(self, entry_init, weights, log2_T: int, box_mn, box_mx, pts, max_res: int = 2048):
        self.log2_T = log2_T
        self.box_mn, self.box_mx = box_mn, box_mx
        self.max_res = max_res
        self.levels, self.n_entries = levels(log2_T, max_res=max_res)
        u = normalize(pts, box_mn, box_mx)
        touched = [corners(u, s, r, dn, log2_T)[0].astype(np.int64).ravel() + off
                   for (s, r, dn, off) in self.levels]
        self.uniq = np.unique(np.concatenate(touched))
        table = np.asarray(entry_init(self.uniq), dtype=np.float64)
        self.table = torch.tensor(table, requires_grad=True)
        w16 = np.asarray(weights, dtype=np.float32).astype(np.float16).astype(np.float64)
        self.weights = torch.tensor(w16, requires_grad=True)

    def encode(self, pts) -> torch.Tensor:
        u = normalize(pts, self.box_mn, self.box_mx)
        feats = []
        tab32 = self.table.detach().numpy().astype(np.float32)
        for (scale, res, dense, off) in self.levels:
            idx, w = corners(u, scale, res, dense, self.log2_T)
            loc = np.searchsorted(self.uniq, idx.astype(np.int64) + off)
            rows = self.table[torch.from_numpy(loc)]
            f = (rows * torch.from_numpy(w.astype(np.float64))[:, :, None]).sum(1)
            f32 = feature32(w, tab32[loc])
            f = f + (torch.from_numpy(f32.astype(np.float64)) - f).detach()
            feats.append(f)
        return _q16(torch.cat(feats, dim=1))
