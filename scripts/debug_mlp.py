"""Diagnose tc vs CUDA-core MLP backward against a float64 torch reference."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib

DEV = "cuda:0"
L = _lib


def ref_fp64(w16, enc, dirs, dsr):
    W = w16.double()
    W1d = W[L.VR_MLP_W1D:L.VR_MLP_W2D].reshape(64, 32).requires_grad_()
    W2d = W[L.VR_MLP_W2D:L.VR_MLP_W1C].reshape(16, 64).requires_grad_()
    W1c = W[L.VR_MLP_W1C:L.VR_MLP_W2C].reshape(64, 32).requires_grad_()
    W2c = W[L.VR_MLP_W2C:L.VR_MLP_W3C].reshape(64, 64).requires_grad_()
    W3c = W[L.VR_MLP_W3C:L.VR_MLP_W3C + 192].reshape(3, 64).requires_grad_()
    x = enc.permute(1, 0, 2).reshape(-1, 32).double().requires_grad_()
    q = lambda t: t + (t.half().double() - t).detach()
    h = q(torch.relu(x @ W1d.T))
    od = h @ W2d.T
    sig = torch.exp(od[:, 0].clamp(-15, 15))
    d = dirs.float().double()
    X, Y, Z = d[:, 0], d[:, 1], d[:, 2]
    import math
    sh = torch.stack([torch.full_like(X, 0.28209479177387814), -0.48860251190291987 * Y, 0.48860251190291987 * Z,
                      -0.48860251190291987 * X, 1.0925484305920792 * X * Y, -1.0925484305920792 * Y * Z,
                      0.94617469575755997 * Z * Z - 0.31539156525251999, -1.0925484305920792 * X * Z,
                      0.54627421529603959 * (X * X - Y * Y), 0.59004358992664352 * Y * (-3 * X * X + Y * Y),
                      2.8906114426405538 * X * Y * Z, 0.45704579946446572 * Y * (1 - 5 * Z * Z),
                      0.3731763325901154 * Z * (5 * Z * Z - 3), 0.45704579946446572 * X * (1 - 5 * Z * Z),
                      1.4453057213202769 * Z * (X * X - Y * Y), 0.59004358992664352 * X * (-X * X + 3 * Y * Y)], 1)
    cin = torch.cat([q(od), q(sh)], 1)
    h1 = q(torch.relu(cin @ W1c.T))
    h2 = q(torch.relu(h1 @ W2c.T))
    rgb = torch.sigmoid(h2 @ W3c.T)
    out = torch.cat([sig[:, None], rgb], 1)
    (out * dsr.double()).sum().backward()
    g = torch.zeros(L.VR_MLP_NPARAMS, dtype=torch.float64, device=DEV)
    g[L.VR_MLP_W1D:L.VR_MLP_W2D] = W1d.grad.reshape(-1)
    g[L.VR_MLP_W2D:L.VR_MLP_W1C] = W2d.grad.reshape(-1)
    g[L.VR_MLP_W1C:L.VR_MLP_W2C] = W1c.grad.reshape(-1)
    g[L.VR_MLP_W2C:L.VR_MLP_W3C] = W2c.grad.reshape(-1)
    g[L.VR_MLP_W3C:L.VR_MLP_W3C + 192] = W3c.grad.reshape(-1)
    return out, g, x.grad


for n in (1000, 40000, 400000):
    g = torch.Generator(device="cpu").manual_seed(n)
    w16 = vr.fields.init_mlp_weights(g).to(DEV).half()
    enc = (torch.randn((16, n, 2), generator=g) * 0.5).half().to(DEV).contiguous()
    R = max(n // 7, 1)
    d = torch.randn((R, 3), generator=g, dtype=torch.float64)
    d = d / d.norm(dim=1, keepdim=True)
    rays = torch.zeros((8, R), dtype=torch.float64)
    rays[3:6] = d.T
    rays = rays.to(DEV)
    rid = torch.randint(0, R, (n,), generator=g, dtype=torch.int32).to(DEV)
    dsr = (torch.randn((n, 4), generator=g) * 0.1).to(DEV)
    s = L.stream_ptr()
    ref_out, ref_g, ref_x = ref_fp64(w16, enc, rays[3:6, rid.long()].T, dsr)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    blocks = [("W1d", L.VR_MLP_W1D, L.VR_MLP_W2D), ("W2d", L.VR_MLP_W2D, L.VR_MLP_W1C),
              ("W1c", L.VR_MLP_W1C, L.VR_MLP_W2C), ("W2c", L.VR_MLP_W2C, L.VR_MLP_W3C),
              ("W3c", L.VR_MLP_W3C, L.VR_MLP_W3C + 192)]
    for fw, bw in (("vr_mlp_fwd", "vr_mlp_bwd"), ("vr_mlp_fwd_tc", "vr_mlp_bwd_tc")):
        o = torch.empty((n, 4), dtype=torch.float32, device=DEV)
        L.call(fw, L.ptr(w16), L.ptr(enc), L.ptr(rays), R, L.ptr(rid), n, L.ptr(o), s)
        gw = torch.zeros(L.VR_MLP_NPARAMS, dtype=torch.float32, device=DEV)
        de = torch.empty((16, n, 2), dtype=torch.float32, device=DEV)
        args = [L.ptr(w16), L.ptr(enc), L.ptr(rays), R, L.ptr(rid), n, L.ptr(dsr)]
        if bw.endswith("_tc"):  # (no forward output: no gradient scaling; no row list)
            args += [None, L.ptr(gw), L.ptr(de), L.ptr(err), 0, None, None]
        else:
            args += [L.ptr(gw), L.ptr(de)]
        L.call(bw, *args, s)
        torch.cuda.synchronize()
        fo = ((o.double() - ref_out).abs().max()).item()
        de2 = de.permute(1, 0, 2).reshape(-1, 32).double()
        rx = ((de2 - ref_x).norm() / ref_x.norm()).item()
        parts = []
        for name, a, b in blocks:
            r = ((gw[a:b].double() - ref_g[a:b]).norm() / ref_g[a:b].norm()).item()
            parts.append(f"{name}={r:.2e}")
        print(f"n={n} {fw}: fwd maxabs={fo:.2e} denc rel={rx:.2e} " + " ".join(parts), flush=True)
    print("err flags", err.item())
