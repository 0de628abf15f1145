"""Time individual C-ABI kernels on synthetic inputs (CUDA events, warm)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200 import _lib as L

DEV = "cuda:0"


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
g = torch.Generator(device="cpu").manual_seed(0)
w16 = vr.fields.init_mlp_weights(g).to(DEV).half()
enc = (torch.randn((16, n, 2), device=DEV) * 0.5).half().contiguous()
R = n // 64
d = torch.randn((R, 3), dtype=torch.float64, device=DEV)
d = d / d.norm(dim=1, keepdim=True)
rays = torch.zeros((8, R), dtype=torch.float64, device=DEV)
rays[3:6] = d.T
rid = (torch.arange(n, device=DEV, dtype=torch.int32) // 64).contiguous()
out = torch.empty((n, 4), device=DEV)
dsr = torch.randn((n, 4), device=DEV) * 0.1
gw = torch.zeros(L.VR_MLP_NPARAMS, device=DEV)
de = torch.empty((16, n, 2), device=DEV)
err = torch.zeros(1, dtype=torch.int32, device=DEV)
s = L.stream_ptr()
f = lambda: L.call("vr_mlp_fwd_tc", L.ptr(w16), L.ptr(enc), L.ptr(rays), R, L.ptr(rid), n, L.ptr(out), s)
bw = lambda: L.call("vr_mlp_bwd_tc", L.ptr(w16), L.ptr(enc), L.ptr(rays), R, L.ptr(rid), n, L.ptr(dsr), None,
                    L.ptr(gw), L.ptr(de), L.ptr(err), 0, s)
tf = timeit(f)
tb = timeit(bw)
print(f"n={n}: mlp_fwd_tc {tf:.3f} ms ({n*18816/tf/1e9:.1f} TFLOP/s)  "
      f"mlp_bwd_tc {tb:.3f} ms ({n*3*18816/tb/1e9:.1f} TFLOP/s)  err={err.item()}")
