"""Where the render e2e time goes: the bench's e2e loop with parts switched off."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2404_16221_b200 as vr
from paper_2404_16221_b200.workloads import CONFIGS, make_rays

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
dev = torch.device("cuda", 0)
pool = bench.build_pool(w, 0, 1, dev, None)
rays_np = make_rays(w)
R = rays_np.shape[1]
rays_h = torch.from_numpy(rays_np).pin_memory()
rays_d = rays_h.to(dev)
out_h = torch.empty((3, R), dtype=torch.float32, pin_memory=True)
copy_stream = torch.cuda.Stream(device=dev)
main = torch.cuda.current_stream()


def step(r, d2h):
    out, _ = pool.render_rays(r, w.dt)
    if d2h:
        out_h.copy_(out[0:3], non_blocking=True)
        main.synchronize()


def run(h2d, d2h, steps=8):
    for _ in range(3):
        step(rays_d, d2h)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    nxt = None
    for k in range(steps):
        if h2d:
            if nxt is None:
                with torch.cuda.stream(copy_stream):
                    nxt = (rays_h.to(dev, non_blocking=True), torch.cuda.Event())
                    nxt[1].record(copy_stream)
            r, ev = nxt
            main.wait_event(ev)
            r.record_stream(main)
            with torch.cuda.stream(copy_stream):
                nxt = (rays_h.to(dev, non_blocking=True), torch.cuda.Event())
                nxt[1].record(copy_stream)
        else:
            r = rays_d
        step(r, d2h)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


for h2d, d2h in ((False, False), (False, True), (True, False), (True, True)):
    print(f"h2d={h2d} d2h={d2h}: {run(h2d, d2h):.2f} ms/step", flush=True)
