"""K1 of two builds (VR_LIB_PATH=<old .so> vs the in-tree one) on the c3 / c4 / c5 batches:
digests of every output (t0, t1, ray_id, offsets, seg_first, ray_te) must be equal.
    python scripts/check_k1_ab.py            # runs both builds in subprocesses"""
import json
import os
import subprocess
import sys

sys.path.insert(0, ".")


def digest(t):
    import torch
    v = t.contiguous().view(-1)
    v = v.view(torch.int64) if v.element_size() == 8 else v.view(torch.int32).to(torch.int64)
    w = torch.arange(1, v.numel() + 1, device=v.device, dtype=torch.int64)
    return [int(v.sum()), int((v * w).sum()), int(v.numel())]


def run():
    import bench
    import torch
    from paper_2404_16221_b200.workloads import CONFIGS, make_rays
    out = {}
    for cfg in ("c3", "c4", "c5"):
        w = CONFIGS[cfg]
        pool = bench.build_pool(w, 0, 1, "cuda:0", None)
        for seed in (0, 1):
            rays = pool.rays_to_device(make_rays(w, seed=seed))
            b = pool.sample(rays, w.dt)
            n = b.n_samples
            out[f"{cfg}/{seed}"] = [digest(b.t0[:n]), digest(b.t1[:n]), digest(b.ray_id[:n]),
                                    digest(b.offsets), digest(b.seg_first), digest(b.ray_te)]
        del pool
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--run":
        run()
        sys.exit(0)
    res = []
    for env in ({"VR_LIB_PATH": sys.argv[1]} if len(sys.argv) > 1 else {}, {}):
        r = subprocess.run([sys.executable, __file__, "--run"], env={**os.environ, **env},
                           capture_output=True, text=True)
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    same = res[0] == res[1]
    for k in res[1]:
        print(k, "equal" if res[0][k] == res[1][k] else f"DIFFERENT {res[0][k]} {res[1][k]}")
    print("K1 outputs bit-identical" if same else "MISMATCH")
