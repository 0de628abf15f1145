"""Step-time drift of the training step: same resident batch vs distinct batches per step.

    python scripts/drift.py --config c3 --steps 60 --batches 8 [--lr 1e-2]

Prints one line per step (ms, loss) so the steady state can be read off.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_16221_b200.workloads import CONFIGS, make_rays, make_targets  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--batches", type=int, default=8)
    ap.add_argument("--lr", type=float, default=1e-2)
    args = ap.parse_args()
    w = CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    pool = bench.build_pool(w, 0, 1, dev, None)
    R = w.n_rays
    batches = [(torch.from_numpy(make_rays(w, seed=s)).to(dev),
                torch.from_numpy(make_targets(R, seed=100 + s)).to(dev))
               for s in range(args.batches)]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    losses = []
    ev[0].record()
    for k in range(args.steps):
        r, t = batches[k % len(batches)]
        losses.append(pool.train_step(r, t, w.dt, lr=args.lr, step=k + 1,
                                      lambda_interlevel=w.interlevel))
        ev[k + 1].record()
    torch.cuda.synchronize()
    for k in range(args.steps):
        print(f"{args.config} step {k:3d} {ev[k].elapsed_time(ev[k + 1]):8.2f} ms  "
              f"loss {losses[k].item():.4e}", flush=True)


if __name__ == "__main__":
    main()
