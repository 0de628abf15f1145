#!/bin/bash
# bench.py at N=2 (two ranks sharing cuda:0 over gloo: plumbing, not a measurement)
set -u
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29577 bench.py --gpus 2 --same-device --backend gloo --config c3 --sub none \
  --steps 2 --warmup 1 --burnin 2 --no-cpu > gpurun_out/n2.log 2>&1
echo "rc=$?"
tail -1 gpurun_out/n2.log | cut -c1-600
